#!/usr/bin/env bash
# GPU round-trip: u-walk combined cells (parity + A/B at C2 and C3-WN).
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "uwalk or generalized or weighted" > gpurun_out/pytest_nbo.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nbo.log
timeout 600 python tools/kernel_ab.py --config c2 --kernels 12 --reps 2 --env SF_UWALK_NBO=0,1 > gpurun_out/ab_nbo_c2.jsonl 2> gpurun_out/ab_nbo_c2.log
timeout 1200 python tools/kernel_ab.py --config c3wn --kernels 12 --reps 1 --env SF_UWALK_NBO=0,1 > gpurun_out/ab_nbo_c3wn.jsonl 2> gpurun_out/ab_nbo_c3wn.log
echo done
