#!/usr/bin/env bash
# GPU round-trip: full parity suite; heavy threshold sweep x split variants.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 2000 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_HEAVY_FRAC=0.025,0.03,0.04,0.05,0.07 > gpurun_out/ab_heavy2.jsonl 2> gpurun_out/ab_heavy2.log
timeout 900 env SF_HEAVY_FRAC=0.03 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_SPLIT_VARIANT=0,6,7 > gpurun_out/ab_var.jsonl 2> gpurun_out/ab_var.log
echo done
