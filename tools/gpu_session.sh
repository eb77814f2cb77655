#!/usr/bin/env bash
# GPU round-trip: integer-limb heavy walk (parity + A/B).
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "split_variants" > gpurun_out/pytest_int.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_int.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 2 --env SF_SPLIT_VARIANT=0,16 > gpurun_out/ab_int.jsonl 2> gpurun_out/ab_int.log
echo done
