#!/usr/bin/env bash
# GPU round-trip: new split variants (parity + A/B), new medium-scale tests.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "split_variants or medium_scale or reference_order_walk" > gpurun_out/pytest_var.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_var.log
timeout 1200 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_SPLIT_VARIANT=0,11,12,13,14,15 > gpurun_out/ab_var3.jsonl 2> gpurun_out/ab_var3.log
echo done
