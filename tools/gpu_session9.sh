#!/usr/bin/env bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "isect or golden" > gpurun_out/pytest_isect2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_isect2.log
timeout 600 python tools/kernel_ab.py --config small --kernels 5,6 --reps 3 > gpurun_out/ab_small2.jsonl 2> gpurun_out/ab_small2.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 5,6 --reps 2 > gpurun_out/ab_c3_2.jsonl 2> gpurun_out/ab_c3_2.log
echo done
