#!/usr/bin/env bash
# Intersection kernel (5): parity first, then A/B vs the sparse walk, then C3 bench.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "isect" > gpurun_out/pytest_isect.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_isect.log
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/kernel_ab.py --config small --kernels 2,5 --reps 3 > gpurun_out/ab_small.jsonl 2> gpurun_out/ab_small.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 2,5 --reps 2 > gpurun_out/ab_c3.jsonl 2> gpurun_out/ab_c3.log
echo done
