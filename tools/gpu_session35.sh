#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "split or isect_is_exact" > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_HEAVY_FRAC=0.008,0.01,0.012,0.014 > gpurun_out/ab_post.jsonl 2> gpurun_out/ab_post.log
echo done
