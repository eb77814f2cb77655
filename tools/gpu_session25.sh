#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "split or isect_is_exact or golden" > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
for rs in 16 8; do SF_SPLIT_RS=$rs timeout 600 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 >> gpurun_out/ab_pp.jsonl 2>> gpurun_out/ab_pp.log; done
echo done
