#!/usr/bin/env bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "split or isect_is_exact" > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
for rs in 4 8 16; do SF_SPLIT_RS=$rs timeout 600 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 >> gpurun_out/ab_rs.jsonl 2>> gpurun_out/ab_rs.log; done
for f in 0.007 0.014; do SF_HEAVY_FRAC=$f timeout 600 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 >> gpurun_out/ab_frac.jsonl 2>> gpurun_out/ab_rs.log; done
echo done
