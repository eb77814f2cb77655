#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_HEAVY_FRAC=0.01,0.012,0.014 > gpurun_out/ab_fix.jsonl 2> gpurun_out/ab_fix.log
echo done
