#!/usr/bin/env bash
mkdir -p gpurun_out
SF_DEBUG=1 timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_HEAVY_FRAC=0.012,0.013,0.01 > gpurun_out/ab_chk2.jsonl 2> gpurun_out/ab_chk2.log
echo done
