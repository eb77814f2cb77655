#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_SPLIT_VARIANT=5,7,8,9 > gpurun_out/ab_var3.jsonl 2> gpurun_out/ab_var.log
echo done
