#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 600 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 >> gpurun_out/ab_v2.jsonl 2>> gpurun_out/ab_v2.log
echo done
