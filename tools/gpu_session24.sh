#!/usr/bin/env bash
mkdir -p gpurun_out
for nw in 4 8 16; do SF_SPLIT_NW=$nw timeout 600 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 >> gpurun_out/ab_nw.jsonl 2>> gpurun_out/ab_nw.log; done
echo done
