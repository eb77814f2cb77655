#!/usr/bin/env bash
# GPU round-trip: entry lists vs row scan at the C5 shard.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 1500 python tools/kernel_ab.py --config c5 --stripes 7108 --kernels 10 --reps 1 --env SF_LIGHT_ENTRY=0,1 > gpurun_out/ab_c5_entry.jsonl 2> gpurun_out/ab_c5_entry.log
echo done
