#!/usr/bin/env bash
# GPU round-trip: plan-creation phase timing; C5 shard at the size-aware threshold.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
SF_DEBUG=1 timeout 900 python tools/e2e_probe.py --config c3 --reps 3 > gpurun_out/e2e_c3.log 2>&1
timeout 1500 python bench.py --config c5 --stripes 7108 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_shard.json 2> gpurun_out/bench_c5_shard.log
echo done
