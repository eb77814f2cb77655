#!/usr/bin/env bash
set -x
mkdir -p gpurun_out
for f in 0.008 0.012 0.016 0.02; do SF_HEAVY_FRAC=$f timeout 600 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 >> gpurun_out/ab_frac16.jsonl 2>> gpurun_out/ab_frac16.log; done
export BENCH_ALLOW_SHORT=1
CMD="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_c3.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_split.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo done
