#!/usr/bin/env bash
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
CMD="python bench.py --config c3 --stripes 1024 --kernel split --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_split_r.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"stripe_split|sp_light" -s 2 -c 2 -o gpurun_out/prof_split_r $CMD > gpurun_out/ncu_split_r.log 2>&1
echo done
