#!/usr/bin/env bash
# ncu of the intersection kernel on a C3 stripe slice; launch list of one C3 step.
set -x
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
CMD="python bench.py --config c3 --stripes 256 --kernel isect --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_isect.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stripe_isect -s 1 -c 1 -o gpurun_out/prof_isect_c3s256 $CMD > gpurun_out/ncu_isect.log 2>&1
CMD2="python bench.py --config c3 --kernel isect --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_isect.csv $CMD2 > gpurun_out/ncu_launch.log 2>&1
echo done
