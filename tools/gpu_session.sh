#!/usr/bin/env bash
# GPU round-trip: heavy-row order A/B at threshold 0.03; ncu of the u-walk (word lists) at C2.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_HEAVY_BY_WEIGHT=,1 > gpurun_out/ab_order.jsonl 2> gpurun_out/ab_order.log
CMD="python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stripe_wuwalk" -s 1 -c 1 -o gpurun_out/prof_wuwalk_c2 $CMD > gpurun_out/ncu_wuwalk.log 2>&1
echo done
