#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 900 python tools/e2e_probe.py --reps 2 > gpurun_out/e2e_probe.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log
echo done
