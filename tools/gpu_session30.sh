#!/usr/bin/env bash
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi30.txt
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/bench_c3b.json 2> gpurun_out/bench_c3b.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 > gpurun_out/ab_chk.jsonl 2> gpurun_out/ab_chk.log
echo done
