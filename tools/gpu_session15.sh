#!/usr/bin/env bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "isect or golden or split" > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 9,10 --reps 2 > gpurun_out/ab_c3_7.jsonl 2> gpurun_out/ab_c3_7.log
for f in 0.005 0.02; do SF_HEAVY_FRAC=$f timeout 600 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 >> gpurun_out/ab_c3_7_frac.jsonl 2>> gpurun_out/ab_c3_7.log; done
export BENCH_ALLOW_SHORT=1
CMD="python bench.py --config c3 --stripes 512 --kernel split --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_split.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"stripe_split|sp_light" -s 2 -c 2 -o gpurun_out/prof_split $CMD > gpurun_out/ncu_split.log 2>&1
echo done
