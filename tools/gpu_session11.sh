#!/usr/bin/env bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "isect" > gpurun_out/pytest_isect2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_isect2.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 5,6 --reps 2 > gpurun_out/ab_c3_3.jsonl 2> gpurun_out/ab_c3_3.log
export BENCH_ALLOW_SHORT=1
CMD="python bench.py --config c3 --stripes 256 --kernel isect2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_isect2.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stripe_isect2 -s 1 -c 1 -o gpurun_out/prof_isect2b $CMD > gpurun_out/ncu_isect2.log 2>&1
echo done
