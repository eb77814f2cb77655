#!/usr/bin/env bash
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/kernel_ab.py --config small --kernels 2,3,4 --reps 3 > gpurun_out/ab_small.jsonl 2> gpurun_out/ab_small.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 2,3,4 --reps 1 > gpurun_out/ab_c3.jsonl 2> gpurun_out/ab_c3.log
CMD="python bench.py --config small --kernel flat32 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
BENCH_ALLOW_SHORT=1 $CMD > gpurun_out/plain_f.log 2>&1 && \
  BENCH_ALLOW_SHORT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stripe_sparse_flat -s 1 -c 1 -o gpurun_out/prof_flat32 $CMD > gpurun_out/ncu_flat.log 2>&1
echo done
