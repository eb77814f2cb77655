#!/usr/bin/env bash
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
export BENCH_ALLOW_SHORT=1
timeout 300 python bench.py --config small --kernel sparse --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/b_small_sparse.json 2> gpurun_out/b_small_sparse.log
timeout 900 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_c3.json 2> gpurun_out/b_c3.log
CMD="python bench.py --config small --kernel sparse --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_s.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stripe_sparse -s 1 -c 1 -o gpurun_out/prof_sparse_v6 $CMD > gpurun_out/ncu_sparse.log 2>&1
echo done
