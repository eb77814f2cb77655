#!/usr/bin/env bash
# session 2: parity (dense + sparse), benches, ncu launch list + full capture of the sparse kernel
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
export BENCH_ALLOW_SHORT=1
timeout 300 python bench.py --config small --kernel dense --steps 3 --no-cpu-baseline > gpurun_out/b_small_dense.json 2> gpurun_out/b_small_dense.log
timeout 300 python bench.py --config small --kernel sparse --steps 3 --no-cpu-baseline > gpurun_out/b_small_sparse.json 2> gpurun_out/b_small_sparse.log
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.log
timeout 600 python bench.py --config c3 --kernel dense --stripes 512 --steps 1 --no-cpu-baseline --no-e2e > gpurun_out/b_c3_dense512.json 2> gpurun_out/b_c3_dense512.log
CMD="python bench.py --config small --kernel sparse --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_small.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_small.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain_small2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stripe_sparse -s 1 -c 1 -o gpurun_out/prof_sparse_small $CMD > gpurun_out/ncu_full.log 2>&1
echo done
