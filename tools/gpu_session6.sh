#!/usr/bin/env bash
# Round-1 re-entry: full GPU suite, default bench, launch list, ncu of K2 sparse.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1; nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt; free -g >> gpurun_out/nproc.txt
ls -la paper_2005_05826_b200/*.so oracle/_ref tools/*.so > gpurun_out/files.txt 2>&1
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log
export BENCH_ALLOW_SHORT=1
CMD="python bench.py --config small --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_small.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_small.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stripe_sparse -s 1 -c 1 -o gpurun_out/prof_sparse_r1 $CMD > gpurun_out/ncu_sparse.log 2>&1
echo done
