#!/usr/bin/env bash
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --e2e-steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log
echo done
