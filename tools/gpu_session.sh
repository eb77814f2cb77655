#!/usr/bin/env bash
# GPU round-trip: full parity suite with pooled device memory, e2e phases, C3 bench.
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
SF_DEBUG=1 timeout 900 python tools/e2e_probe.py --config c3 --reps 4 > gpurun_out/e2e_c3.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.log
timeout 600 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log
echo done
