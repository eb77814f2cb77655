#!/usr/bin/env bash
# GPU round-trip: full parity suite (no -x: every failure listed), heavy-row
# threshold re-sweep with the banded light scatter.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 2000 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_HEAVY_FRAC=0.012,0.016,0.02,0.025 > gpurun_out/ab_heavy.jsonl 2> gpurun_out/ab_heavy.log
echo done
