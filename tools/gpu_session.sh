#!/usr/bin/env bash
# GPU round-trip: generalized + banded parity, C3/C2/C4 bench lines.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "generalized or banded or uwalk" > gpurun_out/pytest_gen.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gen.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.log
timeout 600 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log
timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log
timeout 900 python bench.py --config c3wn --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3wn.json 2> gpurun_out/bench_c3wn.log
echo done
