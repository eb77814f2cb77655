#!/usr/bin/env bash
# GPU round-trip: .strf writer parity, Mantel at C3 scale, C4 fp32 line.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_mantel.py -q -m gpu -k "strf or mantel" > gpurun_out/pytest_strf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_strf.log
timeout 1200 python tools/mantel_bench.py --config c3 --perms 999 > gpurun_out/mantel_c3.json 2> gpurun_out/mantel_c3.log
timeout 900 python bench.py --config c4f32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4f32.json 2> gpurun_out/bench_c4f32.log
echo done
