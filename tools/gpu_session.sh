#!/usr/bin/env bash
# Round-end style GPU pass: smoke, full parity suite, default bench line,
# reference arm, weighted lines.
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log
timeout 600 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log
export BENCH_ALLOW_SHORT=1
timeout 900 python bench.py --config c3wn --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3wn.json 2> gpurun_out/bench_c3wn.log
echo done
