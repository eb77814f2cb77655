#!/usr/bin/env bash
# One GPU round-trip: parity tests, the default bench line, the reference arm,
# the launch list of a bench step and one ncu --set full capture of the
# dominant kernel (each ncu pass only after its command exited 0 without ncu).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.log; echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
BENCH_ALLOW_SHORT=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
BENCH_ALLOW_SHORT=1 timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"stripe_split|sp_light" -s 2 -c 2 -o gpurun_out/prof_split $CMD > gpurun_out/ncu_full.log 2>&1
echo done
