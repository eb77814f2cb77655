#!/usr/bin/env bash
# GPU round-trip: end-to-end phase breakdown (C3 fp64/fp32, C2).
mkdir -p gpurun_out
export SF_DEBUG=1
timeout 900 python tools/e2e_probe.py --config c3 --reps 4 > gpurun_out/e2e_c3.log 2>&1
timeout 900 python tools/e2e_probe.py --config c3f32 --reps 3 > gpurun_out/e2e_c3f32.log 2>&1
timeout 600 python tools/e2e_probe.py --config c2 --reps 4 > gpurun_out/e2e_c2.log 2>&1
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
echo done
