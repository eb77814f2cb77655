#!/usr/bin/env bash
# GPU round-trip: entry-list light scatter (parity + A/B at C3).
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "split or isect_is_exact or medium_scale" > gpurun_out/pytest_entry.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_entry.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 2 --env SF_LIGHT_ENTRY=0,1 > gpurun_out/ab_entry.jsonl 2> gpurun_out/ab_entry.log
timeout 900 env SF_LIGHT_ENTRY=1 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_LIGHT_BAND_MB=16,32,64 > gpurun_out/ab_entry_band.jsonl 2> gpurun_out/ab_entry_band.log
echo done
