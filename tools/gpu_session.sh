#!/usr/bin/env bash
# GPU round-trip: split-kernel occupancy variants (parity + A/B), band size,
# C5 per-GPU shard threshold sweep.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "split_variants or banded or uwalk_word_list" > gpurun_out/pytest_var.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_var.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_SPLIT_VARIANT=0,8,9,10 > gpurun_out/ab_var2.jsonl 2> gpurun_out/ab_var2.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_LIGHT_BAND_MB=12,20,32 > gpurun_out/ab_band2.jsonl 2> gpurun_out/ab_band2.log
timeout 1500 python tools/kernel_ab.py --config c5 --stripes 7108 --kernels 10 --reps 1 --env SF_HEAVY_FRAC=0.01,0.02,0.03 > gpurun_out/ab_c5.jsonl 2> gpurun_out/ab_c5.log
echo done
