#!/usr/bin/env bash
# GPU round-trip: u64 light-sum atomics (parity + A/B).
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "split or isect_is_exact or oracle_random or golden_stripes or stripe_shards" > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 2 --env SF_LIGHT_DRYRUN=0,1 > gpurun_out/ab_u64.jsonl 2> gpurun_out/ab_u64.log
echo done
