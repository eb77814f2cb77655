#!/usr/bin/env bash
# GPU round-trip: light-scatter cost split (dry run), u-walk slot variants.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_LIGHT_DRYRUN=0,1 > gpurun_out/ab_dry.jsonl 2> gpurun_out/ab_dry.log
timeout 900 env SF_LIGHT_BAND_MB=128 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 --env SF_LIGHT_DRYRUN=0,1 > gpurun_out/ab_dry128.jsonl 2> gpurun_out/ab_dry128.log
timeout 600 python tools/kernel_ab.py --config c2 --kernels 12 --reps 2 --env SF_UWALK_VARIANT=0,1,2 > gpurun_out/ab_uwvar.jsonl 2> gpurun_out/ab_uwvar.log
echo done
