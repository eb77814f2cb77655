#!/usr/bin/env bash
# GPU round-trip: weighted sparse walk + generalized parity, C2/C4 benches,
# ncu of the split kernel (1024 stripes) and of the weighted walk at C2.
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "weighted_sparse or generalized or golden_stripes or oracle_random or chunked or partition" > gpurun_out/pytest_w.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_w.log
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log
timeout 600 python bench.py --config c2 --kernel dense --steps 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2_dense.json 2> gpurun_out/bench_c2_dense.log
timeout 900 python bench.py --config c3wn --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3wn.json 2> gpurun_out/bench_c3wn.log
timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log
CMD="python bench.py --config c3 --stripes 1024 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stripe_split" -s 1 -c 1 -o gpurun_out/prof_split1024 $CMD > gpurun_out/ncu_split.log 2>&1
CMD="python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stripe_wsparse" -s 1 -c 1 -o gpurun_out/prof_wsparse_c2 $CMD > gpurun_out/ncu_wsparse.log 2>&1
echo done
