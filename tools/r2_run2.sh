mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or split or exact or golden_stripes or oracle" > gpurun_out/r2_pytest2.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest2.log
BENCH_ALLOW_SHORT=1 timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/r2_bench_c3_gram.json 2> gpurun_out/r2_bench_c3_gram.log; echo "bench rc=$?"
tail -4 gpurun_out/r2_bench_c3_gram.log
