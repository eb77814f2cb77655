set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -x -q -m gpu -k "split or exact or golden_stripes" > gpurun_out/r1_pytest_split.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r1_pytest_split.log
BENCH_ALLOW_SHORT=1 timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/r1_bench_c3.json 2> gpurun_out/r1_bench_c3.log; echo "bench rc=$?"
tail -3 gpurun_out/r1_bench_c3.log
