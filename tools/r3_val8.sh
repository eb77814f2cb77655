# gram epilogue on a 2D grid (no 64-bit division per slot)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_parity_at_scale.py tests/test_abi.py -x -q > gpurun_out/r3_pytest_v8.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_v8.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches_v8.csv python tools/one_step.py c3 1 > gpurun_out/r3_ncu_v8.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r3_bench_v8.json 2> gpurun_out/r3_bench_v8.log; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r3_bench_v8.json')); print(d['ms_per_step'], d['e2e']['seconds_per_dm'], d['roofline']['frac'], d['clocks'])"
