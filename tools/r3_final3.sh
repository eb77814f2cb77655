# last pass at HEAD: smoke, GPU suite, default bench line
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf4_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/rf4_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/rf4_pytest_gpu.log 2>&1; echo "gpu suite rc=$?"; tail -2 gpurun_out/rf4_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/rf4_bench_c3.json 2> gpurun_out/rf4_bench_c3.log; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/rf4_bench_c3.json')); print(d['ms_per_step'], d['e2e']['seconds_per_dm'], d['roofline']['frac'], d['clocks'], d['cpu_baseline']['value'], d['gpu_launches'])"
