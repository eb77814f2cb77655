# validation of the defaults: three-limb chunked light kernel, threshold 0.065
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3_smoke6.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r3_smoke6.log
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r3_pytest_gpu6.log 2>&1; echo "gpu suite rc=$?"; tail -2 gpurun_out/r3_pytest_gpu6.log
timeout 900 python bench.py > gpurun_out/r3_bench6.json 2> gpurun_out/r3_bench6.log; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r3_bench6.json')); print(d['ms_per_step'], d['e2e']['seconds_per_dm'], d['roofline']['frac'], d['roofline']['traffic'], d['clocks'], d['cpu_baseline']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r3_launches_bench6.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3_ncu6.log 2>&1; echo "ncu rc=$?"
