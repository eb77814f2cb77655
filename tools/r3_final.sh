# final pass at HEAD: smoke, GPU suite, default bench line, reference arm, launch list, e2e phases
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf3_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/rf3_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/rf3_pytest_gpu.log 2>&1; echo "gpu suite rc=$?"; tail -2 gpurun_out/rf3_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/rf3_bench_c3.json 2> gpurun_out/rf3_bench_c3.log; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/rf3_bench_c3.json')); print(d['ms_per_step'], d['e2e']['seconds_per_dm'], d['roofline']['frac'], d['clocks'], d['cpu_baseline']['value'], d['gpu_launches'])"
timeout 900 python bench.py --impl reference > gpurun_out/rf3_bench_ref.json 2> gpurun_out/rf3_bench_ref.log; echo "ref rc=$?"; cat gpurun_out/rf3_bench_ref.json
SF_DEBUG=1 timeout 600 python tools/e2e_probe.py --config c3 --reps 3 > gpurun_out/rf3_e2e.log 2>&1; echo "probe rc=$?"; grep "^rep" gpurun_out/rf3_e2e.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/rf3_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/rf3_ncu.log 2>&1; echo "ncu rc=$?"
