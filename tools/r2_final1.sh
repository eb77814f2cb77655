# final measurement pass (round 2)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/rf_pytest_gpu.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/rf_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/rf_smoke.log
timeout 1200 python bench.py > gpurun_out/rf_bench_c3.json 2> gpurun_out/rf_bench_c3.log; echo "bench c3 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/rf_bench_ref.json 2> gpurun_out/rf_bench_ref.log; echo "ref rc=$?"
timeout 900 python bench.py --config c2 > gpurun_out/rf_bench_c2.json 2> gpurun_out/rf_bench_c2.log; echo "c2 rc=$?"
timeout 1200 python bench.py --config c3wn --no-cpu-baseline --e2e-steps 3 > gpurun_out/rf_bench_c3wn.json 2> gpurun_out/rf_bench_c3wn.log; echo "c3wn rc=$?"
timeout 900 python bench.py --config c3f32 --no-cpu-baseline > gpurun_out/rf_bench_c3f32.json 2> gpurun_out/rf_bench_c3f32.log; echo "c3f32 rc=$?"
timeout 1200 python bench.py --steps 2 --warmup 1 > gpurun_out/rf_b_short.json 2> gpurun_out/rf_b_short.log; echo "short bench rc=$?"
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rf_launches_c3.csv python bench.py --steps 2 --warmup 1 > gpurun_out/rf_ncu.log 2>&1; echo "ncu rc=$?"
for f in c3 ref c2 c3wn c3f32; do python -c "import json; d=json.load(open('gpurun_out/rf_bench_$f.json')); print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('seconds_per_dm'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('reasons'))"; done
