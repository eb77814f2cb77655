mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_wsplit.py tests/test_mantel.py -x -q -k "generalized or weighted or wsplit or golden or mantel" > gpurun_out/r2_pytest37.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest37.log
timeout 1500 python tools/wsplit_ab.py --config c4 --fracs 0.6,0.8 --reps 1 --no-uwalk > gpurun_out/r2_c4_ab3.jsonl 2> gpurun_out/r2_c4_ab3.log; cat gpurun_out/r2_c4_ab3.jsonl
timeout 1500 python bench.py --config c4 --no-cpu-baseline --no-dm --e2e-steps 2 > gpurun_out/r2_bench37_c4.json 2> gpurun_out/r2_bench37_c4.log; echo "bench c4 rc=$?"
timeout 1500 python bench.py --config c4f32 --no-cpu-baseline --no-dm --e2e-steps 2 > gpurun_out/r2_bench37_c4f32.json 2> gpurun_out/r2_bench37_c4f32.log; echo "bench c4f32 rc=$?"
timeout 900 python tools/mantel_bench.py --config c4 > gpurun_out/r2_mantel37_c4.json 2> gpurun_out/r2_mantel37_c4.log; echo "mantel rc=$?"; cat gpurun_out/r2_mantel37_c4.json
for f in c4 c4f32; do python -c "import json; d=json.load(open('gpurun_out/r2_bench37_$f.json')); print('$f', d.get('ms_per_step'), (d.get('e2e') or {}).get('seconds_per_dm'), (d.get('roofline') or {}).get('frac'))"; done
