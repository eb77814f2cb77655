mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "default_for_unweighted or fit_probe or over_several" > gpurun_out/r2_pytest16.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest16.log
timeout 1200 python bench.py > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.log; echo "bench c3 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.log; echo "ref rc=$?"
timeout 900 python bench.py --config c2 > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.log; echo "c2 rc=$?"
timeout 900 python bench.py --config c3f32 --no-cpu-baseline > gpurun_out/r2_bench_c3f32.json 2> gpurun_out/r2_bench_c3f32.log; echo "c3f32 rc=$?"
timeout 1200 python bench.py --config c3wn --no-cpu-baseline --no-dm --e2e-steps 2 > gpurun_out/r2_bench_c3wn.json 2> gpurun_out/r2_bench_c3wn.log; echo "c3wn rc=$?"
for f in c3 ref c2 c3f32 c3wn; do python -c "import json,sys; d=json.load(open('gpurun_out/r2_bench_$f.json')); print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('seconds_per_dm'), (d.get('roofline') or {}).get('frac'))"; done
