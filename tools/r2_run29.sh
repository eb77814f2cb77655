# vectorised gram epilogue + measurement pass: tests, C3 step, bench lines, smoke
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split or gram or golden or light" > gpurun_out/r2_pytest29.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest29.log
timeout 600 python tools/one_step.py c3 3 > gpurun_out/r2_os29.log 2>&1; echo "c3 step: $(tail -1 gpurun_out/r2_os29.log)"
timeout 1200 python bench.py > gpurun_out/r2_bench29_c3.json 2> gpurun_out/r2_bench29_c3.log; echo "bench c3 rc=$?"
timeout 900 python bench.py --config c3f32 --no-cpu-baseline > gpurun_out/r2_bench29_c3f32.json 2> gpurun_out/r2_bench29_c3f32.log; echo "bench c3f32 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench29_ref.json 2> gpurun_out/r2_bench29_ref.log; echo "ref rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke29.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke29.log
for f in c3 c3f32 ref; do python -c "import json; d=json.load(open('gpurun_out/r2_bench29_$f.json')); print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('seconds_per_dm'), (d.get('roofline') or {}).get('frac'), (d.get('roofline') or {}).get('traffic'))"; done
