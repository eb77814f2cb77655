# full GPU suite with the weighted split default; C2 / C3-WN bench lines; GEMM traffic capture
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest25_all.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/r2_pytest25_all.log
timeout 900 python bench.py --config c2 > gpurun_out/r2_bench25_c2.json 2> gpurun_out/r2_bench25_c2.log; echo "bench c2 rc=$?"
timeout 1200 python bench.py --config c3wn --no-cpu-baseline --e2e-steps 3 > gpurun_out/r2_bench25_c3wn.json 2> gpurun_out/r2_bench25_c3wn.log; echo "bench c3wn rc=$?"
timeout 600 python tools/one_step.py c3 1 > gpurun_out/r2_os25.log 2>&1; echo "one_step rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:cutlass -c 3 -o gpurun_out/r2_gemm_c3 python tools/one_step.py c3 1 > gpurun_out/r2_ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
for f in c2 c3wn; do python -c "import json; d=json.load(open('gpurun_out/r2_bench25_$f.json')); print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('seconds_per_dm'), (d.get('roofline') or {}).get('frac'))"; done
