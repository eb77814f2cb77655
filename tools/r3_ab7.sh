# dynamic entry hand-out with the chunked light kernel; C3 fp32 and C2 WN bench lines
mkdir -p gpurun_out
L=paper_2005_05826_b200/libstripefrac_cuda.so
timeout 900 python tools/split_ab.py --config c3 --stripes 12500 $L tools/ab/lib_ldyn.so $L tools/ab/lib_ldyn.so > gpurun_out/r3_ab7.jsonl 2> gpurun_out/r3_ab7.log
echo rc=$?
cat gpurun_out/r3_ab7.jsonl
timeout 900 python bench.py --config c3f32 --no-cpu-baseline > gpurun_out/r3_bench7_c3f32.json 2> gpurun_out/r3_bench7_c3f32.log; echo "c3f32 rc=$?"
timeout 900 python bench.py --config c2 > gpurun_out/r3_bench7_c2.json 2> gpurun_out/r3_bench7_c2.log; echo "c2 rc=$?"
for f in c3f32 c2; do python -c "import json; d=json.load(open('gpurun_out/r3_bench7_$f.json')); print('$f', d.get('ms_per_step'), (d.get('e2e') or {}).get('seconds_per_dm'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('reasons'))"; done
