# gram epilogue: Horner over consecutive planes, hoisted second-level total
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_parity_at_scale.py -x -q > gpurun_out/r3_pytest_b4.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_b4.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches_b4.csv python tools/one_step.py c3 1 > gpurun_out/r3_ncu_b4.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sp_gram_epilogue_kernel -c 1 -o gpurun_out/r3_epi_c3 python tools/one_step.py c3 1 > gpurun_out/r3_ncu_epi.log 2>&1; echo "ncu epi rc=$?"
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 2 --env SF_HEAVY_FRAC=,0.05,0.055,0.06 > gpurun_out/r3_heavyfrac_b4.jsonl 2> gpurun_out/r3_heavyfrac_b4.log; echo "ab rc=$?"; cat gpurun_out/r3_heavyfrac_b4.jsonl
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r3_bench_b4.json 2> gpurun_out/r3_bench_b4.log; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r3_bench_b4.json')); print(d['ms_per_step'], d['e2e']['seconds_per_dm'], d['roofline']['frac'], d['clocks'])"
