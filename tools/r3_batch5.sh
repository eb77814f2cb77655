# epilogue with constant limb shifts, heavy threshold 0.055, old column CSR + entry column sums
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_abi.py tests/test_parity_at_scale.py tests/test_dropin.py -x -q > gpurun_out/r3_pytest_b5.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_b5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches_b5.csv python tools/one_step.py c3 1 > gpurun_out/r3_ncu_b5.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sp_gram_epilogue_kernel -c 1 -o gpurun_out/r3_epi2_c3 python tools/one_step.py c3 1 > gpurun_out/r3_ncu_epi2.log 2>&1; echo "ncu epi rc=$?"
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 2 --env SF_GRAM_BK=,512,2048 > gpurun_out/r3_bk_b5.jsonl 2> gpurun_out/r3_bk_b5.log; echo "ab rc=$?"; cat gpurun_out/r3_bk_b5.jsonl
timeout 900 python bench.py > gpurun_out/r3_bench_b5.json 2> gpurun_out/r3_bench_b5.log; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r3_bench_b5.json')); print(d['ms_per_step'], d['e2e']['seconds_per_dm'], d['roofline']['frac'], d['clocks'], d['cpu_baseline']['value'])"
