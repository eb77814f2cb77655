# CTA-histogram column CSR + light column sums from the entries; heavy threshold re-check
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_abi.py tests/test_parity_at_scale.py tests/test_dropin.py -x -q > gpurun_out/r3_pytest_b3.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_b3.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches_b3.csv python tools/one_step.py c3 1 > gpurun_out/r3_ncu_b3.log 2>&1; echo "ncu rc=$?"
timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 2 --env SF_HEAVY_FRAC=,0.035,0.045,0.05 > gpurun_out/r3_heavyfrac_b3.jsonl 2> gpurun_out/r3_heavyfrac_b3.log; echo "ab rc=$?"; cat gpurun_out/r3_heavyfrac_b3.jsonl
SF_DEBUG=1 timeout 600 python tools/e2e_probe.py --config c3 --reps 3 > gpurun_out/r3_e2e_b3.log 2>&1; echo "probe rc=$?"
grep -E "^rep|plan_create" gpurun_out/r3_e2e_b3.log | tail -6
