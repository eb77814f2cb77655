# ncu --set full of the split path's prep kernels (one launch each) at C3
mkdir -p gpurun_out
timeout 300 python tools/one_step.py c3 1 > gpurun_out/r3_os_c3.log 2>&1; echo "one_step rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:sp_light_members_kernel|sp_col_fill_kernel|sp_col_count_kernel|sp_heavy_colsum_kernel|sp_gram_bits_kernel|sp_deep_scatter_kernel" -c 6 -o gpurun_out/r3_prep_c3 python tools/one_step.py c3 1 > gpurun_out/r3_ncu_prep.log 2>&1; echo "ncu rc=$?"
SF_DEBUG=1 timeout 600 python tools/e2e_probe.py --config c3 --reps 3 > gpurun_out/r3_e2e_sched.log 2>&1; echo "probe rc=$?"
grep -E "^rep|plan_create|plan " gpurun_out/r3_e2e_sched.log | tail -14
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_abi.py tests/test_wsplit.py -x -q > gpurun_out/r3_pytest_sched.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_sched.log
