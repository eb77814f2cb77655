# deep scatter warp-per-entry, sliced heavy column sums, earlier table upload
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_abi.py tests/test_parity_at_scale.py tests/test_dropin.py -x -q > gpurun_out/r3_pytest_b2.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_b2.log
SF_DEBUG=1 timeout 600 python tools/e2e_probe.py --config c3 --reps 3 > gpurun_out/r3_e2e_b2.log 2>&1; echo "probe rc=$?"
grep -E "^rep|plan_create|plan " gpurun_out/r3_e2e_b2.log | tail -14
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches_b2.csv python tools/one_step.py c3 1 > gpurun_out/r3_ncu_b2.log 2>&1; echo "ncu rc=$?"
