# e2e: plan creation with the schedule on a host thread; column strips per pass
mkdir -p gpurun_out
SF_DEBUG=1 timeout 600 python tools/e2e_probe.py --config c3 --reps 3 > gpurun_out/r3_e2e_default.log 2>&1; echo "probe rc=$?"
grep -E "^rep|plan_create|plan " gpurun_out/r3_e2e_default.log | tail -16
for g in 12 16 25; do SF_COPY_GROUPS=$g timeout 600 python tools/e2e_probe.py --config c3 --reps 3 > gpurun_out/r3_e2e_groups$g.log 2>&1; echo "groups $g rc=$?"; grep "^rep" gpurun_out/r3_e2e_groups$g.log; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_abi.py tests/test_dropin.py -x -q > gpurun_out/r3_pytest_e2e1.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_e2e1.log
