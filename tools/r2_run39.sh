mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_parity_at_scale.py tests/test_wsplit.py tests/test_mantel.py tests/test_dropin.py -x -q > gpurun_out/r2_pytest39.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_pytest39.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c2_k13_v3.csv python tools/one_step.py c2 1 > gpurun_out/r2_ncu39.log 2>&1; echo "ncu rc=$?"
