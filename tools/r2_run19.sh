# kernel 13 launch lists (C2, C3-WN), tiled gram epilogue check
mkdir -p gpurun_out
export SF_WHEAVY_FRAC=0.2
timeout 300 python tools/one_step.py c2 1 0 13 > gpurun_out/r2_os_c2.log 2>&1; echo "one_step c2 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c2_k13.csv python tools/one_step.py c2 1 0 13 > gpurun_out/r2_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "split or gram or golden" > gpurun_out/r2_pytest19.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest19.log
timeout 600 python tools/one_step.py c3 2 > gpurun_out/r2_os_c3.log 2>&1; echo "one_step c3 rc=$?"; cat gpurun_out/r2_os_c3.log | tail -2
