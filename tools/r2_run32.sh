mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python tools/one_step.py c3 3 > gpurun_out/r2_os32a.log 2>&1; echo "default: $(tail -1 gpurun_out/r2_os32a.log)"
SF_LIGHT_PERSIST=1 timeout 600 python tools/one_step.py c3 3 > gpurun_out/r2_os32b.log 2>&1; echo "persist: $(tail -1 gpurun_out/r2_os32b.log)"
done
SF_LIGHT_PERSIST=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "light_column or split_is_exact" > gpurun_out/r2_pytest32.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2_pytest32.log
