mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split or gram or light" > gpurun_out/r2_pytest30.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest30.log
for i in 1 2; do
timeout 600 python tools/one_step.py c3 3 > gpurun_out/r2_os30a.log 2>&1; echo "stream: $(tail -1 gpurun_out/r2_os30a.log)"
SF_LIB=tools/ab/lib_lnostream.so timeout 600 python tools/one_step.py c3 3 > gpurun_out/r2_os30b.log 2>&1; echo "plain: $(tail -1 gpurun_out/r2_os30b.log)"
done
