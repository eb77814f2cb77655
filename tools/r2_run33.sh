mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wsplit.py tests/test_gpu_parity.py -x -q -k "wsplit or weighted or golden" > gpurun_out/r2_pytest33.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest33.log
timeout 600 python tools/wsplit_ab.py --config c2 --fracs 0.1,0.15,0.2,0.3 2>/dev/null
timeout 1500 python tools/wsplit_ab.py --config c3wn --fracs 0.1,0.15,0.2 --reps 2 --no-uwalk 2>/dev/null
