mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wsplit.py -x -q > gpurun_out/r2_pytest31.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest31.log
timeout 600 python tools/wsplit_ab.py --config c2 --fracs 0.2 --no-uwalk 2>/dev/null
timeout 1200 python tools/wsplit_ab.py --config c3wn --fracs 0.2 --reps 2 --no-uwalk 2>/dev/null
