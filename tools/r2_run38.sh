mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_wsplit.py -x -q > gpurun_out/r2_pytest38.log 2>&1; echo "wsplit tests rc=$?"; tail -3 gpurun_out/r2_pytest38.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_parity_at_scale.py -x -q -k "weighted or generalized or golden or wn" > gpurun_out/r2_pytest38b.log 2>&1; echo "weighted tests rc=$?"; tail -2 gpurun_out/r2_pytest38b.log
timeout 600 python tools/wsplit_ab.py --config c2 --fracs 0.25 --no-uwalk 2>/dev/null
SF_WS_DENSE_EMBED=1 timeout 600 python tools/wsplit_ab.py --config c2 --fracs 0.25 --no-uwalk 2>/dev/null
timeout 1200 python tools/wsplit_ab.py --config c3wn --fracs 0.25 --reps 2 --no-uwalk 2>/dev/null
SF_WS_DENSE_EMBED=1 timeout 1200 python tools/wsplit_ab.py --config c3wn --fracs 0.25 --reps 2 --no-uwalk 2>/dev/null
