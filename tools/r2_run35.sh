mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wsplit.py -x -q > gpurun_out/r2_pytest35.log 2>&1; echo "wsplit tests rc=$?"; tail -2 gpurun_out/r2_pytest35.log
timeout 900 python tools/e2e_probe.py --reps 3 > gpurun_out/r2_e2e35a.log 2>&1; echo "default:"; grep rep gpurun_out/r2_e2e35a.log
SF_LIB=tools/ab/lib_lnostream.so timeout 900 python tools/e2e_probe.py --reps 3 > gpurun_out/r2_e2e35b.log 2>&1; echo "nostream:"; grep rep gpurun_out/r2_e2e35b.log
timeout 1200 python tools/wsplit_ab.py --config c4 --fracs 0.1,0.25 --reps 1 > gpurun_out/r2_c4_ab.jsonl 2> gpurun_out/r2_c4_ab.log; echo "c4 rc=$?"; cat gpurun_out/r2_c4_ab.jsonl
