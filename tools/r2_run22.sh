mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wsplit.py -x -q > gpurun_out/r2_pytest22_wsplit.log 2>&1; echo "wsplit tests rc=$?"; tail -3 gpurun_out/r2_pytest22_wsplit.log
timeout 900 python tools/wsplit_ab.py --config c2 --fracs 0.1,0.2,0.3 > gpurun_out/r2_wsplit_ab3_c2.jsonl 2> gpurun_out/r2_wsplit_ab3_c2.log; echo "ab c2 rc=$?"
cat gpurun_out/r2_wsplit_ab3_c2.jsonl
timeout 1500 python tools/wsplit_ab.py --config c3wn --fracs 0.1,0.2,0.3 --reps 1 --no-uwalk > gpurun_out/r2_wsplit_ab3_c3wn.jsonl 2> gpurun_out/r2_wsplit_ab3_c3wn.log; echo "ab c3wn rc=$?"
cat gpurun_out/r2_wsplit_ab3_c3wn.jsonl
