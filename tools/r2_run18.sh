# kernel 13 correctness + A/B, kernel 10 lazy light sums regression, C5 session
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wsplit.py -x -q > gpurun_out/r2_pytest18_wsplit.log 2>&1; echo "wsplit tests rc=$?"; tail -3 gpurun_out/r2_pytest18_wsplit.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2_pytest18_parity.log 2>&1; echo "parity tests rc=$?"; tail -3 gpurun_out/r2_pytest18_parity.log
timeout 900 python tools/wsplit_ab.py --config c2 --fracs 0.05,0.1,0.2,0.3,0.5 > gpurun_out/r2_wsplit_ab_c2.jsonl 2> gpurun_out/r2_wsplit_ab_c2.log; echo "ab c2 rc=$?"
cat gpurun_out/r2_wsplit_ab_c2.jsonl
timeout 1200 python tools/wsplit_ab.py --config c3wn --fracs 0.1,0.2,0.3 --reps 1 > gpurun_out/r2_wsplit_ab_c3wn.jsonl 2> gpurun_out/r2_wsplit_ab_c3wn.log; echo "ab c3wn rc=$?"
cat gpurun_out/r2_wsplit_ab_c3wn.jsonl
SF_DEBUG=1 timeout 1800 python tools/c5_session.py > gpurun_out/r2_c5_session.jsonl 2> gpurun_out/r2_c5_session.log; echo "c5 rc=$?"
cat gpurun_out/r2_c5_session.jsonl
