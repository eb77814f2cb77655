# kernel 13 v2 (rank starts, one-tile light, conflict-free dense), wu_colsum v2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wsplit.py -x -q > gpurun_out/r2_pytest20_wsplit.log 2>&1; echo "wsplit tests rc=$?"; tail -3 gpurun_out/r2_pytest20_wsplit.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "weighted or uwalk or golden or generalized" > gpurun_out/r2_pytest20_w.log 2>&1; echo "weighted tests rc=$?"; tail -3 gpurun_out/r2_pytest20_w.log
timeout 900 python tools/wsplit_ab.py --config c2 --fracs 0.1,0.2,0.3,0.5 > gpurun_out/r2_wsplit_ab2_c2.jsonl 2> gpurun_out/r2_wsplit_ab2_c2.log; echo "ab c2 rc=$?"
cat gpurun_out/r2_wsplit_ab2_c2.jsonl
export SF_WHEAVY_FRAC=0.2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c2_k13_v2.csv python tools/one_step.py c2 1 0 13 > gpurun_out/r2_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
unset SF_WHEAVY_FRAC
timeout 1500 python tools/wsplit_ab.py --config c3wn --fracs 0.1,0.2,0.3,0.5 --reps 1 > gpurun_out/r2_wsplit_ab2_c3wn.jsonl 2> gpurun_out/r2_wsplit_ab2_c3wn.log; echo "ab c3wn rc=$?"
cat gpurun_out/r2_wsplit_ab2_c3wn.jsonl
