mkdir -p gpurun_out
SF_DEBUG=1 timeout 900 python tools/e2e_probe.py --reps 3 > gpurun_out/r2_e2e36.log 2>&1; grep -E "^rep|light pass|pool" gpurun_out/r2_e2e36.log | head -30
timeout 1200 python tools/wsplit_ab.py --config c4 --fracs 0.25,0.4,0.6 --reps 1 > gpurun_out/r2_c4_ab2.jsonl 2> gpurun_out/r2_c4_ab2.log; echo "c4 rc=$?"; cat gpurun_out/r2_c4_ab2.jsonl
