mkdir -p gpurun_out
SF_DEBUG=1 timeout 900 python tools/e2e_probe.py --reps 3 > gpurun_out/r2_e2e_probe7.log 2>&1; echo "probe rc=$?"
grep -E "^rep|pool|device setup|compute_stripes" gpurun_out/r2_e2e_probe7.log | tail -40
