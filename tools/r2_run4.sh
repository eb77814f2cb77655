mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "light or gemm or split or golden_stripes or pageable" > gpurun_out/r2_pytest4.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest4.log
timeout 1500 python tools/heavy_frac_sweep.py c3 0.02 0.03 0.04 0.05 0.07 > gpurun_out/r2_heavyfrac_c3_col.jsonl 2> gpurun_out/r2_heavyfrac_c3_col.log
echo "sweep rc=$?"; cat gpurun_out/r2_heavyfrac_c3_col.jsonl
SF_DEBUG=1 timeout 900 python tools/e2e_probe.py --reps 2 > gpurun_out/r2_e2e_probe.log 2>&1; echo "probe rc=$?"
grep -E "^rep|compute_stripes|plan_create" gpurun_out/r2_e2e_probe.log | tail -12
