mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "light or heavy_light or gemm or pageable or exact_for_any" > gpurun_out/r2_pytest14.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2_pytest14.log
timeout 1500 python tools/heavy_frac_sweep.py c3 0.03 0.04 0.05 > gpurun_out/r2_heavyfrac_c3_col4.jsonl 2> gpurun_out/r2_heavyfrac_c3_col4.log
echo "sweep rc=$?"; cat gpurun_out/r2_heavyfrac_c3_col4.jsonl
SF_DEBUG=1 timeout 900 python tools/e2e_probe.py --reps 2 > gpurun_out/r2_e2e_probe14.log 2>&1; echo "probe rc=$?"
grep -E "^rep" gpurun_out/r2_e2e_probe14.log
