mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "light or heavy_light or gemm" > gpurun_out/r2_pytest11.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2_pytest11.log
timeout 1500 python tools/heavy_frac_sweep.py c3 0.03 0.04 0.05 0.06 > gpurun_out/r2_heavyfrac_c3_col3.jsonl 2> gpurun_out/r2_heavyfrac_c3_col3.log
echo "sweep rc=$?"; cat gpurun_out/r2_heavyfrac_c3_col3.jsonl
