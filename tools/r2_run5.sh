mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "light or gemm or heavy_light or pageable" > gpurun_out/r2_pytest5.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest5.log
timeout 1500 python tools/heavy_frac_sweep.py c3 0.02 0.025 0.03 0.04 > gpurun_out/r2_heavyfrac_c3_col2.jsonl 2> gpurun_out/r2_heavyfrac_c3_col2.log
echo "sweep column rc=$?"; cat gpurun_out/r2_heavyfrac_c3_col2.jsonl
SF_LIGHT_MODE=band timeout 1500 python tools/heavy_frac_sweep.py c3 0.02 0.025 > gpurun_out/r2_heavyfrac_c3_band.jsonl 2> gpurun_out/r2_heavyfrac_c3_band.log
echo "sweep band rc=$?"; cat gpurun_out/r2_heavyfrac_c3_band.jsonl
