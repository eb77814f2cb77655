mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "exact_for_any or gemm or heavy_light or split_is_exact" > gpurun_out/r2_pytest10.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest10.log
python tools/one_step.py c3 2 > gpurun_out/r2_onestep10.log 2>&1 && cat gpurun_out/r2_onestep10.log && \
ncu --set full --import-source on --clock-control none -k regex:"light_column|cutlass|gram_digits|gram_epilogue" -c 4 -o gpurun_out/r2_c3_main python tools/one_step.py c3 1 > gpurun_out/r2_ncu10.log 2>&1
echo "ncu rc=$?"
