# ncu --set full captures at the full C3 range: two heavy GEMM launches (roofline.traffic) and the light column kernel
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:cutlass -c 2 -o gpurun_out/r3_gemm_c3 python tools/one_step.py c3 1 > gpurun_out/r3_ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:sp_light_column_kernel -c 1 -o gpurun_out/r3_light_c3 python tools/one_step.py c3 1 > gpurun_out/r3_ncu_light.log 2>&1; echo "ncu light rc=$?"
