mkdir -p gpurun_out
export SF_WHEAVY_FRAC=0.2
timeout 300 python tools/one_step.py c2 1 0 13 > gpurun_out/r2_os_c2b.log 2>&1; echo "one_step rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wx_light_kernel -c 1 -o gpurun_out/r2_wx_light_c2_v3 python tools/one_step.py c2 1 0 13 > gpurun_out/r2_ncu_light.log 2>&1; echo "ncu rc=$?"
