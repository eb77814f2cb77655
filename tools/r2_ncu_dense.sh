mkdir -p gpurun_out
timeout 300 python tools/one_step.py c2 1 0 13 > gpurun_out/r2_os28.log 2>&1; echo "one_step rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wx_dense_kernel -c 1 -o gpurun_out/r2_wx_dense_c2 python tools/one_step.py c2 1 0 13 > gpurun_out/r2_ncu_dense.log 2>&1; echo "ncu rc=$?"
