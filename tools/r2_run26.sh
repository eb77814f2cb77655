# ncu of the UW light column kernel (C3) and the weighted light kernel (C2)
mkdir -p gpurun_out
SF_DEBUG=1 timeout 600 python tools/one_step.py c3 2 > gpurun_out/r2_os26.log 2>&1; echo "one_step rc=$?"; grep -E "schedule|validate|plan_create|compute_stripes" gpurun_out/r2_os26.log | tail -6
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:sp_light_column_kernel -c 1 -o gpurun_out/r2_light_col_c3 python tools/one_step.py c3 1 > gpurun_out/r2_ncu_lc.log 2>&1; echo "ncu rc=$?"
