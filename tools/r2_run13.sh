mkdir -p gpurun_out
python tools/one_step.py c3 2 > gpurun_out/r2_onestep13.log 2>&1 && cat gpurun_out/r2_onestep13.log && \
ncu --set full --import-source on --clock-control none -k regex:"light_column|gram_epilogue" -c 2 -o gpurun_out/r2_c3_light python tools/one_step.py c3 1 > gpurun_out/r2_ncu13.log 2>&1
echo "ncu rc=$?"
python tools/one_step.py c3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3_v2.csv python tools/one_step.py c3 1 > gpurun_out/r2_ncu13b.log 2>&1
echo "launches rc=$?"
