mkdir -p gpurun_out
python tools/one_step.py c3 1 > gpurun_out/r2_onestep.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv python tools/one_step.py c3 1 > gpurun_out/r2_ncu_launches.log 2>&1
echo "rc=$?"
