# C5 parity + timing, C4 fp64-vs-fp32 Mantel, C3 launch list (current default)
mkdir -p gpurun_out
timeout 1500 python tools/c5_session.py > gpurun_out/r2_c5_session.jsonl 2> gpurun_out/r2_c5_session.log; echo "c5 rc=$?"
timeout 900 python tools/mantel_bench.py --config c4 > gpurun_out/r2_mantel_c4.json 2> gpurun_out/r2_mantel_c4.log; echo "mantel c4 rc=$?"
timeout 600 python tools/one_step.py c3 2 > gpurun_out/r2_one_step.log 2>&1; echo "one_step rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3_v3.csv python tools/one_step.py c3 2 > gpurun_out/r2_launches.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/r2_c5_session.jsonl gpurun_out/r2_mantel_c4.json
tail -3 gpurun_out/r2_c5_session.log gpurun_out/r2_mantel_c4.log
