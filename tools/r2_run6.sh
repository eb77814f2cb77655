mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "light or gemm or heavy_light or pageable or shards or golden_stripes" > gpurun_out/r2_pytest6.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest6.log
timeout 1200 python bench.py > gpurun_out/r2_bench6_c3.json 2> gpurun_out/r2_bench6_c3.log; echo "bench rc=$?"
tail -5 gpurun_out/r2_bench6_c3.log
SF_DEBUG=1 timeout 900 python tools/e2e_probe.py --reps 2 > gpurun_out/r2_e2e_probe6.log 2>&1; echo "probe rc=$?"
grep -E "^rep|plan   |compute_stripes" gpurun_out/r2_e2e_probe6.log | tail -24
