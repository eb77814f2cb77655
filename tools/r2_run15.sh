mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke.log
SF_PARITY_LOG=gpurun_out/r2_parity_at_scale.jsonl timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r2_pytest_gpu_full.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest_gpu_full.log
cat gpurun_out/r2_parity_at_scale.jsonl
