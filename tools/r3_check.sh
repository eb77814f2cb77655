# session re-entry check: GPU suite, smoke, default bench line
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/c_topo.txt 2>&1; numactl -H >> gpurun_out/c_topo.txt 2>&1; lscpu >> gpurun_out/c_topo.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/c_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c_pytest_gpu.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/c_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/c_bench_c3.json 2> gpurun_out/c_bench_c3.log; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c_bench_c3.json')); print(d['ms_per_step'], d['e2e'], d['roofline']['frac'], d['clocks'])"
