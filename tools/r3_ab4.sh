# light column kernel: prefetch of the next entry's members (none / L2 / L1), C3 full range
mkdir -p gpurun_out
L=paper_2005_05826_b200/libstripefrac_cuda.so
timeout 900 python tools/split_ab.py --config c3 --stripes 12500 tools/ab/lib_lpf0.so $L tools/ab/lib_lpf2.so tools/ab/lib_lpf0.so $L > gpurun_out/r3_ab4.jsonl 2> gpurun_out/r3_ab4.log
echo rc=$?
cat gpurun_out/r3_ab4.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "light or golden or exact or mem16" > gpurun_out/r3_pytest_ab4.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_ab4.log
