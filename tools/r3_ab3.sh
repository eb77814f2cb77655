# light column kernel: dynamic entries / chunked three-limb mode / register cap (C3 full range)
mkdir -p gpurun_out
L=paper_2005_05826_b200/libstripefrac_cuda.so
timeout 900 python tools/split_ab.py --config c3 --stripes 12500 tools/ab/lib_ls0c0m2.so $L tools/ab/lib_ls0c0.so tools/ab/lib_ls1c0.so tools/ab/lib_ls0c1.so tools/ab/lib_ls1c1m2.so tools/ab/lib_ls0c0m2.so > gpurun_out/r3_ab3.jsonl 2> gpurun_out/r3_ab3.log
echo rc=$?
cat gpurun_out/r3_ab3.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "light or golden or exact or mem16 or carry" > gpurun_out/r3_pytest_ab3.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_ab3.log
