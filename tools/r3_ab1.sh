# light column kernel: carry-form adds + vector member loads vs the limb modes (C3 full range)
mkdir -p gpurun_out
timeout 900 python tools/split_ab.py --config c3 --stripes 12500 tools/ab/lib_lcarry0.so paper_2005_05826_b200/libstripefrac_cuda.so tools/ab/lib_lv8u1.so tools/ab/lib_lv8u4.so tools/ab/lib_lv16u1.so tools/ab/lib_lv16u2.so > gpurun_out/r3_ab1.jsonl 2> gpurun_out/r3_ab1.log
echo rc=$?
cat gpurun_out/r3_ab1.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "light or golden or exact or mem16" > gpurun_out/r3_pytest_light.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_light.log
