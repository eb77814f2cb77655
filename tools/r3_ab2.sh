# light column walk variants + tiled gram epilogue (C3 full range)
mkdir -p gpurun_out
L=paper_2005_05826_b200/libstripefrac_cuda.so
timeout 900 python tools/split_ab.py --config c3 --stripes 12500 tools/ab/lib_lold.so $L tools/ab/lib_lv2u2.so tools/ab/lib_lv2u4.so tools/ab/lib_lv4u1.so tools/ab/lib_lcarryu4.so tools/ab/lib_lcarryu8.so > gpurun_out/r3_ab2.jsonl 2> gpurun_out/r3_ab2.log
echo rc=$?
SF_GRAM_TILED=0 timeout 600 python tools/split_ab.py --config c3 --stripes 12500 tools/ab/lib_lold.so $L > gpurun_out/r3_ab2_untiled.jsonl 2>> gpurun_out/r3_ab2.log
cat gpurun_out/r3_ab2.jsonl gpurun_out/r3_ab2_untiled.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_parity_at_scale.py -x -q > gpurun_out/r3_pytest_ab2.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3_pytest_ab2.log
