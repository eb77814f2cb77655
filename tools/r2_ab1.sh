mkdir -p gpurun_out
timeout 1500 python tools/split_ab.py --config c3 --stripes 2048 paper_2005_05826_b200/libstripefrac_cuda.so tools/ab/lib_*.so > gpurun_out/r2_ab1.jsonl 2> gpurun_out/r2_ab1.log
echo rc=$?
cat gpurun_out/r2_ab1.jsonl
