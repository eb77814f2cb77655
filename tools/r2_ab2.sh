mkdir -p gpurun_out
timeout 1500 python tools/split_ab.py --config c3 --stripes 2048 paper_2005_05826_b200/libstripefrac_cuda.so tools/ab/lib_v16u1f16m1.so tools/ab/lib_v16u1f8m1.so tools/ab/lib_v24u1f8m1.so tools/ab/lib_v32u1f8m1.so tools/ab/lib_v16u1f4n4m4.so > gpurun_out/r2_ab2.jsonl 2> gpurun_out/r2_ab2.log
echo rc=$?
cat gpurun_out/r2_ab2.jsonl
