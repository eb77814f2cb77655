mkdir -p gpurun_out
SF_HEAVY_FRAC=0.04 timeout 1500 python tools/split_ab.py --config c3 --stripes 12500 paper_2005_05826_b200/libstripefrac_cuda.so tools/ab/lib_lw12800u8.so tools/ab/lib_lw6400u4.so tools/ab/lib_lw6400u8.so tools/ab/lib_lw4224u4n512.so > gpurun_out/r2_ab_light.jsonl 2> gpurun_out/r2_ab_light.log
echo rc=$?; cat gpurun_out/r2_ab_light.jsonl
