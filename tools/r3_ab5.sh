# light column kernel: chunked three-limb mode (3 shared atomics per pair instead of 4) at threshold 0.055; threshold re-sweep with it
mkdir -p gpurun_out
L=paper_2005_05826_b200/libstripefrac_cuda.so
timeout 900 python tools/split_ab.py --config c3 --stripes 12500 $L tools/ab/lib_lchunk.so $L tools/ab/lib_lchunk.so > gpurun_out/r3_ab5.jsonl 2> gpurun_out/r3_ab5.log
echo rc=$?
cat gpurun_out/r3_ab5.jsonl
SF_LIB=tools/ab/lib_lchunk.so timeout 900 python tools/kernel_ab.py --config c3 --kernels 10 --reps 2 --env SF_HEAVY_FRAC=0.055,0.065,0.075 > gpurun_out/r3_heavyfrac_b6.jsonl 2> gpurun_out/r3_heavyfrac_b6.log; echo "ab rc=$?"; cat gpurun_out/r3_heavyfrac_b6.jsonl
