# light column kernel: member loads in flight per lane (2 / 4 default / 6 / 8) with the three-limb mode, threshold 0.065
mkdir -p gpurun_out
L=paper_2005_05826_b200/libstripefrac_cuda.so
timeout 900 python tools/split_ab.py --config c3 --stripes 12500 $L tools/ab/lib_lu2.so tools/ab/lib_lu6.so tools/ab/lib_lu8.so $L > gpurun_out/r3_ab9.jsonl 2> gpurun_out/r3_ab9.log
echo rc=$?
cat gpurun_out/r3_ab9.jsonl
