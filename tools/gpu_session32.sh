#!/usr/bin/env bash
# A/B the committed sources (tools/_ab_head) against the working tree in one session
mkdir -p gpurun_out
timeout 600 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 > gpurun_out/ab_cur.jsonl 2> gpurun_out/ab_cur.log
cp paper_2005_05826_b200/libstripefrac_cuda.so /tmp/cur.so
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-O3 -shared -Iinclude -Itools/_ab_head tools/_ab_head/sf_api.cu tools/_ab_head/host_prep.cpp -o paper_2005_05826_b200/libstripefrac_cuda.so > gpurun_out/build_head.log 2>&1
timeout 600 python tools/kernel_ab.py --config c3 --kernels 10 --reps 1 > gpurun_out/ab_head.jsonl 2> gpurun_out/ab_head.log
echo done
