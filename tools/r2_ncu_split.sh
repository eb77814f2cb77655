# ncu of the split kernel at C3, 1024 stripes (one launch)
mkdir -p gpurun_out
export BENCH_ALLOW_SHORT=1
CMD="python bench.py --stripes 1024 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/r2_ncu_plain.json 2> gpurun_out/r2_ncu_plain.log && \
ncu --set full --import-source on --clock-control none -k regex:stripe_split -s 3 -c 1 -o gpurun_out/r2_split_c3_1024 $CMD > gpurun_out/r2_ncu.log 2>&1
echo "ncu rc=$?"
