mkdir -p gpurun_out
(bash tools/reference_at_scale.sh > gpurun_out/refscale.txt 2>&1) &
RP=$!
timeout 1500 python tools/heavy_frac_sweep.py c3 0.03 0.02 0.015 0.01 0.0075 0.005 > gpurun_out/r2_heavyfrac_c3.jsonl 2> gpurun_out/r2_heavyfrac_c3.log
echo "sweep rc=$?"
cat gpurun_out/r2_heavyfrac_c3.jsonl
wait $RP
echo "ref rc=$?"
cat gpurun_out/refscale.txt
