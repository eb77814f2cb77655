mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wsplit.py -x -q > gpurun_out/r2_pytest24_wsplit.log 2>&1; echo "wsplit tests rc=$?"; tail -2 gpurun_out/r2_pytest24_wsplit.log
for lib in "" tools/ab/lib_wsr16.so tools/ab/lib_wsu2.so tools/ab/lib_wsu8.so; do
  echo "lib=$lib"
  SF_LIB=$lib timeout 600 python tools/wsplit_ab.py --config c2 --fracs 0.2 --no-uwalk 2>/dev/null
done
timeout 1500 python tools/wsplit_ab.py --config c3wn --fracs 0.15,0.2,0.25 --reps 1 --no-uwalk > gpurun_out/r2_wsplit_ab4_c3wn.jsonl 2> gpurun_out/r2_wsplit_ab4_c3wn.log; echo "ab c3wn rc=$?"
cat gpurun_out/r2_wsplit_ab4_c3wn.jsonl
