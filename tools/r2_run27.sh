# 16-bit light members: tests + C3 A/B; light column params (fixed A/B builds)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "light or split or gram or golden" > gpurun_out/r2_pytest27.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest27.log
timeout 600 python tools/one_step.py c3 3 > gpurun_out/r2_os27a.log 2>&1; echo "16-bit: $(tail -1 gpurun_out/r2_os27a.log)"
SF_LIGHT_MEM16=0 timeout 600 python tools/one_step.py c3 3 > gpurun_out/r2_os27b.log 2>&1; echo "32-bit: $(tail -1 gpurun_out/r2_os27b.log)"
for v in lw12800u8 lw6400u4 lw6400u8 lw4224u4n512; do
  SF_LIB=tools/ab/lib_$v.so timeout 600 python tools/one_step.py c3 3 > gpurun_out/r2_os27_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/r2_os27_$v.log)"
done
