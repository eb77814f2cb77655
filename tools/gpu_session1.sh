#!/usr/bin/env bash
# first GPU session: box facts, GPU tests, smoke, FP peaks, quick benches
set -x
mkdir -p gpurun_out
{ nvidia-smi; nproc; free -g; lscpu | head -20; } > gpurun_out/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python - > gpurun_out/peaks.log 2>&1 <<'PY'
import ctypes as C
lib = C.CDLL("tools/libsf_peaks.so")
for nm in ("sfp_dfma_per_s", "sfp_ffma_per_s"):
    f = getattr(lib, nm); f.restype = C.c_double; f.argtypes = [C.c_int, C.c_int]
    v = [f(0, 4000) for _ in range(3)]
    print(nm, [f"{x/1e12:.3f}e12 FMA/s" for x in v])
PY
timeout 600 python bench.py --config small --steps 3 --no-cpu-baseline > gpurun_out/bench_small.json 2> gpurun_out/bench_small.log
timeout 900 python bench.py --config c3 --steps 1 --stripes 512 --no-cpu-baseline > gpurun_out/bench_c3_512.json 2> gpurun_out/bench_c3_512.log
echo done
