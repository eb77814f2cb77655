#!/usr/bin/env python
"""One plan + N runs of a config (for ncu launch lists / captures).

  python tools/one_step.py CONFIG [RUNS] [STRIPES] [KERNEL]"""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2005_05826_b200 import _native as N  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
stripes = int(sys.argv[3]) if len(sys.argv) > 3 else 0
kernel = int(sys.argv[4]) if len(sys.argv) > 4 else 0
problem = bench.make_problem(cfg)
L = N.lib()
n = problem.n_samples
ex, _keep = N.make_exec([0], kernel)
plan = C.c_void_p()
N.check(L.sf_plan_create(problem.ref, bench.METRIC_CODE[cfg["metric"]], 8 if cfg["precision"] == "fp64" else 4, 0,
                         stripes or n // 2, C.byref(ex), C.byref(plan)))
st = N.sf_stats()
for _ in range(runs):
    N.check(L.sf_plan_run(plan, 1))
    N.check(L.sf_plan_sync(plan))
N.check(L.sf_plan_stats(plan, C.byref(st)))
print("total_ms", st.total_ms, "launches", st.launches, flush=True)
