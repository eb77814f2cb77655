#!/usr/bin/env python
"""Break the end-to-end C-ABI call into its parts (plan create, run, download)
and time sf_compute_stripes itself, with pinned and pageable host buffers."""
import argparse
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2005_05826_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    problem = bench.make_problem(cfg)
    L = N.lib()
    n = problem.n_samples
    S = n // 2
    metric = bench.METRIC_CODE[cfg["metric"]]
    prec = 8 if cfg["precision"] == "fp64" else 4
    import torch
    dt = torch.float64 if prec == 8 else torch.float32
    pinned = [torch.empty((S * n,), dtype=dt, pin_memory=True).numpy() for _ in range(2)]
    pageable = [np.empty((S * n,), dtype=np.float64 if prec == 8 else np.float32) for _ in range(2)]
    ex, _keep = N.make_exec([0], 0)
    for rep in range(args.reps):
        t0 = time.perf_counter()
        plan = C.c_void_p()
        N.check(L.sf_plan_create(problem.ref, metric, prec, 0, S, C.byref(ex), C.byref(plan)))
        t1 = time.perf_counter()
        N.check(L.sf_plan_run(plan, 1))
        N.check(L.sf_plan_sync(plan))
        t2 = time.perf_counter()
        N.check(L.sf_plan_download(plan, N.ptr(pinned[0]), N.ptr(pinned[1])))
        t3 = time.perf_counter()
        L.sf_plan_destroy(plan)
        t4 = time.perf_counter()
        st = N.sf_stats()
        N.check(L.sf_compute_stripes(problem.ref, metric, prec, 0, S, N.ptr(pinned[0]), N.ptr(pinned[1]),
                                     1, C.byref(ex), C.byref(st)))
        t5 = time.perf_counter()
        N.check(L.sf_compute_stripes(problem.ref, metric, prec, 0, S, N.ptr(pageable[0]), N.ptr(pageable[1]),
                                     1, C.byref(ex), C.byref(st)))
        t6 = time.perf_counter()
        print(f"rep {rep}: create {t1-t0:.3f}s run+sync {t2-t1:.3f}s download {t3-t2:.3f}s destroy {t4-t3:.3f}s | "
              f"compute_stripes pinned {t5-t4:.3f}s pageable {t6-t5:.3f}s (device total {st.total_ms:.1f} ms)",
              flush=True)


if __name__ == "__main__":
    main()
