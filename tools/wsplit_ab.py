#!/usr/bin/env python
"""Weighted kernels A/B on one instance: the u-walk (12) vs the weighted
split (13) at several heavy thresholds (SF_WHEAVY_FRAC), device time per
step (CUDA events), the dense part's time, and the max relative difference
of 13 against 12 (both within 1e-12 of the reference; tests/test_wsplit.py).

  python tools/wsplit_ab.py --config c2 [--fracs 0.1,0.2,0.3] [--reps 3]
One JSON line per (kernel, frac)."""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2005_05826_b200 import _native as N  # noqa: E402


def run(problem, metric, prec, kernel, reps, stripes, alpha=1.0):
    L = N.lib()
    n = problem.n_samples
    S = stripes or n // 2
    ex, _keep = N.make_exec([0], kernel, alpha=alpha)
    plan = C.c_void_p()
    N.check(L.sf_plan_create(problem.ref, metric, prec, 0, S, C.byref(ex), C.byref(plan)))
    st = N.sf_stats()
    ms, dense = [], []
    for i in range(reps + 1):
        N.check(L.sf_plan_run(plan, 1))
        N.check(L.sf_plan_sync(plan))
        N.check(L.sf_plan_stats(plan, C.byref(st)))
        if i:
            ms.append(st.total_ms)
            dense.append(st.tensor_ms)
    dt = np.float64 if prec == 8 else np.float32
    d = np.empty((S, n), dt)
    t = np.empty((S, n), dt)
    N.check(L.sf_plan_download(plan, N.ptr(d), N.ptr(t)))
    L.sf_plan_destroy(plan)
    return statistics.median(ms), statistics.median(dense), st, d, t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--fracs", default="0.1,0.2,0.3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--prec", default="")
    ap.add_argument("--stripes", type=int, default=0)
    ap.add_argument("--no-uwalk", action="store_true")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    problem = bench.make_problem(cfg)
    metric = bench.METRIC_CODE[cfg["metric"]]
    prec = {"fp64": 8, "fp32": 4}[args.prec or cfg["precision"]]
    base = None
    if not args.no_uwalk:
        ms, _, st, d12, t12 = run(problem, metric, prec, 12, args.reps, args.stripes, cfg.get("alpha", 1.0))
        base = (d12, t12)
        print(json.dumps({"config": args.config, "kernel": 12, "prec": prec, "device_ms": round(ms, 3),
                          "fp64_ops": st.fp64_ops}), flush=True)
    for f in args.fracs.split(","):
        os.environ["SF_WHEAVY_FRAC"] = f
        ms, dms, st, d, t = run(problem, metric, prec, 13, args.reps, args.stripes, cfg.get("alpha", 1.0))
        rec = {"config": args.config, "kernel": 13, "prec": prec, "heavy_frac": float(f), "device_ms": round(ms, 3),
               "dense_ms": round(dms, 3), "pipe_ops": st.fp64_ops, "updates_exec": st.updates_exec}
        if base is not None:
            for nm, got, want in (("d", d, base[0]), ("t", t, base[1])):
                w = want.astype(np.float64)
                g = got.astype(np.float64)
                nz = w != 0
                rec[f"max_rel_{nm}_vs_12"] = float(np.max(np.abs(g[nz] - w[nz]) / np.abs(w[nz]))) if nz.any() else 0.0
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
