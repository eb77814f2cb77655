#!/usr/bin/env python
"""A/B the stripe kernels on one synthetic instance (generated once).

  python tools/kernel_ab.py --config c3 --kernels 2,3,4 --reps 2 [--stripes N]
Prints one JSON line per kernel: device ms per full run, U_exec, and bitwise
agreement of the stripes with the first kernel listed.
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2005_05826_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="small")
    ap.add_argument("--kernels", default="2,3,4")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--stripes", type=int, default=0)
    ap.add_argument("--metric", default=None)
    ap.add_argument("--precision", default=None)
    ap.add_argument("--env", default="", help="NAME=v1,v2,... : rerun each kernel per value")
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    if args.metric:
        cfg["metric"] = args.metric
    if args.precision:
        cfg["precision"] = args.precision
    problem = bench.make_problem(cfg)
    L = N.lib()
    metric = bench.METRIC_CODE[cfg["metric"]]
    prec = 8 if cfg["precision"] == "fp64" else 4
    n = problem.n_samples
    S = n // 2
    stop = min(S, args.stripes) if args.stripes else S
    ref = None
    import os
    runs = []
    for k in [int(x) for x in args.kernels.split(",")]:
        if args.env:
            name, vals = args.env.split("=")
            runs += [(k, name, v) for v in vals.split(",")]
        else:
            runs.append((k, None, None))
    for k, ename, evalue in runs:
        if ename:
            if evalue == "":
                os.environ.pop(ename, None)  # empty value: variable unset
            else:
                os.environ[ename] = evalue
        ex, _keep = N.make_exec([0], k)
        plan = C.c_void_p()
        N.check(L.sf_plan_create(problem.ref, metric, prec, 0, stop, C.byref(ex), C.byref(plan)))
        st = N.sf_stats()
        times = []
        for _ in range(args.reps + 1):
            N.check(L.sf_plan_run(plan, 1))
            N.check(L.sf_plan_sync(plan))
            N.check(L.sf_plan_stats(plan, C.byref(st)))
            times.append((st.total_ms, st.stripe_ms))
        dt = np.float64 if prec == 8 else np.float32
        d = np.empty((stop, n), dt)
        t = np.empty((stop, n), dt)
        N.check(L.sf_plan_download(plan, N.ptr(d), N.ptr(t)))
        L.sf_plan_destroy(plan)
        same = None
        rel = None
        if ref is None:
            ref = (d, t)
        else:
            same = bool(np.array_equal(ref[0], d) and np.array_equal(ref[1], t))
            rel = max(float(np.max(np.abs(x.astype(np.float64) - y) / np.maximum(np.abs(y), 1e-300)))
                      for x, y in ((d, ref[0]), (t, ref[1])))
        best = min(times[1:])
        print(json.dumps({"kernel": k, "total_ms": best[0], "stripe_ms": best[1],
                          "updates_alg": st.updates_alg, "updates_exec": st.updates_exec,
                          "alg_per_s": st.updates_alg / (best[0] / 1e3), "bitwise_same_as_first": same, "max_rel_diff_vs_first": rel,
                          "env": f"{ename}={evalue}" if ename else None}),
              flush=True)


if __name__ == "__main__":
    main()
