#!/usr/bin/env python
"""A/B of split-kernel tile shapes (tools/build_ab.py libraries) on one
instance: per library, a resident plan over stripes [0, X), device times of
the stripe kernel and the whole step, and a bitwise comparison of the
stripes with the first library's. Usage:
  python tools/split_ab.py --config c3 --stripes 2048 lib1.so lib2.so ..."""
import argparse
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2005_05826_b200 import _native as N  # noqa: E402


def load(path):
    h = C.CDLL(str(path))
    for name, (res, args) in N.SIGNATURES.items():
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = args
    return h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--stripes", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("libs", nargs="+")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    problem = bench.make_problem(cfg)
    n = problem.n_samples
    stop = min(n // 2, args.stripes)
    metric = bench.METRIC_CODE[cfg["metric"]]
    prec = 8 if cfg["precision"] == "fp64" else 4
    ref = None
    for path in args.libs:
        L = load(path)
        ex, _keep = N.make_exec([0], 0)
        plan = C.c_void_p()
        st = N.sf_stats()
        rc = L.sf_plan_create(problem.ref, metric, prec, 0, stop, C.byref(ex), C.byref(plan))
        if rc:
            print(json.dumps({"lib": Path(path).name, "error": L.sf_last_error().decode()}), flush=True)
            continue
        tot, strp = [], []
        for i in range(2 + args.reps):
            L.sf_plan_run(plan, 1)
            L.sf_plan_sync(plan)
            L.sf_plan_stats(plan, C.byref(st))
            if i >= 2:
                tot.append(st.total_ms)
                strp.append(st.stripe_ms)
        d = np.empty((stop, n), np.float64 if prec == 8 else np.float32)
        t = np.empty_like(d)
        L.sf_plan_download(plan, N.ptr(d), N.ptr(t))
        same = None
        if ref is None:
            ref = (d, t)
        else:
            same = bool(np.array_equal(d, ref[0]) and np.array_equal(t, ref[1]))
        rec = {"lib": Path(path).name, "stripes": stop, "total_ms": statistics.median(tot),
               "stripe_ms": statistics.median(strp), "fp64_ops": st.fp64_ops, "bitwise_equal_to_first": same}
        print(json.dumps(rec), flush=True)
        L.sf_plan_destroy(plan)
        L.sf_trim_memory(0)


if __name__ == "__main__":
    main()
