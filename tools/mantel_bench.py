#!/usr/bin/env python
"""Mantel at scale on device: the fp64-vs-fp32 validation of
a benchmark configuration's matrix (acceptance.cpp:282-309's check; C3
unweighted, C4 generalized alpha=0.5), with 999 permutations of the
reference's stream, timed end to end, plus the fp32-vs-fp64 drift
statistics of the two matrices.

  python tools/mantel_bench.py [--config c3|c4] [--perms 999]
Prints one JSON line (r, p, drift, seconds, gathered pairs per second).
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2005_05826_b200 import _native as N  # noqa: E402


def full_matrix(problem, cfg, prec):
    """The n x n matrix through sf_compute_distance_matrix (device-resident
    stripes, device condense)."""
    n = problem.n_samples
    out = np.empty((n, n))
    ex, _keep = N.make_exec([0], alpha=cfg.get("alpha", 1.0))
    N.check(N.lib().sf_compute_distance_matrix(problem.ref, bench.METRIC_CODE[cfg["metric"]], prec, N.ptr(out),
                                               C.byref(ex), None))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--perms", type=int, default=999)
    ap.add_argument("--seed", type=int, default=7)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    problem = bench.make_problem(cfg)
    n = problem.n_samples
    t0 = time.perf_counter()
    m64 = full_matrix(problem, cfg, 8)
    m32 = full_matrix(problem, cfg, 4)
    t1 = time.perf_counter()
    iu = np.triu_indices(n, 1)
    a64, a32 = m64[iu], m32[iu]
    diff = np.abs(a32 - a64)
    nz = a64 != 0
    drift = {"max_abs": float(diff.max()), "mean_abs": float(diff.mean()),
             "max_rel": float(np.max(diff[nz] / a64[nz])) if nz.any() else 0.0,
             "exact_zeros_fp64": int((~nz).sum()), "zeros_mismatched": int(np.sum(~nz & (a32 != 0)))}
    del a64, a32, diff, nz
    r = C.c_double()
    p = C.c_double()
    N.check(N.lib().sf_mantel(n, N.ptr(m64), N.ptr(m32), args.perms, args.seed, 0, C.byref(r), C.byref(p)))
    t2 = time.perf_counter()
    pairs = n * (n - 1) // 2
    # host baseline: one permutation's cross term, vectorised numpy gather
    # (the reference's loop is scalar: validate.cpp:131-149)
    x = m64[iu] - m64[iu].mean()
    perm = np.random.default_rng(0).permutation(n)
    th0 = time.perf_counter()
    y = m32[perm[iu[0]], perm[iu[1]]]
    float(x @ (y - y.mean()))
    host_perm_s = time.perf_counter() - th0
    print(json.dumps({
        "what": f"mantel({cfg['metric']} fp64 DM, fp32 DM) on device, reference permutation stream",
        "config": args.config, "fp32_vs_fp64": drift,
        "workload": cfg["workload"], "n_samples": n, "permutations": args.perms, "seed": args.seed,
        "r": r.value, "r_squared": r.value ** 2, "p_value": p.value,
        "mantel_seconds": t2 - t1, "matrices_seconds": t1 - t0,
        "gathered_pairs_per_s": pairs * (args.perms + 1) / (t2 - t1),
        "host_numpy_seconds_per_permutation": host_perm_s,
        "host_numpy_seconds_extrapolated": host_perm_s * (args.perms + 1),
    }), flush=True)


if __name__ == "__main__":
    main()
