#!/usr/bin/env python
"""Parity evidence at a benchmark configuration too large for the pytest
suite's time budget (C5: 113,721 samples; generating the instance alone
draws n x F = 3.4e10 uniforms, ~4-5 min): the GPU default path on stripe
sub-ranges vs the sparse restatement of the reference (oracle/, pinned bit
for bit to the reference's golden vectors and to the reference itself at C2,
tests/test_oracle.py, tests/test_parity_at_scale.py). One JSON line per check.

  python tools/parity_at_scale.py --config c5 --ranges 0:8,28426:28434,56852:56860
"""
import argparse
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import oracle_port as op  # noqa: E402  (test infrastructure: the checker)
from paper_2005_05826_b200 import _native as N  # noqa: E402


def gpu(problem, metric, prec, start, stop, finalize):
    n = problem.n_samples
    dt = np.float64 if prec == 8 else np.float32
    d = np.full((stop - start, n), np.nan, dt)
    t = np.full((stop - start, n), np.nan, dt)
    ex, _keep = N.make_exec([0])
    N.check(N.lib().sf_compute_stripes(problem.ref, metric, prec, start, stop, N.ptr(d), N.ptr(t), int(finalize),
                                       C.byref(ex), None))
    return d, t


def rel(got, want):
    got, want = got.astype(np.float64), want.astype(np.float64)
    nz = want != 0
    r = float(np.max(np.abs(got - want)[nz] / np.abs(want[nz]))) if nz.any() else 0.0
    return r, int(np.sum(~nz & (got != 0)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--ranges", default="0:8,28426:28434,56852:56860")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    problem = bench.make_problem(cfg)
    gen_s = time.perf_counter() - t0
    metric = bench.METRIC_CODE[cfg["metric"]]
    ulp = float(np.finfo(np.float32).eps)
    for rng in args.ranges.split(","):
        a, b = (int(x) for x in rng.split(":"))
        ref64 = op.sparse_stripes(problem, metric, 8, a, b, finalize=False, threads=threads)
        ref32 = op.sparse_stripes(problem, metric, 4, a, b, finalize=False, threads=threads)
        g64 = gpu(problem, metric, 8, a, b, False)
        g32 = gpu(problem, metric, 4, a, b, False)
        for i, name in enumerate(("d", "t")):
            r64, z64 = rel(g64[i], ref64[i])
            r32, _ = rel(g32[i], ref64[i])
            drift, _ = rel(ref32[i], ref64[i])
            r32r, _ = rel(g32[i], ref32[i])
            rec = {"config": args.config, "workload": cfg["workload"], "stripes": [a, b], "value": name,
                   "fp64_max_rel_vs_reference_restatement": r64, "fp64_zeros_missed": z64,
                   "fp32_max_rel_vs_reference_fp64": r32, "reference_fp32_drift_vs_fp64": drift,
                   "fp32_max_rel_vs_reference_fp32": r32r, "slots": int(ref64[i].size),
                   "gate_fp64": "<= 1e-12 relative", "gate_fp32": "<= 1 fp32 ulp of the reference fp64",
                   "pass": bool(r64 <= 1e-12 and z64 == 0 and r32 <= ulp), "instance_seconds": round(gen_s, 1)}
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
