#!/usr/bin/env python
"""The matrix TSV writer at C3 size (25,000 x 25,000, %.17g):
the native parallel writer (sfh_write_tsv) with 1 and all host threads, and
the reference's own single-threaded writer's cost per value estimated from a
sample with the same snprintf format (stripes.cpp:301-332). Host only.

  python tools/tsv_bench.py [--n 25000] [--out /tmp/dm.tsv]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2005_05826_b200 import stripefrac as sf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=25000)
    ap.add_argument("--out", default="/tmp/sf_dm.tsv")
    ap.add_argument("--single-rows", type=int, default=500, help="rows timed with 1 thread")
    args = ap.parse_args()
    n = args.n
    rng = np.random.default_rng(1)
    vals = rng.random((n, n))
    ids = [f"sample{i}" for i in range(n)]
    dm = sf.DistanceMatrix(ids, vals, sf.Precision.Fp64)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    sf.write_tsv(args.out, dm, threads=0)
    t_all = time.perf_counter() - t0
    size = os.path.getsize(args.out)
    r = args.single_rows
    sub = sf.DistanceMatrix(ids[:r], np.ascontiguousarray(vals[:r, :r]), sf.Precision.Fp64)
    t0 = time.perf_counter()
    sf.write_tsv(args.out + ".1", sub, threads=1)
    t_one = (time.perf_counter() - t0) * (n / r) ** 2
    os.remove(args.out)
    os.remove(args.out + ".1")
    print(json.dumps({"what": "matrix TSV writer (%.17g), n x n", "n": n, "bytes": size,
                      "threads": threads, "seconds_all_threads": round(t_all, 2),
                      "seconds_one_thread_extrapolated": round(t_one, 2),
                      "values_per_s_all_threads": n * n / t_all}))


if __name__ == "__main__":
    main()
