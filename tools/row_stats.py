#!/usr/bin/env python
"""Row-occupancy statistics of a synthetic instance (CPU, numpy): the numbers
behind DESIGN.md §2 (union vs intersection work per slot, the heavy/light
split) — so they can be re-measured.

  python tools/row_stats.py --seed 3 --n 25000 --leaves 300000   # C3, ~3 min

m_e = |S_e| (samples present under row e); X_e = S_e or its complement
(|X_e| = min(m_e, n - m_e)).
  union work per slot        = sum_e [C(n,2) - C(n-m_e,2)] / C(n,2)
  intersection work per slot = sum_e C(|X_e|,2) / C(n,2)
and, per heavy threshold T, the heavy rows' u bits per column and the light
rows' shared rows per slot.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2005_05826_b200 import stripefrac as sf  # noqa: E402


def presence_counts(problem):
    n, E = problem.n_samples, problem.n_rows
    nb = (n + 7) // 8
    rows = np.zeros((E, nb), np.uint8)
    fp, si, lf = problem.feat_ptr, problem.sample_idx, problem.leaf_feature
    for r in range(E):
        f = lf[r]
        if f >= 0:
            b = np.zeros(n, np.uint8)
            b[si[fp[f]:fp[f + 1]]] = 1
            rows[r] = np.packbits(b, bitorder="little")
    for r in range(E):
        q = problem.parent_row[r]
        if q >= 0:
            rows[q] |= rows[r]
    lut = np.array([bin(i).count("1") for i in range(256)], np.int64)
    return lut[rows].sum(1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--n", type=int, default=25000)
    ap.add_argument("--leaves", type=int, default=300000)
    ap.add_argument("--density", type=float, default=0.002)
    args = ap.parse_args()
    t0 = time.time()
    inst = sf.random_instance(args.seed, args.n, args.leaves, args.density, 0, finalize_tree=False)
    p = sf.flatten(inst.tree, inst.table)
    m = presence_counts(p).astype(np.float64)
    n = args.n
    x = np.minimum(m, n - m)
    c2 = lambda v: v * (v - 1) / 2  # noqa: E731
    pairs = c2(n)
    print(f"instance seed={args.seed} n={n} E={p.n_rows} ({time.time() - t0:.0f}s)")
    print(f"mean |S_e| {m.mean():.1f} ({m.mean() / n:.4f} of n)")
    print(f"union work per slot        {(c2(n) - c2(n - m)).sum() / pairs:10.1f}")
    print(f"intersection (S) per slot  {c2(m).sum() / pairs:10.1f}")
    print(f"intersection (X) per slot  {c2(x).sum() / pairs:10.1f}")
    print(f"dense rows (m > n/2)       {(m > n / 2).sum():10d}")
    print("T (|X|>=T heavy)  heavy rows  u-bits/col  heavy shared/slot  light shared/slot")
    for frac in (0.004, 0.008, 0.01, 0.012, 0.016, 0.02, 0.04, 0.06, 0.14):
        T = max(2, int(frac * n))
        h = x >= T
        print(f"{T:6d} ({frac:5.3f}n) {h.sum():10d} {x[h].sum() / n:11.0f} "
              f"{(x[h] ** 2).sum() / n ** 2:18.1f} {(x[~h] ** 2).sum() / n ** 2:18.1f}")


if __name__ == "__main__":
    main()
