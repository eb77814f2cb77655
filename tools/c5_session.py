#!/usr/bin/env python
"""C5 (113,721 samples, 300k-tip tree, UW fp32; the paper's large set) on
one B200, one instance generation (n x F = 3.4e10 draws, minutes):

  * the 1/8 stripe shard of the 8-GPU configuration ([0, S/8)) and the full
    matrix: device time per step (CUDA events) and updates/s;
  * parity on stripe sub-ranges (first, middle, last incl. the wrap): the
    GPU path vs the sparse restatement of the reference (oracle/, test
    infrastructure; pinned bit-for-bit to the reference's own stripes at C2
    and C3), fp64 within 1e-12 relative, fp32 within one fp32 ulp of the
    reference's fp64.

One JSON line per measurement / check."""
import ctypes as C
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import oracle_port as op  # noqa: E402  (the checker)
from paper_2005_05826_b200 import _native as N  # noqa: E402

sys.path.insert(0, str(ROOT / "tools"))
from parity_at_scale import gpu, rel  # noqa: E402


def timed(problem, prec, a, b, reps):
    L = N.lib()
    ex, _keep = N.make_exec([0])
    plan = C.c_void_p()
    t0 = time.perf_counter()
    N.check(L.sf_plan_create(problem.ref, 1, prec, a, b, C.byref(ex), C.byref(plan)))
    create_s = time.perf_counter() - t0
    st = N.sf_stats()
    ms = []
    for i in range(reps + 1):
        N.check(L.sf_plan_run(plan, 1))
        N.check(L.sf_plan_sync(plan))
        N.check(L.sf_plan_stats(plan, C.byref(st)))
        if i:
            ms.append(st.total_ms)
    L.sf_plan_destroy(plan)
    L.sf_trim_memory(0)
    return create_s, statistics.median(ms), st


def main():
    cfg = bench.CONFIGS["c5"]
    t0 = time.perf_counter()
    problem = bench.make_problem(cfg)
    gen_s = time.perf_counter() - t0
    n, E = problem.n_samples, problem.n_rows
    S = n // 2
    threads = os.cpu_count() or 1
    for name, a, b, reps in (("shard 1/8 of the 8-GPU configuration", 0, S // 8, 3), ("full matrix", 0, S, 1)):
        create_s, ms, st = timed(problem, 4, a, b, reps)
        print(json.dumps({"config": "c5", "workload": cfg["workload"], "what": name, "stripes": [a, b],
                          "device_ms_per_step": ms, "updates_per_s": E * (b - a) * n / (ms / 1e3),
                          "plan_create_s": round(create_s, 3), "launches": st.launches,
                          "tensor_ms": st.tensor_ms, "tensor_ops": st.tensor_ops,
                          "instance_seconds": round(gen_s, 1)}), flush=True)
    ulp = float(np.finfo(np.float32).eps)
    for a, b in ((0, 8), (S // 2, S // 2 + 8), (S - 8, S)):
        ref64 = op.sparse_stripes(problem, 1, 8, a, b, finalize=False, threads=threads)
        g64 = gpu(problem, 1, 8, a, b, False)
        g32 = gpu(problem, 1, 4, a, b, False)
        ref32 = op.sparse_stripes(problem, 1, 4, a, b, finalize=False, threads=threads)
        for i, nm in enumerate(("d", "t")):
            r64, z64 = rel(g64[i], ref64[i])
            r32, _ = rel(g32[i], ref64[i])
            drift, _ = rel(ref32[i], ref64[i])
            print(json.dumps({"config": "c5", "check": f"UW {nm} stripes [{a},{b})",
                              "fp64_max_rel_vs_reference_restatement": r64, "fp64_zeros_missed": z64,
                              "fp32_max_rel_vs_reference_fp64": r32, "reference_fp32_drift_vs_fp64": drift,
                              "slots": int(ref64[i].size),
                              "pass": bool(r64 <= 1e-12 and z64 == 0 and r32 <= ulp)}), flush=True)


if __name__ == "__main__":
    main()
