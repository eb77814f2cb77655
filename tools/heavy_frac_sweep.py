#!/usr/bin/env python
"""Heavy/light threshold sweep (SF_HEAVY_FRAC) of the split path on one
instance: device times of the whole step, the heavy phase and the prep +
light scatter, per threshold. Usage: python tools/heavy_frac_sweep.py c3 0.03 0.02 ..."""
import ctypes as C
import json
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2005_05826_b200 import _native as N  # noqa: E402


def main():
    cfg_name = sys.argv[1]
    fracs = sys.argv[2:]
    cfg = bench.CONFIGS[cfg_name]
    problem = bench.make_problem(cfg)
    L = N.lib()
    n = problem.n_samples
    metric = bench.METRIC_CODE[cfg["metric"]]
    prec = 8 if cfg["precision"] == "fp64" else 4
    for f in fracs:
        os.environ["SF_HEAVY_FRAC"] = f
        ex, _keep = N.make_exec([0])
        plan = C.c_void_p()
        N.check(L.sf_plan_create(problem.ref, metric, prec, 0, n // 2, C.byref(ex), C.byref(plan)))
        st = N.sf_stats()
        tot, strp, prep = [], [], []
        for i in range(4):
            N.check(L.sf_plan_run(plan, 1))
            N.check(L.sf_plan_sync(plan))
            N.check(L.sf_plan_stats(plan, C.byref(st)))
            if i >= 1:
                tot.append(st.total_ms)
                strp.append(st.stripe_ms)
                prep.append(st.embed_ms)
        print(json.dumps({"config": cfg_name, "heavy_frac": float(f), "total_ms": statistics.median(tot),
                          "heavy_ms": statistics.median(strp), "prep_light_ms": statistics.median(prep),
                          "light_pairs_plus": st.updates_exec, "gemm": os.environ.get("SF_HEAVY_GEMM", "1")}),
              flush=True)
        L.sf_plan_destroy(plan)


if __name__ == "__main__":
    main()
