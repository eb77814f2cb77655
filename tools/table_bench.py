#!/usr/bin/env python
"""Sparse table ingestion at C3 size: the C3 synthetic table
(25k samples, ~15M entries) written as feature<TAB>sample<TAB>count triplets
in shuffled order, loaded by the reference's own load_table_file
(oracle/_ref/ref_driver table ... time; test infrastructure) and by the
native parallel loader (sfh_load_table_sparse). Host only.

  python tools/table_bench.py [--config c3] [--path /tmp/c3_sparse.tsv]
"""
import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2005_05826_b200 import stripefrac as sf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--path", default="/tmp/sf_sparse_table.tsv")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    inst = sf.random_instance(cfg["seed"], cfg["n"], cfg["leaves"], cfg["density"], 0, finalize_tree=False)
    t = inst.table
    f_of = np.repeat(np.arange(t.n_features()), np.diff(t.feat_ptr))
    perm = np.random.default_rng(0).permutation(f_of.size)
    with open(args.path, "w") as fh:
        fid = t.feature_ids
        sid = t.sample_ids
        fo, si, ct = f_of.tolist(), t.sample_idx.tolist(), t.counts.tolist()
        for i in perm.tolist():
            fh.write(f"{fid[fo[i]]}\t{sid[si[i]]}\t{ct[i]!r}\n")
    size = os.path.getsize(args.path)
    rec = {"what": "sparse TSV table load", "config": args.config, "entries": int(f_of.size), "bytes": size,
           "threads": os.cpu_count()}
    drv = ROOT / "oracle" / "_ref" / "ref_driver"
    if drv.exists():
        out = subprocess.run([str(drv), "table", args.path, "tsv-sparse", "time"], capture_output=True, text=True,
                             check=True).stdout
        ref = json.loads(out)
        rec["reference_seconds"] = ref.get("seconds", ref.get("error"))
    for th in (1, 0):
        t0 = time.perf_counter()
        tab = sf.load_table_file(args.path, "tsv-sparse", threads=th)
        rec[f"native_seconds_threads_{th or 'all'}"] = round(time.perf_counter() - t0, 3)
    assert tab.n_samples() == t.n_samples() and int(tab.feat_ptr[-1]) == int(f_of.size)
    os.remove(args.path)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
