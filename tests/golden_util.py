"""Golden-vector helpers (tests only). Fixtures in tests/golden/ come from the
REFERENCE itself: oracle/_ref/ref_driver golden (see tests/golden/make_golden.sh)."""
import gzip
import json
from pathlib import Path

import numpy as np

from paper_2005_05826_b200 import stripefrac as sf

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str):
    p = GOLDEN / name
    if p.suffix == ".gz":
        with gzip.open(p, "rt") as fh:
            return json.load(fh)
    with open(p) as fh:
        return json.load(fh)


def all_cases():
    cases = [load("demo.json")]
    cases += load("hand.json")
    cases += load("instances_small.json")
    cases += load("instances_medium.json.gz")
    cases += load("instances_wide.json.gz")
    return cases


def case_inputs(case):
    """(tree, table) exactly as the reference built them: feature order and
    sample totals preserved from the fixture."""
    tree = sf.parse_newick(case["newick"])
    lines = case["table"].rstrip("\n").split("\n")
    samples = lines[0].split("\t")[1:]
    index = {s: i for i, s in enumerate(samples)}
    feats = list(case["feature_ids"])
    fidx = {f: i for i, f in enumerate(feats)}
    per = [[] for _ in feats]
    for ln in lines[1:]:
        f, s, v = ln.split("\t")
        per[fidx[f]].append((index[s], float(v)))
    ptr, sidx, vals = [0], [], []
    for ent in per:
        for s, v in ent:
            sidx.append(s)
            vals.append(v)
        ptr.append(len(sidx))
    table = sf.SampleTable(samples, feats, ptr, sidx, vals, case["sample_totals"])
    return tree, table


def result(case, metric: str, precision: str, start=0, stop=None):
    for r in case["results"]:
        if r["metric"] == metric and r["precision"] == precision and r["start"] == start and (
                stop is None or r["stop"] == stop):
            return r
    return None


def stripes(r, n):
    dt = np.float32 if r["precision"] == "fp32" else np.float64
    d = np.array(r["distances"], dtype=np.float64).astype(dt).reshape(-1, n)
    t = np.array(r["totals"], dtype=np.float64).astype(dt).reshape(-1, n) if r["totals"] else None
    return d, t
