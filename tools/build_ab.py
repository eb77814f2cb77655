#!/usr/bin/env python
"""Build A/B variants of the product library (tile shapes of the split
kernel) into tools/ab/lib_<name>.so; run them with SF_LIB=<path>. The
product library itself is built with the defaults (build.py)."""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2005_05826_b200 import build  # noqa: E402

VARIANTS = {
    # light column kernel: window stripes / member loads in flight / threads
    "lw12800u8": dict(SF_LIGHT_WIN=12800, SF_LIGHT_UNROLL=8, SF_LIGHT_NT=1024),
    "lw6400u4": dict(SF_LIGHT_WIN=6400, SF_LIGHT_UNROLL=4, SF_LIGHT_NT=1024),
    "lw6400u8": dict(SF_LIGHT_WIN=6400, SF_LIGHT_UNROLL=8, SF_LIGHT_NT=1024),
    "lw4224u4n512": dict(SF_LIGHT_WIN=4224, SF_LIGHT_UNROLL=4, SF_LIGHT_NT=512),
    "lnostream": dict(SF_LIGHT_STREAM=0),
    "lnochunk": dict(SF_LIGHT_CHUNK=0),
    "lu2": dict(SF_LIGHT_UNROLL=2),
    "lu8": dict(SF_LIGHT_UNROLL=8),
    "lu6": dict(SF_LIGHT_UNROLL=6),
    # weighted split: dense rows per cp.async stage / light member loads in flight
    "wsr16": dict(SF_WS_R=16),
    "wsu2": dict(SF_WS_UNROLL=2),
    "wsu8": dict(SF_WS_UNROLL=8),
    "v16u1f1": dict(V=16, UC=1, NW=8, MINB=2, FG=1),
    "v16u1f4": dict(V=16, UC=1, NW=8, MINB=2, FG=4),
    "v8u2f1": dict(V=8, UC=2, NW=8, MINB=2, FG=1),
    "v8u2f4": dict(V=8, UC=2, NW=8, MINB=2, FG=4),
    "v4u4f4": dict(V=4, UC=4, NW=8, MINB=2, FG=4),
    "v8u1f4m3": dict(V=8, UC=1, NW=8, MINB=3, FG=4),
    "v6u2f2m3": dict(V=6, UC=2, NW=8, MINB=3, FG=2),
    "v4u2f4m4": dict(V=4, UC=2, NW=8, MINB=4, FG=4),
    "v12u1f4": dict(V=12, UC=1, NW=8, MINB=2, FG=4),
    "v8u2f2": dict(V=8, UC=2, NW=8, MINB=2, FG=2),
    "v8u1f2m3": dict(V=8, UC=1, NW=8, MINB=3, FG=2),
    "v4u2f2m3": dict(V=4, UC=2, NW=8, MINB=3, FG=2),
    "v16u1f16m1": dict(V=16, UC=1, NW=8, MINB=1, FG=16),
    "v16u1f8m1": dict(V=16, UC=1, NW=8, MINB=1, FG=8),
    "v24u1f8m1": dict(V=24, UC=1, NW=8, MINB=1, FG=8),
    "v32u1f8m1": dict(V=32, UC=1, NW=4, MINB=1, FG=8),
    "v16u1f4n4m4": dict(V=16, UC=1, NW=4, MINB=4, FG=4),
}


def one(name, cfg):
    defines = [f"-D{k}={v}" if k.startswith("SF_") else f"-DSF_SPLIT_{k}={v}" for k, v in cfg.items()]
    out = ROOT / "tools" / "ab" / f"lib_{name}.so"
    build.build_native(force=True, out=out, defines=defines)
    return name


if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    with ThreadPoolExecutor(4) as ex:
        for n in ex.map(lambda n: one(n, VARIANTS[n]), names):
            print("built", n)
