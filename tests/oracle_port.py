"""ctypes binding of oracle/liboracle_port.so — the CPU restatement.
TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py cpu_baseline)."""
import ctypes as C
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent.parent / "oracle" / "liboracle_port.so"
_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(LIB))
        _lib.orc_compute_stripes.restype = C.c_int
        _lib.orc_compute_stripes.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int]
        _lib.orc_embed_rows.restype = C.c_int
        _lib.orc_embed_rows.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        _lib.orc_condense.restype = C.c_int
        _lib.orc_condense.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    return _lib


def compute_stripes(problem, metric: int, prec: int, start: int = 0, stop: int = -1,
                    finalize: bool = True, threads: int = 1, batch: int = 64):
    """problem: paper_2005_05826_b200._native.Problem (same struct layout)."""
    n = problem.n_samples
    if stop < 0:
        stop = n // 2
    dt = np.float64 if prec == 8 else np.float32
    d = np.zeros((stop - start, n), dt)
    t = np.zeros((stop - start, n), dt)
    rc = lib().orc_compute_stripes(C.cast(C.pointer(problem.struct), C.c_void_p), metric, prec,
                                   start, stop, d.ctypes.data, t.ctypes.data if metric != 2 else None,
                                   int(finalize), threads, batch)
    assert rc == 0
    return d, (t if metric != 2 else None)


def compute_stripes_generalized(problem, alpha: float, prec: int, start: int = 0, stop: int = -1,
                                finalize: bool = True, threads: int = 1, batch: int = 64):
    """Generalized UniFrac (extension; parity unpinned: not in the reference)."""
    n = problem.n_samples
    if stop < 0:
        stop = n // 2
    dt = np.float64 if prec == 8 else np.float32
    d = np.zeros((stop - start, n), dt)
    t = np.zeros((stop - start, n), dt)
    f = lib().orc_compute_stripes_generalized
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                  C.c_int, C.c_int, C.c_int]
    rc = f(C.cast(C.pointer(problem.struct), C.c_void_p), float(alpha), prec, start, stop,
           d.ctypes.data, t.ctypes.data, int(finalize), threads, batch)
    assert rc == 0
    return d, t


def embed_rows(problem, weighted: bool):
    out = np.zeros((problem.n_rows, problem.n_samples), np.float64)
    rc = lib().orc_embed_rows(C.cast(C.pointer(problem.struct), C.c_void_p), int(weighted),
                              out.ctypes.data)
    assert rc == 0
    return out


def condense(prec: int, n: int, dist):
    out = np.zeros((n, n), np.float64)
    rc = lib().orc_condense(prec, n, np.ascontiguousarray(dist).ctypes.data, out.ctypes.data)
    return out if rc == 0 else None


def time_sample(problem, metric: int, prec: int, rows: int, start: int, stop: int, threads: int):
    """Bounded CPU sample (first `rows` postorder rows x stripes [start, stop)):
    returns (seconds, updates). Used by bench.py's cpu_baseline leg only."""
    import time
    n = problem.n_samples
    dt = np.float64 if prec == 8 else np.float32
    d = np.zeros((stop - start, n), dt)
    t = np.zeros((stop - start, n), dt)
    f = lib().orc_compute_stripes_rows
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                  C.c_int, C.c_int, C.c_int, C.c_int]
    t0 = time.perf_counter()
    rc = f(C.cast(C.pointer(problem.struct), C.c_void_p), metric, prec, start, stop, d.ctypes.data,
           t.ctypes.data if metric != 2 else None, 0, threads, 64, rows)
    secs = time.perf_counter() - t0
    assert rc == 0
    return secs, rows * (stop - start) * n


def sparse_stripes(problem, metric: int, prec: int, start: int = 0, stop: int = -1,
                   finalize: bool = True, threads: int = 1):
    """orc_sparse_stripes: the reference's arithmetic over each sample's
    present rows only (no dense embedding): the checker at C3/C5 scale."""
    n = problem.n_samples
    if stop < 0:
        stop = n // 2
    dt = np.float64 if prec == 8 else np.float32
    d = np.zeros((stop - start, n), dt)
    t = np.zeros((stop - start, n), dt)
    f = lib().orc_sparse_stripes
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int]
    rc = f(C.cast(C.pointer(problem.struct), C.c_void_p), metric, prec, start, stop, d.ctypes.data,
           t.ctypes.data if metric != 2 else None, int(finalize), threads)
    assert rc == 0
    return d, (t if metric != 2 else None)
