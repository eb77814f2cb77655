"""Kernel 13 (weighted split: dense heavy rows + exact fixed-point light
scatter, csrc/wsplit_kernels.cuh) against the oracle's restatement of the
reference loops (kernels.hpp:55-66; oracle/stripefrac_oracle.c, pinned to the
reference's own goldens in tests/test_oracle.py).

Gates as for every weighted kernel: fp64 within 1e-12 RELATIVE with exact
zeros exact, fp32 within max(1e-5 |x|, 1e-6). Each case runs with the default
heavy threshold and with the two extreme splits (SF_WHEAVY_FRAC=0: every row
dense; 2: every row light), so both halves are checked on their own.
"""
import ctypes as C

import numpy as np
import pytest

import oracle_port as op
from paper_2005_05826_b200 import _native as N
from paper_2005_05826_b200 import stripefrac as sf
from test_gpu_parity import _assert_close, _dup_table, _gpu_stripes

pytestmark = pytest.mark.gpu

SPLITS = ["0", None, "2"]  # all heavy, default, all light


@pytest.fixture(scope="module")
def device_ok():
    assert N.lib().sf_device_count() >= 1, "no sm_100 device visible (GPU tests need a B200)"


def _run(problem, metric, prec, start, stop, monkeypatch, frac):
    if frac is None:
        monkeypatch.delenv("SF_WHEAVY_FRAC", raising=False)
    else:
        monkeypatch.setenv("SF_WHEAVY_FRAC", frac)
    return _gpu_stripes(problem, metric, prec, start, stop, N.KERNEL_WSPLIT)


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("metric", [2, 3])
def test_wsplit_matches_oracle(device_ok, metric, prec, monkeypatch):
    """Random instances (odd and even n, dense and sparse tables), full,
    partial and single-stripe ranges (the wrap included)."""
    for seed, n, leaves, dens in [(71, 200, 700, 0.01), (72, 97, 300, 0.05), (73, 64, 64, 0.3),
                                  (74, 301, 2000, 0.004)]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        for start, stop in [(0, S), (S // 3, S), (3, 4), (S - 1, S)]:
            wd, wt = op.compute_stripes(problem, metric, prec, start, stop)
            for frac in SPLITS:
                d, t, st = _run(problem, metric, prec, start, stop, monkeypatch, frac)
                _assert_close(metric, prec, False, d, wd, N.KERNEL_WSPLIT)
                if wt is not None:
                    _assert_close(metric, prec, False, t, wt, N.KERNEL_WSPLIT)


@pytest.mark.parametrize("metric", [2, 3])
def test_wsplit_identical_samples_are_exactly_zero(device_ok, metric, monkeypatch):
    """Duplicated samples: the dense terms are |u - u| L = 0 and the light
    part's fixed-point sums cancel exactly (AL_k + AL_l - 2 AL_k = 0)."""
    inst = sf.random_instance(65, 120, 400, 0.03)
    table = _dup_table(inst, {7: 3, 100: 3, 61: 60})
    problem = sf.flatten(inst.tree, table)
    n, S = 120, 60
    wd, _ = op.compute_stripes(problem, metric, 8, 0, S)
    for frac in SPLITS:
        d, t, _ = _run(problem, metric, 8, 0, S, monkeypatch, frac)
        dm = op.condense(8, n, d)
        for a, b in ((3, 7), (3, 100), (7, 100), (60, 61)):
            assert dm[a, b] == 0.0 and dm[b, a] == 0.0
        _assert_close(metric, 8, False, d, wd, N.KERNEL_WSPLIT)


@pytest.mark.parametrize("prec", [8, 4])
def test_wsplit_even_n_duplicate_half_stripe(device_ok, prec, monkeypatch):
    """Even n: the last stripe's two copies of each pair agree bitwise."""
    inst = sf.random_instance(66, 130, 500, 0.02)
    problem = sf.flatten(inst.tree, inst.table)
    for frac in SPLITS:
        d, t, _ = _run(problem, 3, prec, 60, 65, monkeypatch, frac)
        assert np.array_equal(d[-1, :65], d[-1, 65:]) and np.array_equal(t[-1, :65], t[-1, 65:])


def test_wsplit_wide_lengths(device_ok, monkeypatch):
    """Branch lengths over 1e-12 .. 2 (the fixed-point grid keeps the light
    terms exact; the dense part adds them directly)."""
    inst = sf.random_instance(75, 150, 600, 0.02, finalize_tree=False)
    rng = np.random.default_rng(5)
    tree = inst.tree
    tree.length = np.ascontiguousarray(tree.length * 10.0 ** rng.uniform(-12, 0, tree.length.size))
    problem = sf.flatten(tree, inst.table)
    wd, wt = op.compute_stripes(problem, 3, 8, 0, 75)
    for frac in SPLITS:
        d, t, _ = _run(problem, 3, 8, 0, 75, monkeypatch, frac)
        _assert_close(3, 8, False, d, wd, N.KERNEL_WSPLIT)
        _assert_close(3, 8, False, t, wt, N.KERNEL_WSPLIT)


def test_wsplit_rejects_unweighted(device_ok):
    inst = sf.random_instance(3, 10, 12, 0.3)
    problem = sf.flatten(inst.tree, inst.table)
    with pytest.raises(N.NativeError):
        _gpu_stripes(problem, 1, 8, 0, 5, N.KERNEL_WSPLIT)


def _gen13(problem, alpha, prec, start, stop, monkeypatch, frac):
    if frac is None:
        monkeypatch.delenv("SF_WHEAVY_FRAC", raising=False)
    else:
        monkeypatch.setenv("SF_WHEAVY_FRAC", frac)
    n = problem.n_samples
    dt = np.float64 if prec == 8 else np.float32
    d = np.full((stop - start, n), np.nan, dt)
    t = np.full((stop - start, n), np.nan, dt)
    ex, _keep = N.make_exec([0], N.KERNEL_WSPLIT, False, 0, alpha)
    N.check(N.lib().sf_compute_stripes(problem.ref, N.SF_GENERALIZED, prec, start, stop, N.ptr(d), N.ptr(t), 1,
                                       C.byref(ex), None))
    return d, t


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("alpha", [0.0, 0.5, 1.0, 1.7])
def test_wsplit_generalized_matches_oracle(device_ok, alpha, prec, monkeypatch):
    """Generalized UniFrac (extension; parity unpinned: the reference has no
    generalized metric) on the weighted split against the oracle's statement
    of the published form: fp64 within 1e-12 relative (alpha = 0.5 through
    rsqrt, other exponents through pow), fp32 within max(1e-5 |x|, 1e-6)."""
    for seed, n, leaves, dens in [(81, 150, 500, 0.02), (82, 41, 120, 0.1), (83, 200, 900, 0.01)]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        for start, stop in [(0, S), (S // 3, S)]:
            wd, wt = op.compute_stripes_generalized(problem, alpha, prec, start, stop)
            for frac in SPLITS:
                d, t = _gen13(problem, alpha, prec, start, stop, monkeypatch, frac)
                for got, want in ((d, wd), (t, wt)):
                    if prec == 8:
                        err = np.abs(got - want)
                        assert np.all(err <= 1e-12 * np.abs(want)), f"alpha {alpha} frac {frac}: {err.max()}"
                    else:
                        w = want.astype(np.float64)
                        assert np.all(np.abs(got.astype(np.float64) - w) <= np.maximum(1e-5 * np.abs(w), 1e-6))


def test_wsplit_generalized_identical_samples_are_exactly_zero(device_ok, monkeypatch):
    inst = sf.random_instance(65, 120, 400, 0.03)
    table = _dup_table(inst, {7: 3, 100: 3, 61: 60})
    problem = sf.flatten(inst.tree, table)
    for frac in SPLITS:
        d, _ = _gen13(problem, 0.5, 8, 0, 60, monkeypatch, frac)
        dm = op.condense(8, 120, d)
        for a, b in ((3, 7), (3, 100), (7, 100), (60, 61)):
            assert dm[a, b] == 0.0 and dm[b, a] == 0.0


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("metric", [2, 3, 4])
def test_wsplit_sparse_value_build_is_bitwise_the_dense_build(device_ok, metric, prec, monkeypatch):
    """The sparse value build (presence bit rows + pool values, no dense
    embedding rows) gives the chunked dense build's pool bit for bit, so the
    stripes are identical (SF_WS_DENSE_EMBED=1: the dense build)."""
    for seed, n, leaves, dens in [(91, 200, 700, 0.01), (92, 97, 300, 0.05), (93, 64, 64, 0.3)]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        out = []
        for dense in ("0", "1"):
            monkeypatch.setenv("SF_WS_DENSE_EMBED", dense)
            if metric == 4:
                out.append(_gen13(problem, 0.5, prec, 0, S, monkeypatch, None))
            else:
                out.append(_run(problem, metric, prec, 0, S, monkeypatch, None)[:2])
        monkeypatch.delenv("SF_WS_DENSE_EMBED")
        assert np.array_equal(out[0][0], out[1][0])
        if out[0][1] is not None:
            assert np.array_equal(out[0][1], out[1][1])
