"""Mantel test on device (sf_mantel; replaces mantel, validate.cpp:111-159).

Pinned to the reference itself: tests/golden/mantel.json is written by
oracle/_ref/ref_driver (the reference built from its sources) — r, r^2 and
p-values of seeded instances (strongly correlated pairs with p at its floor,
and independent pairs with p in the bulk) and the first permutations of its
stream. The distance matrices fed to the GPU are the oracle's (bit-identical
to the reference's, tests/test_oracle.py).
"""
import numpy as np
import pytest

import golden_util as gu
import oracle_port as op
from paper_2005_05826_b200 import _native as N
from paper_2005_05826_b200 import stripefrac as sf

GOLD = gu.load("mantel.json")


def test_permutation_stream_is_the_references():
    """Host-only: mt19937_64 + std::shuffle seeded from splitmix64 (validate.cpp:133-136)."""
    for e in GOLD["permutations"]:
        assert np.array_equal(sf.mantel_permutation(e["n"], e["seed"], e["p"]), e["perm"])


def test_mantel_argument_errors_without_device():
    with pytest.raises(sf.Error, match="at least 1 permutation"):
        sf.mantel(sf.DistanceMatrix(["a", "b"], np.zeros((2, 2))),
                  sf.DistanceMatrix(["a", "b"], np.zeros((2, 2))), 0)
    with pytest.raises(sf.Error, match="different sizes"):
        sf.mantel(sf.DistanceMatrix(["a", "b"], np.zeros((2, 2))),
                  sf.DistanceMatrix(["a", "b", "c"], np.zeros((3, 3))))
    with pytest.raises(sf.Error, match="sample orderings"):
        sf.mantel(sf.DistanceMatrix(["a", "b"], np.zeros((2, 2))),
                  sf.DistanceMatrix(["b", "a"], np.zeros((2, 2))))


_DM_CACHE = {}


def _dm(seed, n, leaves, dens, which):
    key = (seed, n, leaves, dens, which)
    if key not in _DM_CACHE:
        s = seed + 100 if which.endswith("-other") else seed
        inst = sf.random_instance(s, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        metric = 1 if which.startswith("unweighted") else 3
        prec = 4 if "fp32" in which else 8
        d, _ = op.compute_stripes(problem, metric, prec)
        _DM_CACHE[key] = op.condense(prec, n, d)
    return _DM_CACHE[key]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["cases"],
                         ids=lambda c: f"n{c['n']}-{c['y']}-{c['permutations']}")
def test_mantel_matches_reference(case):
    assert N.lib().sf_device_count() >= 1
    n = case["n"]
    ids = [f"s{i}" for i in range(n)]
    x = sf.DistanceMatrix(ids, _dm(case["seed"], n, case["leaves"], case["density"], case["x"]))
    y = sf.DistanceMatrix(ids, _dm(case["seed"], n, case["leaves"], case["density"], case["y"]))
    res = sf.mantel(x, y, case["permutations"], case["mantel_seed"])
    # same terms, different summation order: r within 1e-12; same permutations: same p
    assert abs(res.r - case["r"]) <= 1e-12 * abs(case["r"]) + 1e-15
    assert res.p_value == case["p_value"]
    assert res.permutations == case["permutations"]


@pytest.mark.gpu
def test_mantel_errors_on_device():
    n = 6
    ids = [f"s{i}" for i in range(n)]
    a = np.random.default_rng(1).random((n, n))
    sym = (a + a.T) / 2
    np.fill_diagonal(sym, 0)
    asym = sym.copy()
    asym[1, 4] += 1e-6
    with pytest.raises(sf.Error, match=r"asymmetric at \(1,4\)"):
        sf.mantel(sf.DistanceMatrix(ids, sym), sf.DistanceMatrix(ids, asym), 9)
    const = np.ones((n, n))
    np.fill_diagonal(const, 0)
    with pytest.raises(sf.Error, match="zero variance"):
        sf.mantel(sf.DistanceMatrix(ids, sym), sf.DistanceMatrix(ids, const), 9)


@pytest.mark.gpu
def test_mantel_identity_relabeling_counts_as_exceed():
    """n = 2 has one pair: every permutation gives r_perm == r exactly (the
    cross term is reduced like the observed one), so p = 1, as in the reference."""
    ids = ["a", "b"]
    x = sf.DistanceMatrix(ids, np.array([[0, 1.0], [1.0, 0]]))
    # a 2x2 matrix has zero variance: the reference raises; use n = 3
    with pytest.raises(sf.Error, match="zero variance"):
        sf.mantel(x, x, 5)
    ids = ["a", "b", "c"]
    m = np.array([[0, 1.0, 2.0], [1.0, 0, 4.0], [2.0, 4.0, 0]])
    res = sf.mantel(sf.DistanceMatrix(ids, m), sf.DistanceMatrix(ids, m), 50, 3)
    perms = [sf.mantel_permutation(3, 3, p) for p in range(50)]
    iu = np.triu_indices(3, 1)
    x = m[iu]
    r_obs = 1.0
    exceed = 0
    for pm in perms:
        yp = m[pm[iu[0]], pm[iu[1]]]
        r = np.corrcoef(x, yp)[0, 1]
        exceed += r >= r_obs - 1e-12
    assert abs(res.r - 1.0) <= 1e-15
    assert res.p_value == (1.0 + exceed) / 51.0
