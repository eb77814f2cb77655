"""GPU parity: the sm_100a path through the C ABI vs the reference's golden
vectors (tests/golden, produced by the reference itself) and vs the CPU
oracle restatement (tests/oracle_port.py) on larger seeded instances.

Tolerances (BASELINE.json north_star, test_kernels.cpp:187-202):
  * unweighted, walk kernels (dense, sparse walk 2, the default under exact
    mode): bit-exact (0/1 products are exact, so FMA and mul+add round
    identically and the per-slot postorder sum is the same);
  * unweighted, split kernel (10, the default): the correctly rounded exact
    sums for any double lengths; fp64 within 1e-12 relative of the
    reference's sequential sums (and bitwise equal to the exact rational sums,
    test_split_is_exact), fp32 within max(1e-5 |x|, 1e-6);
  * weighted fp64 with FMA: |got - want| <= 1e-12 * |want| (relative; exact zeros exact);
  * weighted fp32 with FMA: <= max(1e-5 |want|, 1e-6);
  * weighted, exact (no-FMA) mode: bit-exact in both precisions.
"""
import ctypes as C

import numpy as np
import pytest

import golden_util as gu
import oracle_port as op
from paper_2005_05826_b200 import _native as N
from paper_2005_05826_b200 import stripefrac as sf

pytestmark = pytest.mark.gpu

KERNELS = [N.KERNEL_DENSE, N.KERNEL_SPARSE, N.KERNEL_SPLIT, N.KERNEL_WSPARSE, N.KERNEL_WUWALK]
WALKS = (N.KERNEL_DENSE, N.KERNEL_SPARSE)


def _kernel_serves(kernel, metric):
    """Dense serves every metric; 2-10 are unweighted-only, 11 weighted-only."""
    if kernel == N.KERNEL_DENSE or kernel == N.KERNEL_AUTO:
        return True
    return (metric != 1) if kernel in (N.KERNEL_WSPARSE, N.KERNEL_WUWALK) else (metric == 1)


def _gpu_stripes(problem, metric, prec, start, stop, kernel=N.KERNEL_DENSE, exact=False,
                 finalize=True, mem_budget=0):
    n = problem.n_samples
    dt = np.float64 if prec == 8 else np.float32
    d = np.full((stop - start, n), np.nan, dt)
    t = np.full((stop - start, n), np.nan, dt)
    ex, _keep = N.make_exec([0], kernel, exact, mem_budget)
    st = N.sf_stats()
    N.check(N.lib().sf_compute_stripes(problem.ref, metric, prec, start, stop, N.ptr(d),
                                       N.ptr(t) if metric != 2 else None, int(finalize),
                                       C.byref(ex), C.byref(st)))
    return d, (t if metric != 2 else None), st


def _assert_close(metric, prec, exact, got, want, kernel=N.KERNEL_DENSE):
    bitwise = exact or (metric == 1 and kernel in WALKS)
    if bitwise:
        assert np.array_equal(got, want), f"max |diff| {np.nanmax(np.abs(got - want))}"
    elif metric == 1 and prec == 8:
        # exact fixed-point sums vs the reference's sequential sums: relative
        err = np.abs(got - want)
        assert np.all(err <= 1e-12 * np.abs(want)), f"max rel {np.max(err / np.maximum(np.abs(want), 1e-300))}"
    elif prec == 8:
        # weighted fp64: 1e-12 RELATIVE (north star); an exact zero of the
        # reference (identical samples, t = 0) must be an exact zero here
        err = np.abs(got - want)
        assert np.all(err <= 1e-12 * np.abs(want)), \
            f"max rel {np.max(err / np.maximum(np.abs(want), 1e-300))}, zeros missed {int(np.sum((want == 0) & (got != 0)))}"
    else:
        w = want.astype(np.float64)
        tol = np.maximum(1e-5 * np.abs(w), 1e-6)
        assert np.all(np.abs(got.astype(np.float64) - w) <= tol)


CASES = gu.all_cases()


@pytest.fixture(scope="module")
def device_ok():
    assert N.lib().sf_device_count() >= 1, "no sm_100 device visible (GPU tests need a B200)"


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
@pytest.mark.parametrize("kernel", KERNELS)
def test_golden_stripes(device_ok, case, kernel):
    tree, table = gu.case_inputs(case)
    problem = sf.flatten(tree, table)
    n = table.n_samples()
    for r in case["results"]:
        metric = int(sf.metric_from_name(r["metric"]))
        if not _kernel_serves(kernel, metric):
            continue
        prec = 8 if r["precision"] == "fp64" else 4
        gd, gt = gu.stripes(r, n)
        # kernel 12 has no bitwise mode (exact mode selects kernel 11 under auto)
        for exact in ((False, True) if metric != 1 and kernel != N.KERNEL_WUWALK else (False,)):
            d, t, _ = _gpu_stripes(problem, metric, prec, r["start"], r["stop"], kernel, exact)
            _assert_close(metric, prec, exact, d, gd, kernel)
            if gt is not None:
                _assert_close(metric, prec, exact, t, gt, kernel)


@pytest.mark.parametrize("case", [c for c in CASES if "embedding_weighted" in c],
                         ids=lambda c: c["name"])
def test_golden_embedding_rows(device_ok, case):
    """K1 rows are bit-identical to Embedder::next_batch (embed.cpp:42-82)."""
    tree, table = gu.case_inputs(case)
    problem = sf.flatten(tree, table)
    n = table.n_samples()
    for weighted, key in ((1, "embedding_weighted"), (0, "embedding_unweighted")):
        want = np.array(case[key], dtype=np.float64)
        pad = n + 3
        out = np.full((problem.n_rows, pad), np.nan)
        N.check(N.lib().sf_embed_rows(problem.ref, weighted, 0, problem.n_rows, N.ptr(out), pad, 0))
        assert np.array_equal(out[:, :n], want)
        assert np.all(out[:, n:] == 0.0)


def test_demo_condense_and_tsv_bytes(device_ok):
    """C1: full DM through condense on device, TSV bytes identical (test_cli.cpp:108-139)."""
    case = gu.load("demo.json")
    tree, table = gu.case_inputs(case)
    for entry in case["dm"]:
        m = sf.metric_from_name(entry["metric"])
        p = sf.precision_from_name(entry["precision"])
        cfg = sf.KernelConfig(metric=m, precision=p)
        for exact in (False, True):
            dm = sf.compute_distance_matrix(tree, table, cfg,
                                            exec_options=sf.ExecOptions(exact=exact))
            want = np.array(entry["values"]).reshape(dm.n(), dm.n())
            if exact:
                assert np.array_equal(dm.values, want)
                assert sf.to_tsv(dm) == entry["tsv"]
            elif m == sf.Metric.Unweighted:
                tol = 1e-12 if p == sf.Precision.Fp64 else 1e-5
                assert np.allclose(dm.values, want, rtol=tol, atol=0 if p == sf.Precision.Fp64 else 1e-6)
            else:
                assert np.allclose(dm.values, want, rtol=1e-12 if p == sf.Precision.Fp64 else 1e-5,
                                   atol=0 if p == sf.Precision.Fp64 else 1e-6)


def test_hand_worked_values(device_ok):
    """test_kernels.cpp:49-78: two disjoint leaves give 2.0 / 1.0 / 1.0 exactly."""
    t = sf.parse_newick("(A:1,B:1);")
    table = sf.make_table(["s1", "s2"], ["A", "B"], [[4, 0], [0, 4]])
    for v in sf.Variant:
        wu = sf.compute_distance_matrix(t, table, sf.KernelConfig(sf.Metric.WeightedUnnormalized, v))
        assert wu.values[0, 1] == 2.0
        wn = sf.compute_distance_matrix(t, table, sf.KernelConfig(sf.Metric.WeightedNormalized, v))
        assert wn.values[0, 1] == 1.0
        uw = sf.compute_distance_matrix(t, table, sf.KernelConfig(sf.Metric.Unweighted, v))
        assert uw.values[0, 1] == 1.0
        assert wu.values[0, 0] == 0.0 and wu.values[1, 0] == wu.values[0, 1]
    t3 = sf.parse_newick("((A:1,B:1):1,C:1);")
    tb3 = sf.make_table(["s1", "s2"], ["A", "B", "C"], [[1, 0], [0, 1], [0, 0]])
    uw = sf.compute_distance_matrix(t3, tb3, sf.KernelConfig(sf.Metric.Unweighted))
    assert abs(uw.values[0, 1] - 2.0 / 3.0) <= 1e-12


@pytest.mark.parametrize("metric", [1, 2, 3])
@pytest.mark.parametrize("prec", [8, 4])
def test_oracle_random_instances(device_ok, metric, prec):
    """Seeded instances beyond the fixtures (several CTA tiles, wrap, tails),
    checked against the pinned CPU restatement."""
    for seed, n, leaves, dens, subset in [(11, 67, 150, 0.05, 0), (12, 130, 400, 0.02, 300),
                                          (13, 257, 600, 0.01, 0), (14, 2, 5, 0.5, 0),
                                          (15, 3, 2, 0.9, 0), (16, 300, 90, 0.2, 0)]:
        inst = sf.random_instance(seed, n, leaves, dens, subset)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        for start, stop in [(0, S), (S // 3, S)]:
            if start >= stop:
                continue
            wd, wt = op.compute_stripes(problem, metric, prec, start, stop)
            for exact in (False, True):
                for kernel in (N.KERNEL_DENSE, N.KERNEL_AUTO):
                    d, t, st = _gpu_stripes(problem, metric, prec, start, stop, kernel, exact)
                    used = kernel if kernel != N.KERNEL_AUTO else (
                        (N.KERNEL_WSPARSE if exact else N.KERNEL_WUWALK) if metric != 1 else
                        N.KERNEL_SPARSE if exact else N.KERNEL_SPLIT)
                    _assert_close(metric, prec, exact, d, wd, used)
                    if wt is not None:
                        _assert_close(metric, prec, exact, t, wt, used)
                    assert st.updates_alg == problem.n_rows * (stop - start) * n


def test_chunked_embedding_with_pending_rows(device_ok):
    """A tiny device budget forces many postorder chunks and pending slots;
    results must stay bitwise identical (batch boundaries never change bits)."""
    inst = sf.random_instance(21, 96, 500, 0.05)
    problem = sf.flatten(inst.tree, inst.table)
    for metric in (1, 3):
        full, fullt, st1 = _gpu_stripes(problem, metric, 8, 0, 48, exact=True)
        row_bytes = 4 * 3 if metric == 1 else 8 * 96
        small, smallt, st2 = _gpu_stripes(problem, metric, 8, 0, 48, exact=True,
                                          mem_budget=row_bytes * 37)
        assert st2.n_chunks > 5
        assert np.array_equal(full, small)
        assert np.array_equal(fullt, smallt)


def test_partition_independence_bitwise(device_ok):
    """test_kernels.cpp:154-170 / acceptance.cpp:237-280: any tiling of [0,S)
    condenses to the full-range result bit for bit."""
    inst = sf.random_instance(1234, 17, 40, 0.4)
    cfg = sf.KernelConfig(sf.Metric.WeightedNormalized, sf.Variant.Tiled)
    full = sf.compute_distance_matrix(inst.tree, inst.table, cfg)
    for ranges in ([(0, 8)], [(0, 4), (4, 8)], [(0, 1), (1, 2), (2, 5), (5, 8)]):
        parts = [sf.compute_unifrac(inst.tree, inst.table, cfg, a, b) for a, b in ranges]
        merged = sf.condense(parts, inst.table.sample_ids)
        assert np.array_equal(merged.values, full.values)


def test_batch_api_matches_full_run(device_ok):
    """Embedder + accumulate + finalize (kernels.hpp:232-259) == compute_unifrac."""
    inst = sf.random_instance(777, 23, 48, 0.4)
    for m in (sf.Metric.Unweighted, sf.Metric.WeightedUnnormalized, sf.Metric.WeightedNormalized):
        cfg = sf.KernelConfig(m, sf.Variant.Tiled)
        want = sf.compute_unifrac(inst.tree, inst.table, cfg)
        sh = sf.sheared_to_table(inst.tree, inst.table)
        em = sf.Embedder(sh, inst.table, sf.embed_mode(m), cfg.resolved_step_size())
        sset = sf.allocate_stripes(23, 0, 11, m)
        c = sf.KernelCounters()
        while (b := em.next_batch(5)) is not None:
            sf.accumulate(sset, b, cfg, c)
        sf.finalize(sset)
        assert np.allclose(sset.distances, want.distances, rtol=1e-12, atol=0)
        E = em.total_rows()
        assert c.kernel_passes == -(-E // 5)
        assert c.embedding_reads == 2 * E * 11 * 23


def test_counter_law(device_ok):
    """test_kernels.cpp:123-152: writes = E (naive) or ceil(E/B) per entry."""
    inst = sf.random_instance(31337, 20, 32, 0.4)
    E = 2 * 32 - 2
    c = sf.KernelCounters()
    sf.compute_unifrac(inst.tree, inst.table,
                       sf.KernelConfig(sf.Metric.WeightedUnnormalized, sf.Variant.Batched,
                                       sf.Precision.Fp64, 16), 3, 7, 1, c)
    entries = 4 * 20
    passes = (E + 15) // 16
    assert c.accumulator_writes == passes * entries
    assert c.embedding_reads == 2 * E * entries
    assert c.kernel_passes == passes


def test_misuse_is_rejected(device_ok):
    """test_kernels.cpp:219-264."""
    t = sf.parse_newick("(A:1,B:1);")
    table = sf.make_table(["s1", "s2"], ["A", "B"], [[4, 1], [1, 4]])
    with pytest.raises(sf.Error):
        sf.compute_unifrac(t, table, sf.KernelConfig(sf.Metric.Unweighted), real=np.float32)
    with pytest.raises(sf.Error):
        sf.compute_unifrac(t, table, sf.KernelConfig(sf.Metric.Unweighted, batch_capacity=0))
    with pytest.raises(sf.Error, match="does not fit"):
        sf.compute_unifrac(t, table, sf.KernelConfig(sf.Metric.Unweighted), 0, 2)
    em = sf.Embedder(t, table, sf.EmbedMode.Weighted, 16)
    batch = em.next_batch(64)
    sset = sf.allocate_stripes(2, 0, 1, sf.Metric.WeightedUnnormalized)
    cfg = sf.KernelConfig(sf.Metric.WeightedUnnormalized)
    c = sf.KernelCounters()
    sf.accumulate(sset, batch, cfg, c)
    sf.finalize(sset)
    with pytest.raises(sf.Error):
        sf.accumulate(sset, batch, cfg, c)
    with pytest.raises(sf.Error):
        sf.finalize(sset)
    s2 = sf.allocate_stripes(2, 0, 1, sf.Metric.WeightedUnnormalized)
    with pytest.raises(sf.Error):
        sf.accumulate(s2, sf.EmbeddingBatch(np.zeros((0, 16)), np.zeros(0), 0, 2, 16), cfg, c)
    with pytest.raises(sf.Error):
        sf.accumulate(s2, batch, sf.KernelConfig(sf.Metric.Unweighted), c)
    em2 = sf.Embedder(t, table, sf.EmbedMode.Weighted, 1)
    with pytest.raises(sf.Error):
        sf.accumulate(s2, em2.next_batch(64), cfg, c)


def test_fp32_mantel_against_fp64(device_ok):
    """acceptance.cpp:282-309: fp32 vs fp64, r^2 >= 0.9999, p <= 0.001, drift <= 1e-5."""
    inst = sf.random_instance(60464, 64, 512, 0.3)
    for m in sf.Metric:
        d64 = sf.compute_distance_matrix(inst.tree, inst.table, sf.KernelConfig(m))
        d32 = sf.compute_distance_matrix(inst.tree, inst.table,
                                         sf.KernelConfig(m, precision=sf.Precision.Fp32, step_size=32))
        res = sf.mantel(d64, d32, 999, 4)
        assert res["r_squared"] >= 0.9999 and res["p_value"] <= 0.001
        iu = np.triu_indices(64, 1)
        drift = np.abs(d32.values[iu] - d64.values[iu]) / np.maximum(np.abs(d64.values[iu]), 0.1)
        assert drift.max() <= 1e-5


@pytest.mark.parametrize("prec", [8, 4])
def test_sparse_kernel_matches_dense_bitwise(device_ok, prec):
    """Both unweighted kernels apply the same adds in the same order."""
    for seed, n, leaves, dens, subset in [(41, 200, 800, 0.01, 0), (42, 333, 1500, 0.004, 1000),
                                          (43, 64, 3000, 0.02, 0), (44, 9, 70, 0.3, 0)]:
        inst = sf.random_instance(seed, n, leaves, dens, subset)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        for start, stop in [(0, S), (S // 2, S)]:
            d1, t1, _ = _gpu_stripes(problem, 1, prec, start, stop, kernel=N.KERNEL_DENSE)
            wd, wt = op.compute_stripes(problem, 1, prec, start, stop)
            d2, t2, st = _gpu_stripes(problem, 1, prec, start, stop, kernel=N.KERNEL_SPARSE)
            assert np.array_equal(d1, d2) and np.array_equal(t1, t2)
            assert np.array_equal(d2, wd) and np.array_equal(t2, wt)
            assert 0 < st.updates_exec <= st.updates_alg


def test_isect_is_the_default_for_unweighted(device_ok):
    inst = sf.random_instance(45, 50, 100, 0.1)
    problem = sf.flatten(inst.tree, inst.table)
    d5, t5, st = _gpu_stripes(problem, 1, 8, 0, 25, kernel=N.KERNEL_SPLIT)
    d0, t0, st0 = _gpu_stripes(problem, 1, 8, 0, 25, kernel=N.KERNEL_AUTO)
    assert np.array_equal(d5, d0) and np.array_equal(t5, t0)
    # the split kernel touches far fewer (row, slot) pairs than the reference
    assert 0 < st0.updates_exec < st0.updates_alg
    _, _, st2 = _gpu_stripes(problem, 1, 8, 0, 25, kernel=N.KERNEL_AUTO, exact=True)
    assert 0 < st2.updates_exec < st2.updates_alg  # exact mode: the union walk


def _round_fraction(x, dt):
    """x (a non-negative Fraction) correctly rounded to dt (ties to even)."""
    from fractions import Fraction
    f = float(x)  # correctly rounded to fp64
    if dt == np.float64:
        return np.float64(f)
    c = np.float32(f)
    best = None
    for cand in (np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))):
        if not np.isfinite(cand) or cand < 0:
            continue
        err = abs(Fraction(float(cand)) - x)
        key = (err, int(np.float32(cand).view(np.uint32)) & 1)
        if best is None or key < best[0]:
            best = (key, cand)
    return np.float32(best[1])


def _exact_stripes(problem, prec, start, stop):
    """t and d of every slot as exact rationals (Fraction), rounded once:
    the value a correctly rounded unweighted kernel must return."""
    from fractions import Fraction
    n, E = problem.n_samples, problem.n_rows
    pres = np.zeros((E, n), bool)
    fp, si = problem.feat_ptr, problem.sample_idx
    for r in range(E):
        f = problem.leaf_feature[r]
        if f >= 0:
            pres[r, si[fp[f]:fp[f + 1]]] = True
    for r in range(E):
        q = problem.parent_row[r]
        if q >= 0:
            pres[q] |= pres[r]
    L = problem.lengths if prec == 8 else problem.lengths.astype(np.float32).astype(np.float64)
    Lf = [Fraction(float(x)) for x in L]
    dt = np.float64 if prec == 8 else np.float32
    d = np.zeros((stop - start, n), dt)
    t = np.zeros((stop - start, n), dt)
    for s in range(start, stop):
        for k in range(n):
            l = (k + s + 1) % n
            u, v = pres[:, k], pres[:, l]
            tt = sum((Lf[e] for e in np.nonzero(u | v)[0]), Fraction(0))
            dd = sum((Lf[e] for e in np.nonzero(u ^ v)[0]), Fraction(0))
            t[s - start, k] = _round_fraction(tt, dt)
            d[s - start, k] = _round_fraction(dd, dt)
    return d, t


@pytest.mark.parametrize("prec", [8, 4])
def test_split_is_exact(device_ok, prec, kernel=N.KERNEL_SPLIT):
    """The split kernel returns the correctly rounded exact sums (raw,
    unfinalized), on instances with sparse and dense (complemented) rows,
    wrap, odd/even n and partial ranges."""
    for seed, n, leaves, dens in [(51, 40, 60, 0.05), (52, 33, 50, 0.6), (53, 2, 4, 0.5),
                                  (54, 3, 7, 0.9), (55, 70, 40, 0.3)]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        for start, stop in [(0, S), (S // 2, S)]:
            if start >= stop:
                continue
            wd, wt = _exact_stripes(problem, prec, start, stop)
            d, t, _ = _gpu_stripes(problem, 1, prec, start, stop, kernel, finalize=False)
            assert np.array_equal(d, wd) and np.array_equal(t, wt)


@pytest.mark.parametrize("heavy_frac", ["0.6", "0.0", "0.05"])
@pytest.mark.parametrize("prec", [8, 4])
def test_split_heavy_light_boundary_is_exact(device_ok, prec, heavy_frac, monkeypatch):
    """Kernel 10 with every row light (scatter only), every row heavy (walk
    only) and a mixed split: always the correctly rounded exact sums."""
    monkeypatch.setenv("SF_HEAVY_FRAC", heavy_frac)
    for seed, n, leaves, dens in [(71, 40, 60, 0.05), (72, 33, 50, 0.6), (73, 64, 90, 0.2)]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        for start, stop in [(0, S), (S // 2, S)]:
            wd, wt = _exact_stripes(problem, prec, start, stop)
            d, t, st = _gpu_stripes(problem, 1, prec, start, stop, N.KERNEL_SPLIT, finalize=False)
            assert np.array_equal(d, wd) and np.array_equal(t, wt)


@pytest.mark.parametrize("heavy_frac", ["0.6", "0.0", "0.05"])
@pytest.mark.parametrize("log10_min", [-9, -14, -40, -300])
@pytest.mark.parametrize("prec", [8, 4])
def test_split_exact_for_any_double_lengths(device_ok, prec, log10_min, heavy_frac, monkeypatch):
    """Branch lengths spanning many binades (log-uniform in [10^lo, 2]):
    lengths off the main fixed-point grid take deeper levels, and the result
    is still the correctly rounded exact rational sum — with all rows light,
    all heavy, and mixed; even and odd n, wrap and partial ranges."""
    monkeypatch.setenv("SF_HEAVY_FRAC", heavy_frac)
    rng = np.random.default_rng(abs(log10_min) * 31 + len(heavy_frac))
    for seed, n, leaves, dens in [(75, 40, 60, 0.1), (76, 33, 50, 0.6)]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        problem.lengths[:] = 10.0 ** rng.uniform(log10_min, np.log10(2.0), problem.n_rows)
        S = n // 2
        for start, stop in [(0, S), (S // 2, S)]:
            wd, wt = _exact_stripes(problem, prec, start, stop)
            d, t, _ = _gpu_stripes(problem, 1, prec, start, stop, N.KERNEL_SPLIT, finalize=False)
            assert np.array_equal(d, wd) and np.array_equal(t, wt)


@pytest.mark.parametrize("prec", [8, 4])
def test_split_matches_oracle_larger(device_ok, prec, kernel=N.KERNEL_SPLIT):
    """The split kernel vs the CPU restatement of the reference (sequential sums) on
    instances spanning several CTA tiles and 1024-row groups."""
    for seed, n, leaves, dens, subset in [(61, 300, 1500, 0.01, 0), (62, 517, 2500, 0.004, 2000),
                                          (63, 129, 700, 0.2, 0), (64, 1000, 3000, 0.002, 0)]:
        inst = sf.random_instance(seed, n, leaves, dens, subset)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        for start, stop in [(0, S), (S // 3, S - 1)]:
            wd, wt = op.compute_stripes(problem, 1, prec, start, stop)
            d, t, st = _gpu_stripes(problem, 1, prec, start, stop, kernel)
            _assert_close(1, prec, False, d, wd, kernel)
            _assert_close(1, prec, False, t, wt, kernel)
            assert st.updates_alg == problem.n_rows * (stop - start) * n


@pytest.mark.parametrize("kernel", [N.KERNEL_AUTO, N.KERNEL_DENSE, N.KERNEL_SPARSE])
def test_stripe_shards_match_single_device(device_ok, kernel):
    """The in-process multi-device fan-out (sf_exec.devices, the reference's
    worker split kernels.hpp:302-303) with two or three shards placed on the
    same B200: every shard builds its own embedding and writes its own stripe
    block; the result equals the one-shard run bit for bit."""
    inst = sf.random_instance(91, 300, 900, 0.01)
    problem = sf.flatten(inst.tree, inst.table)
    n = problem.n_samples
    for metric in ((1, 3) if kernel == N.KERNEL_DENSE else (1,)):
        for start, stop in [(0, n // 2), (17, 140)]:
            d1, t1, _ = _gpu_stripes(problem, metric, 8, start, stop, kernel)
            for devs in ([0, 0], [0, 0, 0]):
                d = np.full((stop - start, n), np.nan)
                t = np.full((stop - start, n), np.nan)
                ex, _keep = N.make_exec(devs, kernel)
                st = N.sf_stats()
                N.check(N.lib().sf_compute_stripes(problem.ref, metric, 8, start, stop, N.ptr(d), N.ptr(t),
                                                   1, C.byref(ex), C.byref(st)))
                assert np.array_equal(d, d1) and np.array_equal(t, t1)


@pytest.mark.parametrize("light_pass", ["1", "3", "1000"])
def test_split_light_passes_and_pinned_download(device_ok, light_pass, monkeypatch):
    """Kernel 10 with the light sums built in several stripe passes (as when
    memory is short) and with the chunked, overlapped download into pinned
    host memory: bitwise equal to the single-pass, pageable run."""
    import torch
    inst = sf.random_instance(93, 301, 1200, 0.01)
    problem = sf.flatten(inst.tree, inst.table)
    n = problem.n_samples
    start, stop = 3, n // 2
    want_d, want_t, _ = _gpu_stripes(problem, 1, 8, start, stop, N.KERNEL_SPLIT)
    monkeypatch.setenv("SF_LIGHT_PASS", light_pass)
    monkeypatch.setenv("SF_HEAVY_FRAC", "0.05")
    ref_d, ref_t, _ = _gpu_stripes(problem, 1, 8, start, stop, N.KERNEL_SPLIT)
    assert np.array_equal(ref_d, want_d) and np.array_equal(ref_t, want_t)
    for prec, dt in ((8, torch.float64), (4, torch.float32)):
        d = torch.full(((stop - start) * n,), float("nan"), dtype=dt, pin_memory=True).numpy()
        t = torch.full(((stop - start) * n,), float("nan"), dtype=dt, pin_memory=True).numpy()
        ex, _keep = N.make_exec([0], N.KERNEL_SPLIT)
        st = N.sf_stats()
        N.check(N.lib().sf_compute_stripes(problem.ref, 1, prec, start, stop, N.ptr(d), N.ptr(t), 1,
                                           C.byref(ex), C.byref(st)))
        pd, pt, _ = _gpu_stripes(problem, 1, prec, start, stop, N.KERNEL_SPLIT)
        assert np.array_equal(d.reshape(stop - start, n), pd)
        assert np.array_equal(t.reshape(stop - start, n), pt)


def test_pageable_download_staged_matches_pinned(device_ok):
    """Pageable destinations are staged through a pinned double buffer
    (128 MB blocks, host threads copying out) chunk by chunk while the split
    kernel computes later chunks: bitwise equal to the pinned, overlapped
    download. n = 17,000 gives 4 chunks of ~290 MB (3 staging blocks each);
    the weighted metric takes the download-after-compute path."""
    import torch
    inst = sf.random_instance(97, 17000, 300, 0.01)
    problem = sf.flatten(inst.tree, inst.table)
    n = problem.n_samples
    start, stop = 0, n // 2
    for metric, kernel in ((1, N.KERNEL_SPLIT), (3, 0)):
        pd = torch.full(((stop - start) * n,), float("nan"), dtype=torch.float64, pin_memory=True).numpy()
        pt = torch.full(((stop - start) * n,), float("nan"), dtype=torch.float64, pin_memory=True).numpy()
        ex, _keep = N.make_exec([0], kernel)
        st = N.sf_stats()
        N.check(N.lib().sf_compute_stripes(problem.ref, metric, 8, start, stop, N.ptr(pd), N.ptr(pt), 1,
                                           C.byref(ex), C.byref(st)))
        d, t, _ = _gpu_stripes(problem, metric, 8, start, stop, kernel)
        assert not np.isnan(d).any() and not np.isnan(t).any()
        assert np.array_equal(d, pd.reshape(stop - start, n))
        assert np.array_equal(t, pt.reshape(stop - start, n))
        del pd, pt, d, t


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("metric", [2, 3])
def test_weighted_sparse_walk_matches_dense_bitwise(device_ok, metric, prec):
    """Kernel 11 (the weighted default) skips rows absent from both samples —
    they add exactly +0.0 — and applies the reference's update to the rest in
    postorder: bit for bit the dense kernel in exact mode, also across
    chunked embeddings (pool per chunk), partial and wrapped stripe ranges."""
    for seed, n, leaves, dens in [(31, 200, 700, 0.01), (32, 97, 300, 0.05), (33, 64, 64, 0.3)]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        for start, stop in [(0, S), (S // 2, S), (3, 4)]:
            d1, t1, s1 = _gpu_stripes(problem, metric, prec, start, stop, N.KERNEL_DENSE, exact=True)
            d2, t2, s2 = _gpu_stripes(problem, metric, prec, start, stop, N.KERNEL_WSPARSE, exact=True)
            assert np.array_equal(d1, d2)
            if t1 is not None:
                assert np.array_equal(t1, t2)
            assert s2.updates_exec < s2.updates_alg
        # a budget of ~40 rows: 32-row chunks, pending slots, per-chunk pools
        d3, t3, s3 = _gpu_stripes(problem, metric, prec, 0, S, N.KERNEL_WSPARSE, exact=True,
                                  mem_budget=40 * 8 * (n + 1) * 2)
        d1, t1, _ = _gpu_stripes(problem, metric, prec, 0, S, N.KERNEL_DENSE, exact=True)
        assert s3.n_chunks > 1
        assert np.array_equal(d1, d3)
        if t1 is not None:
            assert np.array_equal(t1, t3)
        # FMA form: within the stated tolerance of the oracle
        wd, wt = op.compute_stripes(problem, metric, prec, 0, S)
        d4, t4, _ = _gpu_stripes(problem, metric, prec, 0, S, N.KERNEL_WSPARSE)
        _assert_close(metric, prec, False, d4, wd, N.KERNEL_WSPARSE)
        if wt is not None:
            _assert_close(metric, prec, False, t4, wt, N.KERNEL_WSPARSE)


def test_weighted_sparse_rejects_unweighted(device_ok):
    inst = sf.random_instance(3, 10, 12, 0.3)
    problem = sf.flatten(inst.tree, inst.table)
    with pytest.raises(N.NativeError, match="weighted metrics only"):
        _gpu_stripes(problem, 1, 8, 0, 5, N.KERNEL_WSPARSE)


def _gpu_generalized(problem, alpha, prec, start, stop, exact=False, mem_budget=0):
    n = problem.n_samples
    dt = np.float64 if prec == 8 else np.float32
    d = np.full((stop - start, n), np.nan, dt)
    t = np.full((stop - start, n), np.nan, dt)
    ex, _keep = N.make_exec([0], N.KERNEL_AUTO, exact, mem_budget, alpha)
    st = N.sf_stats()
    N.check(N.lib().sf_compute_stripes(problem.ref, N.SF_GENERALIZED, prec, start, stop, N.ptr(d),
                                       N.ptr(t), 1, C.byref(ex), C.byref(st)))
    return d, t, st


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("alpha", [0.0, 0.5, 1.0, 1.7])
def test_generalized_matches_oracle(device_ok, alpha, prec):
    """Generalized UniFrac (extension; parity unpinned — the reference has no
    generalized metric): kernel 11 vs the oracle's statement of the published
    form. CUDA pow differs from glibc's by <= 2 ulp, so fp64 is held to 1e-12
    relative (not bitwise, even in exact mode); fp32 to max(1e-5|x|, 1e-6)."""
    for seed, n, leaves, dens in [(51, 150, 500, 0.02), (52, 41, 120, 0.1)]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        for start, stop in [(0, S), (S // 3, S)]:
            wd, wt = op.compute_stripes_generalized(problem, alpha, prec, start, stop)
            for exact in (False, True):
                d, t, _ = _gpu_generalized(problem, alpha, prec, start, stop, exact)
                for got, want in ((d, wd), (t, wt)):
                    if prec == 8:
                        assert np.all(np.abs(got - want) <= 1e-12 * np.abs(want))
                    else:
                        w = want.astype(np.float64)
                        assert np.all(np.abs(got.astype(np.float64) - w) <= np.maximum(1e-5 * np.abs(w), 1e-6))


def test_generalized_alpha1_matches_weighted_normalized(device_ok):
    inst = sf.random_instance(53, 120, 400, 0.03)
    problem = sf.flatten(inst.tree, inst.table)
    S = 60
    gd, gt, _ = _gpu_generalized(problem, 1.0, 8, 0, S)
    wd, wt, _ = _gpu_stripes(problem, 3, 8, 0, S)
    assert np.allclose(gd, wd, rtol=1e-12, atol=0)
    assert np.allclose(gt, wt, rtol=1e-12, atol=0)


def test_generalized_rejects_bad_alpha_and_dense(device_ok):
    inst = sf.random_instance(54, 10, 12, 0.3)
    problem = sf.flatten(inst.tree, inst.table)
    with pytest.raises(N.NativeError, match="alpha"):
        _gpu_generalized(problem, -1.0, 8, 0, 5)
    with pytest.raises(N.NativeError, match="alpha"):
        _gpu_generalized(problem, float("nan"), 8, 0, 5)
    ex, _keep = N.make_exec([0], N.KERNEL_DENSE, False, 0, 0.5)
    d = np.zeros((5, 10))
    with pytest.raises(N.NativeError, match="weighted kernels"):
        N.check(N.lib().sf_compute_stripes(problem.ref, N.SF_GENERALIZED, 8, 0, 5, N.ptr(d), N.ptr(d),
                                           1, C.byref(ex), None))


def test_generalized_python_mirror(device_ok):
    inst = sf.random_instance(55, 30, 70, 0.1)
    cfg = sf.KernelConfig(sf.Metric.Generalized, alpha=0.5)
    dm = sf.compute_distance_matrix(inst.tree, inst.table, cfg)
    problem = sf.flatten(inst.tree, inst.table)
    wd, _ = op.compute_stripes_generalized(problem, 0.5, 8)
    want = op.condense(8, 30, wd)
    assert np.allclose(dm.values, want, rtol=1e-12, atol=0)


@pytest.mark.parametrize("band_mb,light_pass", [("0.05", "0"), ("0.3", "7"), ("1000", "0")])
def test_split_banded_light_scatter_is_bitwise_the_one_shot_scatter(device_ok, band_mb, light_pass,
                                                                    monkeypatch):
    """The column-owned light scatter (shared-memory windows per column, the
    default) and the banded one (member CSR + per-band partners, atomics into
    an L2-sized block) add exactly the same limbs to exactly the same slots
    as the one-shot scatter: integer atomics are order-free, so the results
    are bit-identical — for tiny bands, multi-pass light sums, even n
    (duplicated half stripe), wrapped and partial ranges."""
    for seed, n, leaves, dens in [(94, 300, 1100, 0.01), (95, 257, 700, 0.03)]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        for start, stop in [(0, n // 2), (5, n // 2 - 3)]:
            monkeypatch.setenv("SF_HEAVY_FRAC", "0.05")
            monkeypatch.setenv("SF_LIGHT_SCATTER", "0")
            want_d, want_t, ws = _gpu_stripes(problem, 1, 8, start, stop, N.KERNEL_SPLIT)
            monkeypatch.delenv("SF_LIGHT_SCATTER")
            monkeypatch.setenv("SF_LIGHT_BAND_MB", band_mb)
            if light_pass != "0":
                monkeypatch.setenv("SF_LIGHT_PASS", light_pass)
            # column-owned (default; three exact limb modes) and banded
            for mode, limbs in (("column", "0"), ("column", "1"), ("column", "2"), ("band", "0")):
                monkeypatch.setenv("SF_LIGHT_MODE", mode)
                monkeypatch.setenv("SF_LIGHT_LIMB_MODE", limbs)
                d, t, gs = _gpu_stripes(problem, 1, 8, start, stop, N.KERNEL_SPLIT)
                assert np.array_equal(d, want_d) and np.array_equal(t, want_t)
                assert gs.updates_exec == ws.updates_exec  # same light pairs counted
            monkeypatch.delenv("SF_LIGHT_MODE")
            monkeypatch.delenv("SF_LIGHT_LIMB_MODE")
            monkeypatch.delenv("SF_LIGHT_BAND_MB")
            monkeypatch.delenv("SF_LIGHT_PASS", raising=False)
            wd, wt = op.compute_stripes(problem, 1, 8, start, stop)
            _assert_close(1, 8, False, d, wd, N.KERNEL_SPLIT)


def _dup_table(inst, dups):
    """The instance's table with sample columns `dups` = {dst: src} copied."""
    t = inst.table
    n, F = t.n_samples(), t.n_features()
    dense = np.zeros((F, n))
    for f in range(F):
        a, b = t.feat_ptr[f], t.feat_ptr[f + 1]
        dense[f, t.sample_idx[a:b]] = t.counts[a:b]
    for dst, src in dups.items():
        dense[:, dst] = dense[:, src]
    return sf.make_table(t.sample_ids, t.feature_ids, dense)


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("metric", [2, 3])
def test_weighted_uwalk_matches_oracle(device_ok, metric, prec):
    """Kernel 12 (the weighted default): u-present rows walked warp-uniformly,
    v-only rows as A_l - B in double-double. Same terms as the reference,
    different summation: fp64 within 1e-12 * |x| (relative), fp32 within
    max(1e-5|x|, 1e-6); chunked embeddings (the pool is filled chunk by
    chunk), partial and wrapped ranges, even and odd n."""
    for seed, n, leaves, dens in [(61, 200, 700, 0.01), (62, 97, 300, 0.05), (63, 64, 64, 0.3),
                                  (64, 301, 1500, 0.004)]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        S = n // 2
        for start, stop in [(0, S), (S // 2, S), (3, 4)]:
            wd, wt = op.compute_stripes(problem, metric, prec, start, stop)
            d, t, st = _gpu_stripes(problem, metric, prec, start, stop, N.KERNEL_WUWALK)
            _assert_close(metric, prec, False, d, wd, N.KERNEL_WUWALK)
            if wt is not None:
                _assert_close(metric, prec, False, t, wt, N.KERNEL_WUWALK)
        d3, t3, s3 = _gpu_stripes(problem, metric, prec, 0, S, N.KERNEL_WUWALK,
                                  mem_budget=40 * 8 * (n + 1) * 2)
        assert s3.n_chunks > 1
        wd, wt = op.compute_stripes(problem, metric, prec, 0, S)
        _assert_close(metric, prec, False, d3, wd, N.KERNEL_WUWALK)


@pytest.mark.parametrize("metric", [2, 3, 4])
def test_weighted_uwalk_identical_samples_are_exactly_zero(device_ok, metric):
    """Duplicated samples: the v-only remainder A_l - B cancels exactly (same
    double-double terms in the same order), so d is exactly 0 like the
    reference's |u - u| = 0 sums; other pairs stay within tolerance."""
    inst = sf.random_instance(65, 120, 400, 0.03)
    table = _dup_table(inst, {7: 3, 100: 3, 61: 60})
    problem = sf.flatten(inst.tree, table)
    n = 120
    S = n // 2
    if metric == 4:
        ex, _keep = N.make_exec([0], N.KERNEL_WUWALK, False, 0, 0.5)
        d = np.zeros((S, n)); t = np.zeros((S, n))
        N.check(N.lib().sf_compute_stripes(problem.ref, 4, 8, 0, S, N.ptr(d), N.ptr(t), 1, C.byref(ex), None))
    else:
        d, t, _ = _gpu_stripes(problem, metric, 8, 0, S, N.KERNEL_WUWALK)
    dm = op.condense(8, n, d)
    for a, b in ((3, 7), (3, 100), (7, 100), (60, 61)):
        assert dm[a, b] == 0.0 and dm[b, a] == 0.0
    if metric != 4:
        wd, _ = op.compute_stripes(problem, metric, 8, 0, S)
        _assert_close(metric, 8, False, d, wd, N.KERNEL_WUWALK)


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("metric", [2, 3, 4])
def test_weighted_uwalk_even_n_duplicate_half_stripe(device_ok, metric, prec):
    """Even n: the last stripe holds each pair twice; condense() requires the
    copies to agree (stripes.cpp:115-122) — bitwise for fp64."""
    inst = sf.random_instance(66, 130, 500, 0.02)
    m = sf.Metric(metric)
    cfg = sf.KernelConfig(m, precision=sf.Precision.Fp64 if prec == 8 else sf.Precision.Fp32,
                          alpha=0.5 if metric == 4 else 1.0)
    part = sf.compute_unifrac(inst.tree, inst.table, cfg, 60, 65)  # last stripe is 64
    last = part.distances[-1]
    assert np.array_equal(last[:65], last[65:])
    dm = sf.compute_distance_matrix(inst.tree, inst.table, cfg)  # condense checks the copies
    assert np.allclose(dm.values, dm.values.T, rtol=0, atol=0)


@pytest.mark.parametrize("metric", [3, 4])
def test_weighted_uwalk_word_list_is_bitwise_the_full_scan(device_ok, metric, monkeypatch):
    """Walking only the nonzero words (per-column masks + L1 prefetch) visits
    the same words in the same order as scanning every word: bit-identical."""
    inst = sf.random_instance(67, 210, 900, 0.01)
    problem = sf.flatten(inst.tree, inst.table)
    S = 105
    out = []
    for lst in ("1", "0"):
        monkeypatch.setenv("SF_UWALK_LIST", lst)
        ex, _keep = N.make_exec([0], N.KERNEL_WUWALK, False, 0, 0.5)
        d = np.zeros((S, 210)); t = np.zeros((S, 210))
        N.check(N.lib().sf_compute_stripes(problem.ref, metric, 8, 0, S, N.ptr(d), N.ptr(t), 1,
                                           C.byref(ex), None))
        out.append((d, t))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_plan_write_strf_matches_reference_files(device_ok, tmp_path):
    """sf_plan_write_strf streams the stripes from device into the .strf
    format byte for byte as the reference's write_stripe_file
    (tests/golden/*.strf written by oracle/_ref; exact mode: the stripes
    themselves are bitwise the reference's)."""
    case = gu.load("demo.json")
    tree, table = gu.case_inputs(case)
    for name, m, p, a, b in (("demo_wn_fp64_0_4", sf.Metric.WeightedNormalized, sf.Precision.Fp64, 0, 4),
                             ("demo_uw_fp32_1_3", sf.Metric.Unweighted, sf.Precision.Fp32, 1, 3),
                             ("demo_wu_fp64_0_4", sf.Metric.WeightedUnnormalized, sf.Precision.Fp64, 0, 4)):
        out = tmp_path / f"{name}.strf"
        sf.compute_unifrac_to_strf(tree, table, sf.KernelConfig(m, precision=p), str(out), a, b,
                                   exec_options=sf.ExecOptions(exact=True))
        want = (gu.GOLDEN / f"{name}.strf").read_bytes()
        assert out.read_bytes() == want


def test_plan_write_strf_equals_host_writer(device_ok, tmp_path):
    """Larger instance, several 64 MB-free chunks aside: same bytes as the host
    writer on the downloaded stripes; refuses unfinalized and generalized."""
    inst = sf.random_instance(71, 700, 2000, 0.01)
    for m in (sf.Metric.Unweighted, sf.Metric.WeightedNormalized):
        cfg = sf.KernelConfig(m)
        p1 = tmp_path / "dev.strf"
        sf.compute_unifrac_to_strf(inst.tree, inst.table, cfg, str(p1), 10, 300)
        part = sf.compute_unifrac(inst.tree, inst.table, cfg, 10, 300)
        p2 = tmp_path / "host.strf"
        sf.write_stripe_file(str(p2), part)
        assert p1.read_bytes() == p2.read_bytes()
    problem = sf.flatten(inst.tree, inst.table)
    ex, _keep = N.make_exec([0])
    plan = C.c_void_p()
    N.check(N.lib().sf_plan_create(problem.ref, 1, 8, 0, 5, C.byref(ex), C.byref(plan)))
    N.check(N.lib().sf_plan_run(plan, 0))
    assert N.lib().sf_plan_write_strf(plan, str(tmp_path / "x.strf").encode()) == N.SF_EINVAL
    assert "unfinalized" in N.lib().sf_last_error().decode()
    N.lib().sf_plan_destroy(plan)
    with pytest.raises(sf.Error, match="no .strf metric code"):
        sf.compute_unifrac_to_strf(inst.tree, inst.table, sf.KernelConfig(sf.Metric.Generalized, alpha=0.5),
                                   str(tmp_path / "g.strf"), 0, 5)


def test_medium_scale_against_oracle(device_ok):
    """A size the oracle finishes in seconds on host threads (n = 1,200,
    E ~ 12k: ~9e9 reference updates per metric): default kernels vs the
    pinned C restatement — UW split (1e-12 relative), WN u-walk and
    generalized (1e-12 relative)."""
    import os
    inst = sf.random_instance(81, 1200, 6000, 0.005)
    problem = sf.flatten(inst.tree, inst.table)
    S = 600
    th = os.cpu_count() or 4
    for metric in (1, 3):
        wd, wt = op.compute_stripes(problem, metric, 8, 0, S, threads=th)
        d, t, _ = _gpu_stripes(problem, metric, 8, 0, S, N.KERNEL_AUTO)
        used = N.KERNEL_SPLIT if metric == 1 else N.KERNEL_WUWALK
        _assert_close(metric, 8, False, d, wd, used)
        _assert_close(metric, 8, False, t, wt, used)
    gd, gt = op.compute_stripes_generalized(problem, 0.5, 8, 0, S, threads=th)
    d, t, _ = _gpu_generalized(problem, 0.5, 8, 0, S)
    assert np.all(np.abs(d - gd) <= 1e-12 * np.abs(gd))
    assert np.all(np.abs(t - gt) <= 1e-12 * np.abs(gt))


def test_split_vs_reference_order_walk_at_4k_samples(device_ok):
    """Size-independent check at a realistic shape (4,000 samples, 40k-tip
    tree, EMP density): the default split kernel (exact fixed-point sums) vs
    the bitwise walk (the reference's adds in the reference's order) — the
    same matrix within 1e-12 relative everywhere; d <= t; 0 <= d/t <= 1."""
    inst = sf.random_instance(7, 4000, 40000, 0.002)
    problem = sf.flatten(inst.tree, inst.table)
    S = 2000
    d0, t0, _ = _gpu_stripes(problem, 1, 8, 0, S, N.KERNEL_SPARSE, finalize=False)
    d1, t1, _ = _gpu_stripes(problem, 1, 8, 0, S, N.KERNEL_SPLIT, finalize=False)
    assert np.all(np.abs(d1 - d0) <= 1e-12 * np.abs(d0))
    assert np.all(np.abs(t1 - t0) <= 1e-12 * np.abs(t0))
    assert np.all(d1 <= t1)
    f, _, _ = _gpu_stripes(problem, 1, 8, 0, S, N.KERNEL_SPLIT)
    assert np.all((f >= 0) & (f <= 1))


@pytest.mark.parametrize("metric", [2, 3, 4])
def test_weighted_uwalk_combined_cells_bitwise(device_ok, metric, monkeypatch):
    """Combined (offset, presence word) cells feed the u-walk the same words
    and offsets as the separate arrays: bit-identical."""
    inst = sf.random_instance(68, 230, 900, 0.01)
    problem = sf.flatten(inst.tree, inst.table)
    S = 115
    out = []
    for nbo in ("1", "0"):
        monkeypatch.setenv("SF_UWALK_NBO", nbo)
        ex, _keep = N.make_exec([0], N.KERNEL_WUWALK, False, 0, 0.5)
        d = np.zeros((S, 230)); t = np.zeros((S, 230))
        N.check(N.lib().sf_compute_stripes(problem.ref, metric, 8, 0, S, N.ptr(d), N.ptr(t) if metric != 2 else None,
                                           1, C.byref(ex), None))
        out.append((d, t))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("prec", [8, 4])
def test_heavy_gemm_is_bitwise_the_dfma_walk(device_ok, prec, monkeypatch):
    """Heavy rows on the tensor cores (int8 digit-plane GEMMs, the default)
    and on the DFMA walk (SF_HEAVY_GEMM=0) compute the same exact integer
    sums: bit-identical stripes — mixed, all-heavy and all-light splits,
    several light passes, wide branch lengths (deep levels), odd/even n,
    wrap and partial ranges, GEMM blocks narrower than the range."""
    rng = np.random.default_rng(5)
    for seed, n, leaves, dens, frac, lp, wide, bk in [
            (111, 300, 1100, 0.01, "0.02", "0", False, "0"), (112, 257, 700, 0.03, "0.0", "7", False, "64"),
            (113, 130, 500, 0.05, "0.05", "0", True, "0"), (114, 64, 90, 0.3, "0.6", "0", False, "16")]:
        inst = sf.random_instance(seed, n, leaves, dens)
        problem = sf.flatten(inst.tree, inst.table)
        if wide:
            problem.lengths[:] = 10.0 ** rng.uniform(-30, 0.3, problem.n_rows)
        monkeypatch.setenv("SF_HEAVY_FRAC", frac)
        if lp != "0":
            monkeypatch.setenv("SF_LIGHT_PASS", lp)
        if bk != "0":
            monkeypatch.setenv("SF_GRAM_BK", bk)
        for start, stop in [(0, n // 2), (3, n // 2 - 2)]:
            monkeypatch.setenv("SF_HEAVY_GEMM", "0")
            wd, wt, _ = _gpu_stripes(problem, 1, prec, start, stop, N.KERNEL_SPLIT)
            monkeypatch.delenv("SF_HEAVY_GEMM")
            d, t, _ = _gpu_stripes(problem, 1, prec, start, stop, N.KERNEL_SPLIT)
            assert np.array_equal(d, wd) and np.array_equal(t, wt)
        for var in ("SF_LIGHT_PASS", "SF_GRAM_BK"):
            monkeypatch.delenv(var, raising=False)


def test_fit_probe_fallback_sizing_matches(device_ok, monkeypatch):
    """With the pool fit probes disabled (SF_FORCE_PROBE_FAIL=1) the plans
    size their chunks and light passes from free device memory instead: the
    results are bit-identical (the fallback was untested)."""
    inst = sf.random_instance(131, 300, 1200, 0.01)
    problem = sf.flatten(inst.tree, inst.table)
    for metric in (1, 3):
        want = _gpu_stripes(problem, metric, 8, 0, 150, N.KERNEL_AUTO)
        monkeypatch.setenv("SF_FORCE_PROBE_FAIL", "1")
        got = _gpu_stripes(problem, metric, 8, 0, 150, N.KERNEL_AUTO)
        monkeypatch.delenv("SF_FORCE_PROBE_FAIL")
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_plan_write_strf_over_several_devices(device_ok, tmp_path):
    """A plan sharded over devices writes the same .strf as a one-device
    plan (each device's chunks are recorded on events of its own device —
    ADVICE r1). Distinct devices when the box has them, else two shards of
    device 0."""
    inst = sf.random_instance(132, 400, 1500, 0.01)
    problem = sf.flatten(inst.tree, inst.table)
    ndev = min(2, N.lib().sf_device_count())
    devs = list(range(ndev)) if ndev >= 2 else [0, 0]
    paths = []
    for dl in ([0], devs):
        ex, _keep = N.make_exec(dl)
        plan = C.c_void_p()
        N.check(N.lib().sf_plan_create(problem.ref, 1, 8, 0, 200, C.byref(ex), C.byref(plan)))
        N.check(N.lib().sf_plan_run(plan, 1))
        p = tmp_path / f"p{len(dl)}.strf"
        N.check(N.lib().sf_plan_write_strf(plan, str(p).encode()))
        N.lib().sf_plan_destroy(plan)
        paths.append(p.read_bytes())
    assert paths[0] == paths[1]


def test_light_column_16bit_members_are_bitwise_the_32bit(device_ok, monkeypatch):
    """The column kernel reads 16-bit member lists when n <= 65536: the same
    exact light sums as the 32-bit lists (SF_LIGHT_MEM16=0), bit for bit."""
    inst = sf.random_instance(141, 900, 5000, 0.01)
    problem = sf.flatten(inst.tree, inst.table)
    for prec in (8, 4):
        want = _gpu_stripes(problem, 1, prec, 0, 450, N.KERNEL_SPLIT)
        monkeypatch.setenv("SF_LIGHT_MEM16", "0")
        got = _gpu_stripes(problem, 1, prec, 0, 450, N.KERNEL_SPLIT)
        monkeypatch.delenv("SF_LIGHT_MEM16")
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("chunk", ["1", "3", "64"])
def test_light_column_carry_folding_is_exact(device_ok, chunk, monkeypatch):
    """Three 21-bit limbs for every column, with the planes' carries folded
    into a fourth plane between entry chunks: any chunk size (tiny ones here,
    so cells fold many times, and lengths at the top of the grid so every
    limb carries) gives the same exact light sums as the four 16-bit limb
    mode (SF_LIGHT_LIMB_MODE=1), bit for bit, and matches the oracle."""
    inst = sf.random_instance(142, 700, 4000, 0.02)
    problem = sf.flatten(inst.tree, inst.table)
    rng = np.random.default_rng(int(chunk))
    problem.lengths[:] = np.where(rng.random(problem.n_rows) < 0.5, 2.0 - 1e-9 * rng.random(problem.n_rows),
                                  rng.random(problem.n_rows) * 2.0)
    monkeypatch.setenv("SF_HEAVY_FRAC", "0.3")
    for prec in (8, 4):
        monkeypatch.setenv("SF_LIGHT_LIMB_MODE", "1")
        want = _gpu_stripes(problem, 1, prec, 0, 350, N.KERNEL_SPLIT)
        monkeypatch.delenv("SF_LIGHT_LIMB_MODE")
        monkeypatch.setenv("SF_LIGHT_CHUNK_ENTRIES", chunk)
        got = _gpu_stripes(problem, 1, prec, 0, 350, N.KERNEL_SPLIT)
        monkeypatch.delenv("SF_LIGHT_CHUNK_ENTRIES")
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    wd, wt = op.compute_stripes(problem, 1, 8, 0, 350)
    got = _gpu_stripes(problem, 1, 8, 0, 350, N.KERNEL_SPLIT)
    _assert_close(1, 8, False, got[0], wd, N.KERNEL_SPLIT)


@pytest.mark.parametrize("metric", [1, 3])
def test_plan_create_rejects_invalid_problems(device_ok, metric):
    """sf_plan_create validates the tree before starting the schedule thread
    and the table after starting the table upload: every invalid problem is
    rejected with SF_EINVAL and its message, with no plan and no hang, on the
    split (unweighted) and weighted-split paths; a valid problem still plans."""
    inst = sf.random_instance(143, 40, 120, 0.2)
    base = sf.flatten(inst.tree, inst.table)

    def fresh():
        return N.Problem(base.parent_row.copy(), base.lengths.copy(), base.leaf_feature.copy(), base.n_samples,
                         base.feat_ptr.copy(), base.sample_idx.copy(), base.counts.copy(),
                         base.sample_totals.copy())

    def create(p):
        ex, _keep = N.make_exec([0], 0)
        plan = C.c_void_p()
        rc = N.lib().sf_plan_create(p.ref, metric, 8, 0, p.n_samples // 2, C.byref(ex), C.byref(plan))
        if plan.value:
            N.lib().sf_plan_destroy(plan)
        return rc, N.lib().sf_last_error().decode()

    def bad_length(p):
        p.lengths[3] = -1.0

    def bad_parent(p):
        p.parent_row[5] = 2

    def bad_order(p):
        f = int(np.argmax(np.diff(p.feat_ptr) >= 2))
        a = int(p.feat_ptr[f])
        p.sample_idx[a], p.sample_idx[a + 1] = p.sample_idx[a + 1], p.sample_idx[a]

    def bad_count(p):
        p.counts[7] = -2.0

    def bad_total(p):
        p.sample_totals[4] = 0.0

    for mutate, msg in ((bad_length, "branch length"), (bad_parent, "parent row"),
                        (bad_order, "ascending"), (bad_count, "non-negative"), (bad_total, "no counts")):
        p = fresh()
        mutate(p)
        rc, err = create(p)
        assert rc == N.SF_EINVAL and msg in err, (mutate.__name__, rc, err)
    assert create(fresh())[0] == 0
