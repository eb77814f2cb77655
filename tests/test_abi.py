"""CPU: the C-ABI library loads and exports every symbol include/*.h declares;
host-side API behaviour that needs no device."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2005_05826_b200 import _native as N
from paper_2005_05826_b200 import stripefrac as sf

ROOT = Path(__file__).resolve().parent.parent


def declared_functions():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(sfh?_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_every_declared_symbol_is_exported():
    lib = N.lib()
    decl = declared_functions()
    assert len(decl) >= 20
    missing = [nm for nm in decl if not hasattr(lib, nm)]
    assert not missing, missing
    # and the ctypes table covers the whole header surface
    assert set(decl) == set(N.SIGNATURES), set(decl) ^ set(N.SIGNATURES)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(N.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_device_means_loud_failure():
    """Without an sm_100 device every compute entry point fails (no CPU fallback)."""
    if N.lib().sf_device_count() > 0:
        pytest.skip("a device is present")
    inst = sf.random_instance(1, 8, 6, 0.5)
    with pytest.raises(sf.Error):
        sf.compute_unifrac(inst.tree, inst.table, sf.KernelConfig())


def test_stripe_addressing():
    """test_stripes.cpp:15-29."""
    with pytest.raises(sf.Error):
        sf.total_stripes(1)
    assert sf.total_stripes(2) == 1 and sf.total_stripes(5) == 2 and sf.total_stripes(64) == 32
    assert sf.stripe_pair(5, 0, 4) == (4, 0)
    assert sf.stripe_pair(5, 1, 3) == (3, 0)
    assert sf.stripe_pair(6, 2, 5) == (5, 2)
    with pytest.raises(sf.Error):
        sf.stripe_pair(6, 3, 0)


def test_stripe_coverage():
    """acceptance.cpp:197-235: odd n covers each pair once, even n doubles n/2
    pairs, all in the last stripe."""
    for n in range(2, 65):
        S = n // 2
        hits = {}
        for s in range(S):
            for k in range(n):
                a, b = sf.stripe_pair(n, s, k)
                hits.setdefault((min(a, b), max(a, b)), []).append(s)
        assert len(hits) == n * (n - 1) // 2
        doubled = [v for v in hits.values() if len(v) == 2]
        assert all(v == [S - 1, S - 1] for v in doubled)
        assert len(doubled) == (n // 2 if n % 2 == 0 else 0)


def test_allocation_shapes():
    wu = sf.allocate_stripes(10, 1, 4, sf.Metric.WeightedUnnormalized)
    assert wu.distances.shape == (3, 10) and wu.totals.size == 0
    uw = sf.allocate_stripes(10, 0, 5, sf.Metric.Unweighted, sf.Precision.Fp32)
    assert uw.totals.shape == (5, 10) and uw.distances.dtype == np.float32
    for a, b, n in ((3, 3, 10), (0, 6, 10), (-1, 2, 10), (0, 1, 1)):
        with pytest.raises(sf.Error):
            sf.allocate_stripes(n, a, b, sf.Metric.Unweighted)


def test_stripe_file_round_trip_and_corruption(tmp_path):
    """test_stripes.cpp:186-260: round trip, bad magic, checksum."""
    rng = np.random.default_rng(3)
    s = sf.allocate_stripes(9, 1, 3, sf.Metric.WeightedNormalized)
    s.distances[:] = rng.random(s.distances.shape)
    s.totals[:] = 1.0
    s.finalized = True
    p = tmp_path / "part.strf"
    sf.write_stripe_file(str(p), s)
    got = sf.read_stripe_file(str(p))
    assert got.start == 1 and got.stop == 3 and got.n_samples == 9
    assert np.array_equal(got.distances, s.distances) and np.array_equal(got.totals, s.totals)
    blob = bytearray(p.read_bytes())
    blob[40] ^= 0xFF
    p.write_bytes(bytes(blob))
    with pytest.raises(sf.Error, match="checksum"):
        sf.read_stripe_file(str(p))
    p.write_bytes(b"XXXX" + bytes(blob[4:]))
    with pytest.raises(sf.Error, match="magic"):
        sf.read_stripe_file(str(p))
    s.finalized = False
    with pytest.raises(sf.Error):
        sf.write_stripe_file(str(p), s)


def test_condense_rejects_bad_tilings():
    """test_stripes.cpp:134-157 (validation happens before any device work)."""
    def parts(ranges, metric=sf.Metric.WeightedUnnormalized):
        out = []
        for a, b in ranges:
            s = sf.allocate_stripes(12, a, b, metric)
            s.finalized = True
            out.append(s)
        return out
    with pytest.raises(sf.Error, match="gap"):
        sf.condense(parts([(0, 2), (3, 6)]))
    with pytest.raises(sf.Error, match="overlap"):
        sf.condense(parts([(0, 3), (2, 6)]))
    with pytest.raises(sf.Error, match="gap"):
        sf.condense(parts([(0, 5)]))
    with pytest.raises(sf.Error):
        sf.condense([])
    mixed = parts([(0, 3)]) + parts([(3, 6)], sf.Metric.Unweighted)
    with pytest.raises(sf.Error):
        sf.condense(mixed)


MALFORMED = ["", ";", "(A:1,B:2", "(A:1,B:2));", "A:1,B:2);", "(A:1,,B:2);", "(A:1 B:2);",
             "(A:;", "(A:1e);", "(A:-1);", "(A:1,A:2);", "(A:1)extra:1;trailing",
             "('unterminated:1);", "(A:1,B:nan);", "(:1,:2);"]


@pytest.mark.parametrize("text", MALFORMED)
def test_newick_malformed_inputs_raise_positioned_errors(text):
    """acceptance.cpp:326-366."""
    with pytest.raises(sf.ParseError) as ei:
        sf.parse_newick(text)
    assert "character" in str(ei.value) and ei.value.offset <= len(text)


def test_newick_parse_basics():
    t = sf.parse_newick("((A:1,B:2)ab:0.5,'C''x':3e0)root:7;")
    assert t.n_leaves == 3 and t.leaf_names == ["A", "B", "C'x"]
    assert [t.names[v] for v in t.postorder] == ["A", "B", "ab", "C'x"]
    assert t.length[t.root] == 0.0


def test_tables_dense_and_sparse():
    dense = sf.load_table("#id\ts1\ts2\tA\n" if False else "#id\ts1\ts2\nA\t4\t0\nB\t0\t2\n", "tsv-dense")
    assert dense.feature_ids == ["A", "B"] and dense.sample_totals.tolist() == [4.0, 2.0]
    sparse = sf.load_table("#samples\ts1\ts2\nB\ts2\t1\nA\ts1\t2\nB\ts2\t1\n", "tsv-sparse")
    assert sparse.feature_ids == ["A", "B"]
    assert sparse.entries(1) == [(1, 2.0)]
    with pytest.raises(sf.Error):
        sf.load_table("#id\ts1\nA\t-1\n", "tsv-dense")
    with pytest.raises(sf.Error):
        sf.load_table("#id\ts1\ts2\nA\t0\t1\n", "tsv-dense")  # s1 has no counts


def test_counter_law_is_host_side():
    cfg = sf.KernelConfig(sf.Metric.WeightedNormalized, sf.Variant.Naive, batch_capacity=4)
    c = sf._counters_for(cfg, 10, 50, 3)
    assert (c.accumulator_writes, c.embedding_reads, c.kernel_passes) == (500, 1000, 3)
