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


def test_native_tsv_writer_is_the_reference_bytes(tmp_path):
    """sfh_write_tsv (parallel host writer) writes the reference's own TSV
    bytes (goldens written by write_tsv, stripes.cpp:311-340) for every demo
    matrix, with any thread count, and agrees with the Python to_tsv on
    random and edge values (0, 1, tiny, huge, fp32 digits)."""
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import golden_util as gu
    case = gu.load("demo.json")
    tree, table = gu.case_inputs(case)
    for entry in case["dm"]:
        n = table.n_samples()
        dm = sf.DistanceMatrix(list(table.sample_ids), np.array(entry["values"]).reshape(n, n),
                               sf.precision_from_name(entry["precision"]))
        for threads in (1, 3, 0):
            path = tmp_path / f"dm{threads}.tsv"
            sf.write_tsv(str(path), dm, threads=threads)
            assert path.read_bytes() == entry["tsv"].encode()
    rng = np.random.default_rng(3)
    n = 77
    vals = rng.random((n, n)) ** 7
    vals[0, :5] = [0.0, 1.0, 5e-324, 1.7976931348623157e308, 0.1]
    for prec in (sf.Precision.Fp64, sf.Precision.Fp32):
        dm = sf.DistanceMatrix([f"s{i}" for i in range(n)], vals, prec)
        path = tmp_path / "r.tsv"
        sf.write_tsv(str(path), dm, threads=5)
        assert path.read_text() == sf.to_tsv(dm)
    with pytest.raises(sf.Error):
        sf.write_tsv(str(tmp_path / "no" / "such" / "dir.tsv"), dm)


def _sparse_cases():
    rng = np.random.default_rng(11)
    cases = {}
    # random triplets, unordered, duplicates, some zero values, CRLF, blank lines
    lines = []
    for _ in range(4000):
        f = f"feat{rng.integers(0, 300)}"
        s = f"s{rng.integers(0, 40)}"
        v = float(rng.choice([0.0, 1.0, 2.5, 1e-3, 7.0, 0.1]))
        lines.append(f"{f}\t{s}\t{v!r}")
    for i in range(0, len(lines), 97):
        lines.insert(i, "")
    cases["unpinned"] = "\n".join(lines) + "\n"
    cases["crlf"] = "\r\n".join(lines)
    cases["pinned"] = "#samples\t" + "\t".join(f"s{i}" for i in range(40)) + "\n" + "\n".join(lines)
    cases["blank_then_header"] = "\n\n#samples\ts1\ts2\nB\ts2\t1\nA\ts1\t2\nB\ts2\t1\n"
    cases["unicode_and_bytes"] = "ét\ts1\t1\nZ\ts1\t1\n_a\ts2\t3\n"
    return cases


@pytest.mark.parametrize("name", list(_sparse_cases()))
def test_native_sparse_loader_matches_the_reference_restatement(tmp_path, name):
    """sfh_load_table_sparse (parallel native loader) vs the Python statement
    of load_sparse (table.cpp:105-168): identical ids, CSR and totals, bit for
    bit, with any thread count."""
    text = _sparse_cases()[name]
    path = tmp_path / "t.tsv"
    path.write_bytes(text.encode())
    want = sf.load_table(text, "tsv-sparse")
    for threads in (1, 4, 0):
        got = sf.load_table_file(str(path), "tsv-sparse", threads=threads)
        assert got.sample_ids == want.sample_ids and got.feature_ids == want.feature_ids
        assert np.array_equal(got.feat_ptr, want.feat_ptr)
        assert np.array_equal(got.sample_idx, want.sample_idx)
        assert np.array_equal(got.counts, want.counts)
        assert np.array_equal(got.sample_totals, want.sample_totals)


@pytest.mark.parametrize("text,msg", [
    ("A\ts1\n", "line 1: expected feature<TAB>sample<TAB>value"),
    ("A\ts1\t1\n\t\ts2\n", "line 2: feature id is empty"),
    ("A\ts1\t1\nB\ts1\t1\t2\n", "line 2: expected feature<TAB>sample<TAB>value"),
    ("A\ts1\t1\n\ts1\t1\n", "line 2: feature id is empty"),
    ("A\ts1\t1\nB\t\t1\n", "line 2: sample id is empty"),
    ("A\ts1\t1x\n", "line 1: bad count '1x'"),
    ("A\ts1\tinf\n", "line 1: count must be finite"),
    ("A\ts1\t-1\n", "line 1: count must be non-negative"),
    ("#samples\ts1\nA\ts2\t1\n", "line 2: sample 's2' not in the #samples header"),
    ("#samples\n", "#samples header names no samples"),
    ("#samples\ts1\ts1\n", "duplicate sample id 's1'"),
    ("", "sparse table names no samples"),
    ("#samples\ts1\ts2\nA\ts1\t1\n", "sample 's2' has no counts"),
    ("A\ts1\t0\n", "sample 's1' has no counts"),
])
def test_native_sparse_loader_errors(tmp_path, text, msg):
    """The reference's first error, prefixed by the path (table.cpp:180-183)."""
    path = tmp_path / "bad.tsv"
    path.write_bytes(text.encode())
    with pytest.raises(sf.Error) as e:
        sf.load_table_file(str(path), "tsv-sparse")
    assert str(e.value) == f"{path}: {msg}"
    with pytest.raises(sf.Error):
        sf.load_table(text, "tsv-sparse")


REF_DRIVER = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "ref_driver"


@pytest.mark.skipif(not REF_DRIVER.exists(), reason="reference not built (oracle/_ref)")
@pytest.mark.parametrize("name", list(_sparse_cases()) + ["err_fields", "err_pinned", "err_nocounts"])
def test_native_sparse_loader_is_the_reference_loader(tmp_path, name):
    """Against the reference's own load_table_file (oracle/_ref/ref_driver
    table, compiled from /root/reference): same ids, CSR, counts and totals
    (printed %.17g: exact), or the same error message."""
    import json
    import subprocess
    text = {**_sparse_cases(), "err_fields": "A\ts1\t1\nB\ts1\n", "err_pinned": "#samples\ts1\nA\ts9\t1\n",
            "err_nocounts": "#samples\ts1\ts2\nA\ts1\t1\n"}[name]
    path = tmp_path / "t.tsv"
    path.write_bytes(text.encode())
    ref = json.loads(subprocess.run([str(REF_DRIVER), "table", str(path), "tsv-sparse"], capture_output=True,
                                    text=True, check=True).stdout)
    if "error" in ref:
        with pytest.raises(sf.Error) as e:
            sf.load_table_file(str(path), "tsv-sparse")
        assert str(e.value) == ref["error"]
        return
    got = sf.load_table_file(str(path), "tsv-sparse", threads=3)
    assert got.sample_ids == ref["samples"] and got.feature_ids == ref["features"]
    assert got.feat_ptr.tolist() == ref["feat_ptr"] and got.sample_idx.tolist() == ref["sample_idx"]
    assert got.counts.tolist() == ref["counts"] and got.sample_totals.tolist() == ref["totals"]
