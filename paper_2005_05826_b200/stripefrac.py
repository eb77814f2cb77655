"""Python mirror of the reference ``stripefrac`` API, served by the B200 C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/stripefrac/*.hpp) so tests read like the
reference's own. Everything numeric on the hot path — embedding (K1), stripe
update (K2), finalize (K3), condense (K4) — runs in the sm_100a library
through ``_native``; this module only parses inputs, flattens trees, applies
the reference's preconditions and counter law, and handles file formats.
There is no CPU fallback: without the CUDA library or an sm_100 device the
compute entry points raise.
"""
from __future__ import annotations

import ctypes as C
import enum
import io
import math
import os
import struct
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

import numpy as np

from . import _native as N


# --------------------------------------------------------------------- errors
class Error(RuntimeError):
    """stripefrac::Error (common.hpp:14-17)."""


class ParseError(Error):
    """Newick parse error with a character offset (newick.hpp:35-43)."""

    def __init__(self, msg: str, offset: int):
        super().__init__(f"{msg} (at character {offset})")
        self.offset = offset


def _call(status: int) -> None:
    if status != N.SF_OK:
        raise Error(N.lib().sf_last_error().decode("utf-8", "replace"))


# ---------------------------------------------------------------------- enums
class Metric(enum.IntEnum):  # common.hpp:19; values are the .strf metric codes
    Unweighted = 1
    WeightedUnnormalized = 2
    WeightedNormalized = 3
    # extension, not in the reference (parity unpinned): generalized UniFrac
    # with exponent KernelConfig.alpha (SF_GENERALIZED in the C ABI)
    Generalized = 4


class Variant(enum.IntEnum):  # common.hpp:20
    Naive = 0
    Batched = 1
    Tiled = 2


class Precision(enum.IntEnum):  # common.hpp:21; values are scalar widths
    Fp32 = 4
    Fp64 = 8


_METRIC_NAMES = {Metric.Unweighted: "unweighted", Metric.WeightedUnnormalized: "weighted-unnormalized",
                 Metric.WeightedNormalized: "weighted-normalized", Metric.Generalized: "generalized"}
_VARIANT_NAMES = {Variant.Naive: "naive", Variant.Batched: "batched", Variant.Tiled: "tiled"}


def name(x) -> str:
    """name(Metric|Variant|Precision) (common.cpp:9-29)."""
    if isinstance(x, Metric):
        return _METRIC_NAMES[x]
    if isinstance(x, Variant):
        return _VARIANT_NAMES[x]
    if isinstance(x, Precision):
        return "fp32" if x == Precision.Fp32 else "fp64"
    raise Error(f"no name for {x!r}")


def metric_from_name(s: str) -> Metric:
    for k, v in _METRIC_NAMES.items():
        if v == s:
            return k
    raise Error(f"unknown metric '{s}'")


def variant_from_name(s: str) -> Variant:
    for k, v in _VARIANT_NAMES.items():
        if v == s:
            return k
    raise Error(f"unknown variant '{s}'")


def precision_from_name(s: str) -> Precision:
    if s == "fp32":
        return Precision.Fp32
    if s == "fp64":
        return Precision.Fp64
    raise Error(f"unknown precision '{s}'")


def metric_has_totals(m: Metric) -> bool:
    return m != Metric.WeightedUnnormalized


def _dtype(p: Precision):
    return np.float32 if p == Precision.Fp32 else np.float64


@dataclass
class KernelConfig:
    """KernelConfig (kernels.hpp:15-26). variant/batch/step do not change bits."""

    metric: Metric = Metric.Unweighted
    variant: Variant = Variant.Tiled
    precision: Precision = Precision.Fp64
    batch_capacity: int = 64
    step_size: int = 0
    alpha: float = 1.0  # Metric.Generalized only (extension)

    def resolved_step_size(self) -> int:
        if self.step_size > 0:
            return self.step_size
        return 32 if self.precision == Precision.Fp32 else 16


@dataclass
class KernelCounters:
    """KernelCounters (kernels.hpp:33-44): exact accounting from loop bounds."""

    accumulator_writes: int = 0
    embedding_reads: int = 0
    kernel_passes: int = 0

    def __iadd__(self, o: "KernelCounters") -> "KernelCounters":
        self.accumulator_writes += o.accumulator_writes
        self.embedding_reads += o.embedding_reads
        self.kernel_passes += o.kernel_passes
        return self


# ----------------------------------------------------------------------- tree
class PhyloTree:
    """Rooted phylogeny (newick.hpp:23-33) over parent links.

    ``parent[i] = -1`` for the root; ``names[i]`` is the label ('' if none).
    children / postorder / leaf_names follow finalize_topology
    (newick.cpp:169-219): children in node-index order, iterative postorder
    without the root.
    """

    def __init__(self, parent, length, names=None, finalize: bool = True):
        self.parent = np.ascontiguousarray(parent, dtype=np.int32)
        self.length = np.ascontiguousarray(length, dtype=np.float64)
        self._names = names
        self.root = -1
        if finalize:
            self._finalize()

    # names are materialised lazily for synthetic trees ("f<i>" for leaves)
    @property
    def names(self) -> List[str]:
        if self._names is None:
            n = self.n_nodes
            is_leaf = self._leaf_mask()
            self._names = [f"f{i}" if is_leaf[i] else "" for i in range(n)]
        return self._names

    @property
    def n_nodes(self) -> int:
        return int(self.parent.shape[0])

    def _leaf_mask(self) -> np.ndarray:
        has_child = np.zeros(self.n_nodes, dtype=bool)
        p = self.parent[self.parent >= 0]
        has_child[p] = True
        return ~has_child

    def _finalize(self) -> None:
        n = self.n_nodes
        if n == 0:
            raise Error("tree has no nodes")
        ln = self.length
        if not np.all(np.isfinite(ln)) or np.any(ln < 0):
            raise Error("branch length must be finite and non-negative")
        roots = np.flatnonzero(self.parent < 0)
        if len(roots) > 1:
            raise Error("tree has more than one root")
        if len(roots) == 0:
            raise Error("tree has no root")
        if np.any(self.parent >= n):
            raise Error("parent index out of range")
        self.root = int(roots[0])
        children: List[List[int]] = [[] for _ in range(n)]
        for i in range(n):
            p = int(self.parent[i])
            if p >= 0:
                children[p].append(i)
        self.children = children
        post = []
        stack = [(self.root, 0)]
        visited = 0
        while stack:
            node, slot = stack[-1]
            kids = children[node]
            if slot < len(kids):
                stack[-1] = (node, slot + 1)
                stack.append((kids[slot], 0))
            else:
                visited += 1
                if node != self.root:
                    post.append(node)
                stack.pop()
        if visited != n:
            raise Error("tree has nodes unreachable from the root")
        self.postorder = post
        names = self.names
        leaf_names, seen = [], set()
        for i in range(n):
            if children[i]:
                continue
            nm = names[i]
            if not nm:
                raise Error("leaf with empty name")
            if nm in seen:
                raise Error(f"duplicate leaf name '{nm}'")
            seen.add(nm)
            leaf_names.append(nm)
        self.leaf_names = leaf_names

    def is_leaf(self, i: int) -> bool:
        return not self.children[i]

    @property
    def n_leaves(self) -> int:
        return len(self.leaf_names)


_UNQUOTED_STOP = "()[]{}:;,'"
_SPACE = " \t\n\r\v\f"


def parse_newick(text: str) -> PhyloTree:
    """parse_newick (newick.cpp:140-156): positioned errors, quoted labels,
    multifurcations, missing lengths = 0, root length ignored."""
    pos = 0
    nodes_parent: List[int] = []
    nodes_len: List[float] = []
    nodes_name: List[str] = []
    seen = set()
    n = len(text)

    def fail(msg, at=None):
        raise ParseError(msg, pos if at is None else at)

    def skip_ws():
        nonlocal pos
        while pos < n and text[pos] in _SPACE:
            pos += 1

    def parse_label():
        nonlocal pos
        skip_ws()
        if pos >= n:
            return ""
        if text[pos] == "'":
            pos += 1
            out = []
            while True:
                if pos >= n:
                    fail("unterminated quoted label")
                c = text[pos]
                pos += 1
                if c == "'":
                    if pos < n and text[pos] == "'":
                        out.append("'")
                        pos += 1
                    else:
                        return "".join(out)
                else:
                    out.append(c)
        begin = pos
        while pos < n and text[pos] not in _SPACE and text[pos] not in _UNQUOTED_STOP:
            pos += 1
        return text[begin:pos]

    def parse_length():
        nonlocal pos
        skip_ws()
        if pos < n and text[pos] == "+":
            pos += 1
        # std::from_chars general format: [-]digits[.digits][e[+-]digits], inf, nan
        j = pos
        if j < n and text[j] == "-":
            j += 1
        k = j
        low = text[k:k + 8].lower()
        if low.startswith("infinity"):
            k += 8
        elif low.startswith("inf") or low.startswith("nan"):
            k += 3
            if low.startswith("nan") and k < n and text[k] == "(":
                close = text.find(")", k)
                if close >= 0:
                    k = close + 1
        else:
            digits = 0
            while k < n and text[k].isdigit():
                k += 1
                digits += 1
            if k < n and text[k] == ".":
                k += 1
                while k < n and text[k].isdigit():
                    k += 1
                    digits += 1
            if digits == 0:
                fail("expected a branch length")
            if k < n and text[k] in "eE":
                e = k + 1
                if e < n and text[e] in "+-":
                    e += 1
                if e < n and text[e].isdigit():
                    while e < n and text[e].isdigit():
                        e += 1
                    k = e
        if k == pos:
            fail("expected a branch length")
        try:
            value = float(text[pos:k])
        except ValueError:
            fail("expected a branch length")
        pos = k
        if not math.isfinite(value):
            fail("branch length must be finite")
        if value < 0.0:
            fail("branch length must be non-negative")
        return value

    def new_node():
        nodes_parent.append(-1)
        nodes_len.append(0.0)
        nodes_name.append("")
        return len(nodes_parent) - 1

    def parse_subtree():
        nonlocal pos
        skip_ws()
        if pos >= n:
            fail("unexpected end of input")
        if text[pos] == "(":
            pos += 1
            kids = []
            while True:
                kids.append(parse_subtree())
                skip_ws()
                if pos >= n:
                    fail("unbalanced parentheses")
                c = text[pos]
                if c == ",":
                    pos += 1
                    continue
                if c == ")":
                    pos += 1
                    break
                fail("expected ',' or ')'")
            node = new_node()
            nodes_name[node] = parse_label()
            for k in kids:
                nodes_parent[k] = node
            skip_ws()
            if pos < n and text[pos] == ":":
                pos += 1
                nodes_len[node] = parse_length()
            return node
        label_pos = pos
        label = parse_label()
        if not label:
            pos = label_pos
            fail("expected a leaf name")
        if label in seen:
            pos = label_pos
            fail(f"duplicate leaf name '{label}'")
        seen.add(label)
        node = new_node()
        nodes_name[node] = label
        skip_ws()
        if pos < n and text[pos] == ":":
            pos += 1
            nodes_len[node] = parse_length()
        return node

    import sys
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 10 * n + 1000))
    try:
        skip_ws()
        if pos >= n:
            fail("empty input")
        root = parse_subtree()
        skip_ws()
        if pos >= n:
            fail("unbalanced parentheses")
        if text[pos] != ";":
            fail("expected ';'")
        pos += 1
        skip_ws()
        if pos < n:
            fail("trailing text after ';'")
    finally:
        sys.setrecursionlimit(old)
    nodes_len[root] = 0.0
    nodes_parent[root] = -1
    return PhyloTree(nodes_parent, nodes_len, nodes_name)


def parse_newick_file(path: str) -> PhyloTree:
    """parse_newick_file (newick.cpp:158-167): everything through the first ';'."""
    try:
        with open(path, "r", encoding="utf-8", newline="") as fh:
            text = fh.read()
    except OSError:
        raise Error(f"cannot open tree file '{path}'") from None
    semi = text.find(";")
    if semi < 0:
        raise Error(f"tree file '{path}' has no ';'")
    return parse_newick(text[:semi + 1])


# ---------------------------------------------------------------------- table
class SampleTable:
    """Sparse feature-by-sample counts (table.hpp:17-25), CSR by feature."""

    def __init__(self, sample_ids, feature_ids, feat_ptr, sample_idx, counts, sample_totals=None):
        self.sample_ids = list(sample_ids)
        self.feature_ids = list(feature_ids)
        self.feat_ptr = np.ascontiguousarray(feat_ptr, dtype=np.int64)
        self.sample_idx = np.ascontiguousarray(sample_idx, dtype=np.int32)
        self.counts = np.ascontiguousarray(counts, dtype=np.float64)
        if sample_totals is None:
            sample_totals = _sample_totals(len(self.sample_ids), self.sample_idx, self.counts)
        self.sample_totals = np.ascontiguousarray(sample_totals, dtype=np.float64)
        for s, t in enumerate(self.sample_totals):
            if not t > 0.0:
                raise Error(f"sample '{self.sample_ids[s]}' has no counts")

    def n_samples(self) -> int:
        return len(self.sample_ids)

    def n_features(self) -> int:
        return len(self.feature_ids)

    def entries(self, f: int):
        a, b = int(self.feat_ptr[f]), int(self.feat_ptr[f + 1])
        return list(zip(self.sample_idx[a:b].tolist(), self.counts[a:b].tolist()))


def _sample_totals(n, sidx, counts) -> np.ndarray:
    # check_sample_totals (table.cpp:55-62): sequential sum in entry order
    tot = [0.0] * n
    for s, c in zip(sidx.tolist(), counts.tolist()):
        tot[s] += c
    return np.array(tot, dtype=np.float64)


def _check_unique(ids, what):
    seen = set()
    for i in ids:
        if not i:
            raise Error(f"{what} id is empty")
        if i in seen:
            raise Error(f"duplicate {what} id '{i}'")
        seen.add(i)


def make_table(sample_ids, feature_ids, counts) -> SampleTable:
    """make_table (table.cpp:186-206)."""
    counts = np.asarray(counts, dtype=np.float64)
    if counts.shape != (len(feature_ids), len(sample_ids)):
        raise Error("make_table: counts shape does not match ids")
    _check_unique(sample_ids, "sample")
    _check_unique(feature_ids, "feature")
    if not np.all(np.isfinite(counts)) or np.any(counts < 0):
        raise Error("make_table: bad count")
    ptr, sidx, vals = [0], [], []
    for f in range(counts.shape[0]):
        nz = np.flatnonzero(counts[f] > 0)
        sidx.extend(nz.tolist())
        vals.extend(counts[f, nz].tolist())
        ptr.append(len(sidx))
    return SampleTable(sample_ids, feature_ids, ptr, sidx, vals)


def _parse_count(cell: str, line_no: int) -> float:
    try:
        if cell.strip() != cell or not cell or cell.lower() in ("infinity", "+inf", "inf", "nan"):
            raise ValueError
        v = float(cell)
    except ValueError:
        raise Error(f"line {line_no}: bad count '{cell}'") from None
    if not math.isfinite(v):
        raise Error(f"line {line_no}: count must be finite")
    if v < 0.0:
        raise Error(f"line {line_no}: count must be non-negative")
    return v


def load_table(stream, fmt: str = "tsv-dense") -> SampleTable:
    """load_table (table.cpp:72-174): 'tsv-dense' or 'tsv-sparse'."""
    if isinstance(stream, str):
        stream = io.StringIO(stream)
    lines = [ln[:-1] if ln.endswith("\r") else ln for ln in stream.read().split("\n")]
    if lines and lines[-1] == "":
        lines.pop()
    if fmt == "tsv-dense":
        if not lines:
            raise Error("dense table is empty")
        header = lines[0].split("\t")
        if not header or header[0] != "#id":
            raise Error("dense table header must start with '#id'")
        if len(header) < 2:
            raise Error("dense table header names no samples")
        samples = header[1:]
        _check_unique(samples, "sample")
        feats, ptr, sidx, vals = [], [0], [], []
        for i, line in enumerate(lines[1:], start=2):
            if not line:
                continue
            cells = line.split("\t")
            if len(cells) != len(header):
                raise Error(f"line {i}: expected {len(header)} fields, got {len(cells)}")
            feats.append(cells[0])
            for s, cell in enumerate(cells[1:]):
                v = _parse_count(cell, i)
                if v > 0.0:
                    sidx.append(s)
                    vals.append(v)
            ptr.append(len(sidx))
        _check_unique(feats, "feature")
        return SampleTable(samples, feats, ptr, sidx, vals)
    if fmt == "tsv-sparse":
        order: List[str] = []
        index = {}
        pinned = False
        features = {}
        first = True
        for i, line in enumerate(lines, start=1):
            if not line:
                continue
            cells = line.split("\t")
            if first and cells[0] == "#samples":
                first = False
                if len(cells) < 2:
                    raise Error("#samples header names no samples")
                order = cells[1:]
                _check_unique(order, "sample")
                index = {s: j for j, s in enumerate(order)}
                pinned = True
                continue
            first = False
            if len(cells) != 3:
                raise Error(f"line {i}: expected feature<TAB>sample<TAB>value")
            if not cells[0]:
                raise Error(f"line {i}: feature id is empty")
            if not cells[1]:
                raise Error(f"line {i}: sample id is empty")
            v = _parse_count(cells[2], i)
            if cells[1] not in index:
                if pinned:
                    raise Error(f"line {i}: sample '{cells[1]}' not in the #samples header")
                index[cells[1]] = len(order)
                order.append(cells[1])
            s = index[cells[1]]
            row = features.setdefault(cells[0], {})
            row[s] = row.get(s, 0.0) + v
        if not order:
            raise Error("sparse table names no samples")
        feats, ptr, sidx, vals = [], [0], [], []
        for fid in sorted(features, key=lambda x: x.encode()):
            feats.append(fid)
            for s in sorted(features[fid]):
                if features[fid][s] > 0.0:
                    sidx.append(s)
                    vals.append(features[fid][s])
            ptr.append(len(sidx))
        return SampleTable(order, feats, ptr, sidx, vals)
    raise Error(f"unknown table format '{fmt}'")


def _load_sparse_native(path: str, threads: int = 0) -> SampleTable:
    """load_table_file(path, TsvSparse) through the native parallel loader
    (sfh_load_table_sparse): the same table bit for bit, the same errors."""
    L = N.lib()
    h = C.c_void_p()
    st = L.sfh_load_table_sparse(str(path).encode(), int(threads), C.byref(h))
    if st != 0:
        raise Error(L.sf_last_error().decode("utf-8", "replace"))
    try:
        ns, nf, nnz = L.sfh_table_n_samples(h), L.sfh_table_n_features(h), L.sfh_table_nnz(h)
        samples = [L.sfh_table_sample_id(h, i).decode() for i in range(ns)]
        feats = [L.sfh_table_feature_id(h, i).decode() for i in range(nf)]
        ptr = np.ctypeslib.as_array(L.sfh_table_feat_ptr(h), shape=(nf + 1,)).copy()
        sidx = np.ctypeslib.as_array(L.sfh_table_sample_idx(h), shape=(max(nnz, 1),))[:nnz].copy()
        cnt = np.ctypeslib.as_array(L.sfh_table_counts(h), shape=(max(nnz, 1),))[:nnz].copy()
        tot = np.ctypeslib.as_array(L.sfh_table_sample_totals(h), shape=(ns,)).copy()
    finally:
        L.sfh_table_free(h)
    return SampleTable(samples, feats, ptr, sidx, cnt, tot)


def load_table_file(path: str, fmt: str = "tsv-dense", threads: int = 0) -> SampleTable:
    """load_table_file (table.cpp:176-184); 'tsv-sparse' files go through the
    native parallel loader."""
    if fmt == "tsv-sparse":
        return _load_sparse_native(path, threads)
    try:
        with open(path, "r", encoding="utf-8", newline="") as fh:
            text = fh.read()
    except OSError:
        raise Error(f"cannot open table file '{path}'") from None
    try:
        return load_table(text, fmt)
    except Error as e:
        raise Error(f"{path}: {e}") from None


# ----------------------------------------------------------------- synthetic
@dataclass
class SynthInstance:
    tree: PhyloTree
    table: SampleTable


def random_instance(seed: int, n_samples: int, n_leaves: int, density: float = 0.3,
                    table_features: int = 0, finalize_tree: bool = True) -> SynthInstance:
    """random_instance (synth.cpp:70-83), generated natively on the same
    <random> engines, so the instance is the reference's bit for bit."""
    L = N.lib()
    h = L.sfh_random_instance(int(seed), int(n_samples), int(n_leaves), float(density),
                              int(table_features))
    if not h:
        raise Error(L.sf_last_error().decode())
    try:
        nn = L.sfh_instance_n_nodes(h)
        F = L.sfh_instance_n_features(h)
        nnz = L.sfh_instance_nnz(h)

        def arr(fn, ctype, count, dtype):
            p = C.cast(fn(h), C.POINTER(ctype))
            return np.ctypeslib.as_array(p, shape=(count,)).astype(dtype, copy=True) if count else np.zeros(0, dtype)

        parent = arr(L.sfh_instance_parent, C.c_int32, nn, np.int32)
        length = arr(L.sfh_instance_length, C.c_double, nn, np.float64)
        fleaf = arr(L.sfh_instance_feature_leaf, C.c_int32, F, np.int32)
        fptr = arr(L.sfh_instance_feat_ptr, C.c_int64, F + 1, np.int64)
        sidx = arr(L.sfh_instance_sample_idx, C.c_int32, nnz, np.int32)
        cnts = arr(L.sfh_instance_counts, C.c_double, nnz, np.float64)
        tots = arr(L.sfh_instance_sample_totals, C.c_double, n_samples, np.float64)
    finally:
        L.sfh_instance_free(h)
    tree = PhyloTree(parent, length, None, finalize=finalize_tree)
    table = SampleTable([f"s{j}" for j in range(n_samples)], [f"f{int(i)}" for i in fleaf],
                        fptr, sidx, cnts, tots)
    table._feature_leaf = fleaf  # fast path for flatten: leaves are nodes f<i> = i
    return SynthInstance(tree, table)


# --------------------------------------------------------------- flattening
def flatten(tree: PhyloTree, table: SampleTable) -> N.Problem:
    """sheared_to_table (embed.cpp:8-15) + postorder rows -> sf_problem."""
    fleaf = getattr(table, "_feature_leaf", None)
    if fleaf is None:
        index = {}
        is_leaf = tree._leaf_mask()
        names = tree.names
        for i in np.flatnonzero(is_leaf).tolist():
            index[names[i]] = i
        fleaf = np.empty(table.n_features(), dtype=np.int32)
        for f, fid in enumerate(table.feature_ids):
            if fid not in index:
                raise Error(f"table feature '{fid}' is not a leaf of the tree")
            fleaf[f] = index[fid]
    fleaf = np.ascontiguousarray(fleaf, dtype=np.int32)
    nn = tree.n_nodes
    parent_row = np.empty(nn, dtype=np.int32)
    lengths = np.empty(nn, dtype=np.float64)
    leaf_feature = np.empty(nn, dtype=np.int32)
    n_rows = C.c_int32(0)
    L = N.lib()
    _call(L.sfh_flatten(nn, N.ptr(tree.parent), N.ptr(tree.length), len(fleaf), N.ptr(fleaf),
                        C.byref(n_rows), N.ptr(parent_row), N.ptr(lengths), N.ptr(leaf_feature)))
    E = n_rows.value
    return N.Problem(parent_row[:E], lengths[:E], leaf_feature[:E], table.n_samples(),
                     table.feat_ptr, table.sample_idx, table.counts, table.sample_totals)


# -------------------------------------------------------------------- stripes
def total_stripes(n_samples: int) -> int:
    """total_stripes (stripes.cpp:17-21)."""
    if n_samples < 2:
        raise Error(f"need at least 2 samples, got {n_samples}")
    return n_samples // 2


def stripe_pair(n_samples: int, stripe: int, k: int):
    """stripe_pair (stripes.cpp:23-28)."""
    S = total_stripes(n_samples)
    if stripe < 0 or stripe >= S:
        raise Error("stripe index out of range")
    if k < 0 or k >= n_samples:
        raise Error("stripe slot out of range")
    return k, (k + stripe + 1) % n_samples


@dataclass
class StripeSet:
    """StripeSet<Real> (stripes.hpp:25-37); dtype carries the precision."""

    n_samples: int
    start: int
    stop: int
    metric: Metric
    distances: np.ndarray
    totals: np.ndarray
    finalized: bool = False

    def n_stripes(self) -> int:
        return self.stop - self.start

    def has_totals(self) -> bool:
        return metric_has_totals(self.metric)

    @property
    def precision(self) -> Precision:
        return Precision.Fp32 if self.distances.dtype == np.float32 else Precision.Fp64


def allocate_stripes(n_samples: int, start: int, stop: int, metric: Metric,
                     precision: Precision = Precision.Fp64) -> StripeSet:
    """allocate_stripes (stripes.cpp:30-44)."""
    S = total_stripes(n_samples)
    if start < 0 or stop > S or start >= stop:
        raise Error(f"stripe range {start}:{stop} does not fit in [0,{S})")
    dt = _dtype(precision)
    d = np.zeros((stop - start, n_samples), dtype=dt)
    t = np.zeros((stop - start, n_samples), dtype=dt) if metric_has_totals(metric) else np.zeros((0, 0), dt)
    return StripeSet(n_samples, start, stop, Metric(metric), d, t)


@dataclass
class DistanceMatrix:
    """DistanceMatrix (stripes.hpp:44-50): values in double, precision tag."""

    sample_ids: List[str]
    values: np.ndarray
    precision: Precision = Precision.Fp64

    def n(self) -> int:
        return int(self.values.shape[0])


@dataclass
class ExecOptions:
    """Device placement / kernel selection for this implementation (not in
    the reference API; defaults reproduce the reference semantics)."""

    devices: Optional[Sequence[int]] = None
    kernel: int = N.KERNEL_AUTO
    exact: bool = False
    mem_budget_bytes: int = 0


def _counters_for(cfg: KernelConfig, rows: int, entries: int, passes: int) -> KernelCounters:
    # counter law (kernels.hpp:202-207, 246, 292)
    writes = (rows if cfg.variant == Variant.Naive else passes) * entries
    return KernelCounters(writes, 2 * rows * entries, passes)


def _check_cfg(cfg: KernelConfig, real=None):
    if real is not None:
        want = Precision.Fp32 if np.dtype(real) == np.float32 else Precision.Fp64
        if cfg.precision != want:
            raise Error(f"config asks for {name(cfg.precision)} but compute_unifrac was "
                        f"instantiated for {name(want)}")
    if cfg.batch_capacity < 1:
        raise Error("batch capacity must be >= 1")
    if cfg.resolved_step_size() < 1:
        raise Error("step size must be >= 1")


def compute_unifrac(tree: PhyloTree, table: SampleTable, cfg: KernelConfig, start: int = 0,
                    stop: int = -1, threads: int = 1, counters: Optional[KernelCounters] = None,
                    real=None, exec_options: Optional[ExecOptions] = None,
                    stats: Optional[dict] = None) -> StripeSet:
    """compute_unifrac<Real> (kernels.hpp:268-316) on the B200 path.

    ``threads`` is accepted for API parity; work is sharded over devices
    instead (``exec_options.devices``). Counters follow the reference law.
    """
    _check_cfg(cfg, real)
    S = total_stripes(table.n_samples())
    if stop < 0:
        stop = S
    problem = flatten(tree, table)
    sset = allocate_stripes(table.n_samples(), start, stop, cfg.metric, cfg.precision)
    eo = exec_options or ExecOptions()
    ex, _keep = N.make_exec(eo.devices, eo.kernel, eo.exact, eo.mem_budget_bytes, cfg.alpha)
    st = N.sf_stats()
    tot_ptr = N.ptr(sset.totals) if sset.has_totals() else None
    _call(N.lib().sf_compute_stripes(problem.ref, int(cfg.metric), int(cfg.precision), start, stop,
                                     N.ptr(sset.distances), tot_ptr, 1, C.byref(ex), C.byref(st)))
    sset.finalized = True
    if counters is not None:
        E = problem.n_rows
        passes = -(-E // cfg.batch_capacity)
        counters += _counters_for(cfg, E, sset.n_stripes() * table.n_samples(), passes)
    if stats is not None:
        stats.update(st.as_dict())
    return sset


def compute_unifrac_to_strf(tree: PhyloTree, table: SampleTable, cfg: KernelConfig, path: str,
                            start: int = 0, stop: int = -1,
                            exec_options: Optional[ExecOptions] = None) -> None:
    """compute_unifrac + write_stripe_file (stripes.cpp:179-201) without a
    host copy of the stripes: sf_plan_write_strf streams them from device."""
    _check_cfg(cfg)
    if stop < 0:
        stop = total_stripes(table.n_samples())
    problem = flatten(tree, table)
    eo = exec_options or ExecOptions()
    ex, _keep = N.make_exec(eo.devices, eo.kernel, eo.exact, eo.mem_budget_bytes, cfg.alpha)
    plan = C.c_void_p()
    _call(N.lib().sf_plan_create(problem.ref, int(cfg.metric), int(cfg.precision), start, stop,
                                 C.byref(ex), C.byref(plan)))
    try:
        _call(N.lib().sf_plan_run(plan, 1))
        _call(N.lib().sf_plan_write_strf(plan, str(path).encode()))
    finally:
        N.lib().sf_plan_destroy(plan)


def compute_distance_matrix(tree: PhyloTree, table: SampleTable, cfg: KernelConfig,
                            threads: int = 1, counters: Optional[KernelCounters] = None,
                            real=None, exec_options: Optional[ExecOptions] = None) -> DistanceMatrix:
    """compute_distance_matrix<Real> (kernels.hpp:319-326): the stripes stay
    on the device; condense (stripes.cpp:68-129) runs there and the n x n
    matrix is copied to the host once (sf_compute_distance_matrix)."""
    _check_cfg(cfg, real)
    n = table.n_samples()
    S = total_stripes(n)
    problem = flatten(tree, table)
    eo = exec_options or ExecOptions()
    ex, _keep = N.make_exec(eo.devices, eo.kernel, eo.exact, eo.mem_budget_bytes, cfg.alpha)
    out = np.empty((n, n), dtype=np.float64)
    st = N.sf_stats()
    rc = N.lib().sf_compute_distance_matrix(problem.ref, int(cfg.metric), int(cfg.precision), N.ptr(out),
                                            C.byref(ex), C.byref(st))
    if rc != N.SF_OK:
        msg = N.lib().sf_last_error().decode()
        if "duplicated" in msg:
            raise Error("condense: duplicated slot disagrees")
        raise Error(msg)
    if counters is not None:
        E = problem.n_rows
        counters += _counters_for(cfg, E, S * n, -(-E // cfg.batch_capacity))
    return DistanceMatrix(list(table.sample_ids), out, cfg.precision)


# --------------------------------------------------------------- embedding
@dataclass
class EmbeddingBatch:
    """EmbeddingBatch<Real> (embed.hpp:19-26)."""

    emb: np.ndarray
    lengths: np.ndarray
    filled: int = 0
    n_samples: int = 0
    n_samples_padded: int = 0


class EmbedMode(enum.IntEnum):
    Unweighted = 0
    Weighted = 1


def embed_mode(m: Metric) -> EmbedMode:
    return EmbedMode.Unweighted if m == Metric.Unweighted else EmbedMode.Weighted


def sheared_to_table(tree: PhyloTree, table: SampleTable) -> PhyloTree:
    """sheared_to_table (embed.cpp:8-15), as a PhyloTree over the flattened rows."""
    leaves = set(tree.leaf_names)
    for f in table.feature_ids:
        if f not in leaves:
            raise Error(f"table feature '{f}' is not a leaf of the tree")
    if table.n_features() == tree.n_leaves:
        return tree
    return shear(tree, table.feature_ids)


def shear(tree: PhyloTree, keep: Sequence[str]) -> PhyloTree:
    """shear (newick.cpp:311-331): restrict to `keep`, fold unary chains."""
    if not keep:
        raise Error("shear: leaf set is empty")
    have = set(tree.leaf_names)
    want = list(dict.fromkeys(keep))
    for nm in want:
        if nm not in have:
            raise Error(f"shear: '{nm}' is not a leaf of the tree")
    names = tree.names
    index = {names[i]: i for i in range(tree.n_nodes) if not tree.children[i]}
    fleaf = np.array([index[nm] for nm in want], dtype=np.int32)
    nn = tree.n_nodes
    parent_row = np.empty(nn, dtype=np.int32)
    lengths = np.empty(nn, dtype=np.float64)
    leaf_feature = np.empty(nn, dtype=np.int32)
    n_rows = C.c_int32(0)
    _call(N.lib().sfh_flatten(nn, N.ptr(tree.parent), N.ptr(tree.length), len(fleaf), N.ptr(fleaf),
                              C.byref(n_rows), N.ptr(parent_row), N.ptr(lengths), N.ptr(leaf_feature)))
    E = n_rows.value
    # rows -> a tree with the root appended as node E
    par = np.where(parent_row[:E] < 0, E, parent_row[:E]).astype(np.int32)
    parent = np.concatenate([par, np.array([-1], np.int32)])
    length = np.concatenate([lengths[:E], np.array([0.0])])
    nm = [want[f] if f >= 0 else "" for f in leaf_feature[:E].tolist()] + [""]
    return PhyloTree(parent, length, nm)


class Embedder:
    """Embedder (embed.hpp:45-67): postorder row cursor. Rows are built on the
    device by K1 (sf_embed_rows) and handed out in batches."""

    def __init__(self, tree: PhyloTree, table: SampleTable, mode: EmbedMode, pad_multiple: int = 1):
        if pad_multiple < 1:
            raise Error("pad multiple must be >= 1")
        if table.n_features() != tree.n_leaves:
            raise Error("tree leaves and table features differ; shear the tree first")
        leaves = set(tree.leaf_names)
        for f in table.feature_ids:
            if f not in leaves:
                raise Error(f"tree leaf '{f}' is not a table feature; shear the tree first")
        self._n = table.n_samples()
        self._padded = -(-self._n // pad_multiple) * pad_multiple
        self._problem = flatten(tree, table)
        self._mode = mode
        self._rows: Optional[np.ndarray] = None
        self._cursor = 0

    def total_rows(self) -> int:
        return self._problem.n_rows

    def rows_emitted(self) -> int:
        return self._cursor

    def n_samples(self) -> int:
        return self._n

    def n_samples_padded(self) -> int:
        return self._padded

    def _materialise(self, device: int = 0) -> None:
        E = self._problem.n_rows
        out = np.zeros((E, self._padded), dtype=np.float64)
        _call(N.lib().sf_embed_rows(self._problem.ref, int(self._mode == EmbedMode.Weighted), 0, E,
                                    N.ptr(out), self._padded, device))
        self._rows = out

    def next_batch(self, capacity: int) -> Optional[EmbeddingBatch]:
        if capacity < 1:
            raise Error("batch capacity must be >= 1")
        E = self._problem.n_rows
        if self._cursor >= E:
            return None
        if self._rows is None:
            self._materialise()
        take = min(capacity, E - self._cursor)
        a, b = self._cursor, self._cursor + take
        self._cursor = b
        return EmbeddingBatch(self._rows[a:b].copy(), self._problem.lengths[a:b].copy(), take,
                              self._n, self._padded)


def cast_batch(b: EmbeddingBatch, real) -> EmbeddingBatch:
    """cast_batch<Real> (embed.hpp:71-84): one rounding of rows and lengths."""
    if np.dtype(real) == np.float64:
        return b
    return EmbeddingBatch(b.emb.astype(np.float32), b.lengths.astype(np.float32), b.filled,
                          b.n_samples, b.n_samples_padded)


def accumulate(sset: StripeSet, batch: EmbeddingBatch, cfg: KernelConfig,
               counters: KernelCounters, device: int = 0) -> None:
    """accumulate (kernels.hpp:232-248): fold one batch into the set on device."""
    if sset.finalized:
        raise Error("cannot accumulate into a finalized stripe set")
    if batch.filled < 1:
        raise Error("embedding batch is empty")
    if batch.n_samples != sset.n_samples:
        raise Error("batch and stripe set disagree on the sample count")
    if batch.emb.ndim != 2 or batch.emb.shape[0] < batch.filled or batch.emb.shape[1] != batch.n_samples_padded:
        raise Error("embedding batch shape is inconsistent")
    if cfg.metric != sset.metric:
        raise Error("kernel metric does not match the stripe set")
    if cfg.variant == Variant.Tiled and batch.n_samples_padded % cfg.resolved_step_size() != 0:
        raise Error("batch padding is not a multiple of the step size")
    dt = sset.distances.dtype
    emb = np.ascontiguousarray(batch.emb[:batch.filled], dtype=dt)
    lens = np.ascontiguousarray(batch.lengths[:batch.filled], dtype=dt)
    prec = Precision.Fp32 if dt == np.float32 else Precision.Fp64
    tot_ptr = N.ptr(sset.totals) if sset.has_totals() else None
    _call(N.lib().sf_accumulate_batch(N.ptr(emb), N.ptr(lens), batch.filled, sset.n_samples,
                                      batch.n_samples_padded, int(sset.metric), int(prec),
                                      sset.start, sset.stop, N.ptr(sset.distances), tot_ptr, device))
    counters.kernel_passes += 1
    entries = sset.n_stripes() * sset.n_samples
    counters.accumulator_writes += (batch.filled if cfg.variant == Variant.Naive else 1) * entries
    counters.embedding_reads += 2 * batch.filled * entries


def finalize(sset: StripeSet, device: int = 0) -> None:
    """finalize (kernels.hpp:251-259), on device."""
    if sset.finalized:
        raise Error("stripe set was already finalized")
    if sset.has_totals():
        prec = sset.precision
        _call(N.lib().sf_finalize(int(prec), sset.distances.size, N.ptr(sset.distances),
                                  N.ptr(sset.totals), device))
    sset.finalized = True


def condense(parts: Sequence[StripeSet], sample_ids: Optional[Sequence[str]] = None,
             device: int = 0) -> DistanceMatrix:
    """condense (stripes.cpp:68-129): validation on host, scatter on device."""
    if not parts:
        raise Error("condense: no stripe sets given")
    n = parts[0].n_samples
    metric = parts[0].metric
    S = total_stripes(n)
    for p in parts:
        if p.n_samples != n:
            raise Error("condense: sample counts differ")
        if p.metric != metric:
            raise Error("condense: metrics differ")
        if not p.finalized:
            raise Error("condense: stripe set was not finalized")
    order = sorted(parts, key=lambda p: p.start)
    cursor = 0
    for p in order:
        if p.start > cursor:
            raise Error(f"condense: stripe ranges leave a gap at [{cursor},{p.start})")
        if p.start < cursor:
            raise Error(f"condense: stripe ranges overlap at [{p.start},{cursor})")
        cursor = p.stop
    if cursor != S:
        raise Error(f"condense: stripe ranges leave a gap at [{cursor},{S})")
    if sample_ids:
        if len(sample_ids) != n:
            raise Error("condense: sample id count does not match the matrix")
        ids = list(sample_ids)
    else:
        ids = [str(i) for i in range(n)]
    out = np.zeros((n, n), dtype=np.float64)
    prec = order[0].precision
    for p in order:
        d = np.ascontiguousarray(p.distances, dtype=_dtype(prec))
        st = N.lib().sf_condense(int(prec), n, p.start, p.stop, N.ptr(d), N.ptr(out), device)
        if st != N.SF_OK:
            msg = N.lib().sf_last_error().decode()
            if "duplicated" in msg:
                raise Error("condense: duplicated slot disagrees")
            raise Error(msg)
    return DistanceMatrix(ids, out, prec)


# ----------------------------------------------------------------- strf files
_MAGIC = b"STRF"


def fnv1a64(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    """fnv1a64 (common.cpp:50-57), vectorised over bytes."""
    arr = np.frombuffer(data, dtype=np.uint8)
    prime = 0x100000001B3
    for b in arr.tolist():
        h ^= b
        h = (h * prime) & 0xFFFFFFFFFFFFFFFF
    return h


def _fnv_fast(data: bytes) -> int:
    buf = C.create_string_buffer(data, len(data)) if data else C.create_string_buffer(1)
    return int(N.lib().sfh_fnv1a64(C.cast(buf, C.c_void_p), len(data), 0xCBF29CE484222325))


def write_stripe_file(path: str, sset: StripeSet) -> None:
    """write_stripe_file (stripes.cpp:179-201): 32-byte header, payload, FNV-1a."""
    if not sset.finalized:
        raise Error("refusing to write an unfinalized stripe set")
    w = sset.distances.dtype.itemsize
    header = _MAGIC + bytes([1, w, int(sset.metric), 0]) + struct.pack(
        "<QQQ", sset.n_samples, sset.start, sset.stop)
    payload = np.ascontiguousarray(sset.distances).tobytes()
    if sset.has_totals():
        payload += np.ascontiguousarray(sset.totals).tobytes()
    try:
        with open(path, "wb") as fh:
            fh.write(header + payload + struct.pack("<Q", _fnv_fast(payload)))
    except OSError:
        raise Error(f"cannot open '{path}' for writing") from None


def read_stripe_file(path: str) -> StripeSet:
    """read_stripe_file (stripes.cpp:237-274)."""
    try:
        with open(path, "rb") as fh:
            blob = fh.read()
    except OSError:
        raise Error(f"cannot open '{path}'") from None
    if len(blob) < 32 + 8:
        raise Error(f"{path}: truncated stripe file")
    if blob[:4] != _MAGIC:
        raise Error(f"{path}: not a stripe file (bad magic)")
    if blob[4] != 1:
        raise Error(f"{path}: unsupported version {blob[4]}")
    w = blob[5]
    if w not in (4, 8):
        raise Error(f"{path}: unsupported precision byte {w}")
    if blob[6] not in (1, 2, 3):
        raise Error(f"{path}: unknown metric code {blob[6]}")
    metric = Metric(blob[6])
    n, start, stop = struct.unpack("<QQQ", blob[8:32])
    if n < 2:
        raise Error(f"{path}: sample count {n} is invalid")
    if stop <= start or stop > n // 2:
        raise Error(f"{path}: stripe range {start}:{stop} is invalid")
    payload = blob[32:-8]
    (stored,) = struct.unpack("<Q", blob[-8:])
    if _fnv_fast(payload) != stored:
        raise Error(f"{path}: checksum mismatch, file is corrupt")
    rows = stop - start
    plane = rows * n * w
    want = 2 * plane if metric_has_totals(metric) else plane
    if len(payload) != want:
        raise Error(f"{path}: payload is {len(payload)} bytes, expected {want}")
    dt = np.float32 if w == 4 else np.float64
    d = np.frombuffer(payload[:plane], dtype=dt).reshape(rows, n).copy()
    t = (np.frombuffer(payload[plane:], dtype=dt).reshape(rows, n).copy()
         if metric_has_totals(metric) else np.zeros((0, 0), dt))
    return StripeSet(int(n), int(start), int(stop), metric, d, t, finalized=True)


def merge_stripe_files(paths: Sequence[str], sample_ids: Optional[Sequence[str]] = None) -> DistanceMatrix:
    """merge_stripe_files (stripes.cpp:276-297)."""
    if not paths:
        raise Error("merge: no input files")
    loaded = [read_stripe_file(p) for p in paths]
    fp32 = loaded[0].distances.dtype == np.float32
    for p, s in zip(paths[1:], loaded[1:]):
        if (s.distances.dtype == np.float32) != fp32:
            raise Error(f"merge: '{p}' has a different precision than '{paths[0]}'")
    return condense(loaded, sample_ids)


# ------------------------------------------------------------------ matrix TSV
def _fmt_g(v: float, digits: int) -> str:
    return "%.*g" % (digits, v)


def to_tsv(dm: DistanceMatrix) -> str:
    """to_tsv (stripes.cpp:311-332): %.17g for fp64, %.9g for fp32."""
    n = dm.n()
    if len(dm.sample_ids) != n:
        raise Error(f"distance matrix has {len(dm.sample_ids)} ids for {n} samples")
    digits = 9 if dm.precision == Precision.Fp32 else 17
    out = ["\t".join(dm.sample_ids), "\n"]
    for i in range(n):
        out.append(dm.sample_ids[i])
        for v in dm.values[i].tolist():
            out.append("\t")
            out.append(_fmt_g(v, digits))
        out.append("\n")
    return "".join(out)


def write_tsv(path: str, dm: DistanceMatrix, threads: int = 0) -> None:
    """write_tsv (stripes.cpp:334-340) through the native parallel writer
    (sfh_write_tsv): the same bytes as to_tsv, formatted by `threads` host
    threads (0 = all)."""
    n = dm.n()
    if len(dm.sample_ids) != n:
        raise Error(f"distance matrix has {len(dm.sample_ids)} ids for {n} samples")
    digits = 9 if dm.precision == Precision.Fp32 else 17
    ids = (C.c_char_p * max(n, 1))(*[s.encode() for s in dm.sample_ids])
    vals = np.ascontiguousarray(dm.values, dtype=np.float64)
    _call(N.lib().sfh_write_tsv(str(path).encode(), n, ids, N.ptr(vals), digits, int(threads)))


def read_tsv_file(path: str) -> DistanceMatrix:
    """read_tsv_file (stripes.cpp:342-398)."""
    try:
        with open(path, "r", encoding="utf-8", newline="") as fh:
            lines = [ln[:-1] if ln.endswith("\r") else ln for ln in fh.read().split("\n")]
    except OSError:
        raise Error(f"cannot open '{path}'") from None
    if not lines or (len(lines) == 1 and lines[0] == ""):
        raise Error(f"{path}: empty matrix file")
    ids = lines[0].split("\t")
    n = len(ids)
    vals = np.zeros((n, n))
    for i in range(n):
        if i + 1 >= len(lines) or (lines[i + 1] == "" and i + 2 >= len(lines)):
            raise Error(f"{path}: expected {n} matrix rows")
        cells = lines[i + 1].split("\t")
        if cells[0] != ids[i]:
            raise Error(f"{path}: row {i + 1} id '{cells[0]}' does not match the header order")
        if len(cells) - 1 > n:
            raise Error(f"{path}: row {i + 1} is too wide")
        if len(cells) - 1 != n:
            raise Error(f"{path}: row {i + 1} has {len(cells) - 1} values, expected {n}")
        try:
            vals[i] = [float(c) for c in cells[1:]]
        except ValueError:
            raise Error(f"{path}: bad value in row {i + 1}") from None
    return DistanceMatrix(ids, vals)


# ---------------------------------------------------------------- validation
def condensed_upper(dm: DistanceMatrix) -> np.ndarray:
    """condensed_upper (validate.cpp:83-97)."""
    n = dm.n()
    if dm.values.shape[1] != n:
        raise Error("distance matrix is not square")
    if n < 2:
        raise Error("distance matrix needs at least 2 samples")
    v = dm.values
    iu = np.triu_indices(n, 1)
    if np.any(np.abs(v[iu] - v.T[iu]) > 1e-12):
        raise Error("distance matrix is asymmetric")
    return v[iu].copy()


@dataclass
class MantelResult:
    """MantelResult (validate.hpp:25-31)."""

    r: float = 0.0
    r_squared: float = 0.0
    p_value: float = 1.0
    permutations: int = 0
    seed: int = 0

    def __getitem__(self, key):  # dict-style access kept for callers of the old mirror
        return getattr(self, key)


def mantel(m1: DistanceMatrix, m2: DistanceMatrix, permutations: int = 999, seed: int = 1,
           device: int = 0) -> MantelResult:
    """mantel (validate.cpp:111-159) on device through sf_mantel: the
    reference's r and its permutation stream (mt19937_64 + std::shuffle from
    splitmix64 seeds), so p-values match the reference draw for draw."""
    if permutations < 1:
        raise Error("mantel: need at least 1 permutation")
    if m1.n() != m2.n():
        raise Error("mantel: matrices have different sizes")
    if m1.sample_ids and m2.sample_ids and list(m1.sample_ids) != list(m2.sample_ids):
        raise Error("mantel: matrices have different sample orderings")
    n = m1.n()
    x = np.ascontiguousarray(m1.values, dtype=np.float64)
    y = np.ascontiguousarray(m2.values, dtype=np.float64)
    if x.shape != (n, n) or y.shape != (n, n):
        raise Error("distance matrix is not square")
    r = C.c_double()
    p = C.c_double()
    _call(N.lib().sf_mantel(n, N.ptr(x), N.ptr(y), int(permutations), int(seed) & (2**64 - 1),
                            int(device), C.byref(r), C.byref(p)))
    return MantelResult(r.value, r.value * r.value, p.value, int(permutations), int(seed))


def mantel_permutation(n: int, seed: int, p: int) -> np.ndarray:
    """Permutation p of the reference's Mantel stream (host-only helper)."""
    out = np.empty(n, np.int32)
    _call(N.lib().sf_mantel_permutation(int(n), int(seed) & (2**64 - 1), int(p), N.ptr(out)))
    return out
