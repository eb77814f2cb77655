"""ctypes binding of the C ABI (include/stripefrac_cuda.h, include/stripefrac_host.h).

The shared object is built in-tree (``paper_2005_05826_b200/libstripefrac_cuda.so``)
by ``__graft_entry__.build()``. There is no fallback: if it is missing, loading
fails loudly.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

import os

LIB_PATH = Path(__file__).resolve().parent / "libstripefrac_cuda.so"
# A/B only: SF_LIB names an alternative build of the same library (tools/build_ab.sh)
if os.environ.get("SF_LIB"):
    LIB_PATH = Path(os.environ["SF_LIB"]).resolve()

SF_OK, SF_EINVAL, SF_ENOMEM, SF_ECUDA, SF_ESTATE = 0, 1, 2, 3, 4
SF_UNWEIGHTED, SF_WEIGHTED_UNNORMALIZED, SF_WEIGHTED_NORMALIZED = 1, 2, 3
SF_GENERALIZED = 4  # extension: generalized UniFrac (sf_exec.alpha); not in the reference
SF_FP32, SF_FP64 = 4, 8
SF_EXEC_EXACT_NO_FMA = 1
KERNEL_AUTO, KERNEL_DENSE, KERNEL_SPARSE = 0, 1, 2  # auto, dense tiled (every metric), bitwise union walk (UW)
KERNEL_SPLIT = 10  # unweighted: heavy walk + light scatter, exact fixed-point sums (the default)
KERNEL_WSPARSE = 11  # weighted metrics: present-row walk (bitwise; the exact-mode default)
KERNEL_WUWALK = 12  # weighted metrics: warp-uniform u-walk + double-double remainder
KERNEL_WSPLIT = 13  # weighted / generalized: dense heavy rows (FP64) + exact fixed-point light scatter (the default)


class sf_problem(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int32),
        ("parent_row", C.POINTER(C.c_int32)),
        ("lengths", C.POINTER(C.c_double)),
        ("leaf_feature", C.POINTER(C.c_int32)),
        ("n_samples", C.c_int32),
        ("n_features", C.c_int32),
        ("feat_ptr", C.POINTER(C.c_int64)),
        ("sample_idx", C.POINTER(C.c_int32)),
        ("counts", C.POINTER(C.c_double)),
        ("sample_totals", C.POINTER(C.c_double)),
    ]


class sf_exec(C.Structure):
    _fields_ = [
        ("n_devices", C.c_int32),
        ("devices", C.POINTER(C.c_int32)),
        ("mem_budget_bytes", C.c_int64),
        ("kernel", C.c_int32),
        ("flags", C.c_int32),
        ("alpha", C.c_double),  # SF_GENERALIZED only (ABI v3)
    ]


class sf_stats(C.Structure):
    _fields_ = [
        ("updates_alg", C.c_uint64),
        ("updates_exec", C.c_uint64),
        ("launches", C.c_uint64),
        ("n_chunks", C.c_uint64),
        ("embed_ms", C.c_double),
        ("stripe_ms", C.c_double),
        ("finalize_ms", C.c_double),
        ("total_ms", C.c_double),
        ("fp64_ops", C.c_uint64),
        ("tensor_ops", C.c_uint64),
        ("tensor_ms", C.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


# every exported symbol of the two public headers, with its signature
_P = C.c_void_p
SIGNATURES = {
    "sf_last_error": (C.c_char_p, []),
    "sf_version": (C.c_char_p, []),
    "sf_device_count": (C.c_int32, []),
    "sf_compute_stripes": (C.c_int, [C.POINTER(sf_problem), C.c_int, C.c_int, C.c_int32, C.c_int32,
                                     _P, _P, C.c_int32, C.POINTER(sf_exec), C.POINTER(sf_stats)]),
    "sf_plan_create": (C.c_int, [C.POINTER(sf_problem), C.c_int, C.c_int, C.c_int32, C.c_int32,
                                 C.POINTER(sf_exec), C.POINTER(_P)]),
    "sf_plan_condense": (C.c_int, [_P, _P]),
    "sf_compute_distance_matrix": (C.c_int, [C.POINTER(sf_problem), C.c_int, C.c_int, _P, C.POINTER(sf_exec),
                                             C.POINTER(sf_stats)]),
    "sf_trim_memory": (C.c_int, [C.c_int32]),
    "sf_plan_run": (C.c_int, [_P, C.c_int32]),
    "sf_plan_sync": (C.c_int, [_P]),
    "sf_plan_download": (C.c_int, [_P, _P, _P]),
    "sf_plan_stats": (C.c_int, [_P, C.POINTER(sf_stats)]),
    "sf_plan_destroy": (None, [_P]),
    "sf_plan_write_strf": (C.c_int, [_P, C.c_char_p]),
    "sf_accumulate_batch": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int, C.c_int,
                                      C.c_int32, C.c_int32, _P, _P, C.c_int32]),
    "sf_embed_rows": (C.c_int, [C.POINTER(sf_problem), C.c_int32, C.c_int32, C.c_int32, _P,
                                C.c_int32, C.c_int32]),
    "sf_finalize": (C.c_int, [C.c_int, C.c_int64, _P, _P, C.c_int32]),
    "sf_condense": (C.c_int, [C.c_int, C.c_int32, C.c_int32, C.c_int32, _P, _P, C.c_int32]),
    "sf_mantel": (C.c_int, [C.c_int32, _P, _P, C.c_int32, C.c_uint64, C.c_int32,
                            C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "sf_mantel_permutation": (C.c_int, [C.c_int32, C.c_uint64, C.c_int32, _P]),
    "sfh_flatten": (C.c_int, [C.c_int32, _P, _P, C.c_int32, _P, C.POINTER(C.c_int32), _P, _P, _P]),
    "sfh_fnv1a64": (C.c_uint64, [_P, C.c_uint64, C.c_uint64]),
    "sfh_write_tsv": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_char_p), _P, C.c_int32, C.c_int32]),
    "sfh_load_table_sparse": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(_P)]),
    "sfh_table_free": (None, [_P]),
    "sfh_table_n_samples": (C.c_int32, [_P]),
    "sfh_table_n_features": (C.c_int32, [_P]),
    "sfh_table_nnz": (C.c_int64, [_P]),
    "sfh_table_sample_id": (C.c_char_p, [_P, C.c_int32]),
    "sfh_table_feature_id": (C.c_char_p, [_P, C.c_int32]),
    "sfh_table_feat_ptr": (C.POINTER(C.c_int64), [_P]),
    "sfh_table_sample_idx": (C.POINTER(C.c_int32), [_P]),
    "sfh_table_counts": (C.POINTER(C.c_double), [_P]),
    "sfh_table_sample_totals": (C.POINTER(C.c_double), [_P]),
    "sfh_random_instance": (_P, [C.c_uint64, C.c_int32, C.c_int32, C.c_double, C.c_int32]),
    "sfh_instance_free": (None, [_P]),
    "sfh_instance_n_nodes": (C.c_int32, [_P]),
    "sfh_instance_n_samples": (C.c_int32, [_P]),
    "sfh_instance_n_features": (C.c_int32, [_P]),
    "sfh_instance_nnz": (C.c_int64, [_P]),
    "sfh_instance_parent": (_P, [_P]),
    "sfh_instance_length": (_P, [_P]),
    "sfh_instance_feature_leaf": (_P, [_P]),
    "sfh_instance_feat_ptr": (_P, [_P]),
    "sfh_instance_sample_idx": (_P, [_P]),
    "sfh_instance_counts": (_P, [_P]),
    "sfh_instance_sample_totals": (_P, [_P]),
}

_lib = None


class NativeError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def lib() -> C.CDLL:
    """Load the in-tree CUDA library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != SF_OK:
        msg = lib().sf_last_error().decode("utf-8", "replace")
        raise NativeError(status, msg)


def ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def typed_ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class Problem:
    """Owns the numpy arrays behind an sf_problem (keeps them alive)."""

    def __init__(self, parent_row, lengths, leaf_feature, n_samples, feat_ptr, sample_idx,
                 counts, sample_totals):
        self.parent_row = np.ascontiguousarray(parent_row, dtype=np.int32)
        self.lengths = np.ascontiguousarray(lengths, dtype=np.float64)
        self.leaf_feature = np.ascontiguousarray(leaf_feature, dtype=np.int32)
        self.feat_ptr = np.ascontiguousarray(feat_ptr, dtype=np.int64)
        self.sample_idx = np.ascontiguousarray(sample_idx, dtype=np.int32)
        self.counts = np.ascontiguousarray(counts, dtype=np.float64)
        self.sample_totals = np.ascontiguousarray(sample_totals, dtype=np.float64)
        self.n_samples = int(n_samples)
        self.n_rows = int(self.parent_row.shape[0])
        self.n_features = int(self.feat_ptr.shape[0] - 1)
        self.struct = sf_problem(
            self.n_rows, typed_ptr(self.parent_row, C.c_int32), typed_ptr(self.lengths, C.c_double),
            typed_ptr(self.leaf_feature, C.c_int32), self.n_samples, self.n_features,
            typed_ptr(self.feat_ptr, C.c_int64), typed_ptr(self.sample_idx, C.c_int32),
            typed_ptr(self.counts, C.c_double), typed_ptr(self.sample_totals, C.c_double))

    @property
    def ref(self):
        return C.byref(self.struct)

    @property
    def nnz(self) -> int:
        return int(self.feat_ptr[-1])


def make_exec(devices=None, kernel: int = KERNEL_AUTO, exact: bool = False,
              mem_budget_bytes: int = 0, alpha: float = 1.0):
    """Build an sf_exec (returned with its device array to keep it alive)."""
    dev_arr = None
    if devices is not None:
        dev_arr = (C.c_int32 * len(devices))(*devices)
    ex = sf_exec(len(devices) if devices is not None else 0,
                 C.cast(dev_arr, C.POINTER(C.c_int32)) if dev_arr is not None else None,
                 int(mem_budget_bytes), int(kernel), SF_EXEC_EXACT_NO_FMA if exact else 0,
                 float(alpha))
    return ex, dev_arr
