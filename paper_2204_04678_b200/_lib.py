"""ctypes binding of the C-ABI in include/pinla.h (libpinla.so, in-tree).

There is deliberately no CPU fallback: if the shared library is missing or
no CUDA device is visible, every product entry point raises
:class:`~.errors.EngineError`.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import EngineError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpinla.so")

c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_dp = ctypes.POINTER(ctypes.c_double)


class PinlaModel(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("m", ctypes.c_int64),
        ("d", ctypes.c_int32),
        ("family", ctypes.c_int32),
        ("noise_theta", ctypes.c_int32),
        ("noise_precision", ctypes.c_double),
        ("p_indptr", c_i64p),
        ("p_indices", c_i64p),
        ("n_terms", ctypes.c_int64),
        ("term_entry", c_i64p),
        ("term_gain", c_i32p),
        ("term_coef", c_dp),
        ("p_const", c_dp),
        ("n_gains", ctypes.c_int32),
        ("gain_kind", c_i32p),
        ("gain_theta", c_i32p),
        ("gain_sub", c_i32p),
        ("a_indptr", c_i64p),
        ("a_indices", c_i64p),
        ("a_data", c_dp),
        ("y", c_dp),
        ("offsets", c_dp),
        ("exposures", c_dp),
        ("hyper_shape", c_dp),
        ("hyper_rate", c_dp),
        ("perm", c_i64p),
        ("n_dense", ctypes.c_int64),
        ("tile_bounds", c_i64p),
        ("n_tile_bounds", ctypes.c_int64),
        ("n_logdet_terms", ctypes.c_int32),
        ("ld_kind", c_i32p),
        ("ld_theta", c_i32p),
        ("ld_dims", c_i64p),
        ("ld_value", c_dp),
    ]


class PinlaOptions(ctypes.Structure):
    _fields_ = [
        ("max_slots", ctypes.c_int32),
        ("max_inner", ctypes.c_int32),
        ("inner_tol", ctypes.c_double),
        ("device", ctypes.c_int32),
        ("selinv_slots", ctypes.c_int32),
        ("analytic_prior_logdet", ctypes.c_int32),
    ]


class PinlaStats(ctypes.Structure):
    _fields_ = [
        ("n_evaluations", ctypes.c_int64),
        ("n_factorizations", ctypes.c_int64),
        ("n_solves", ctypes.c_int64),
        ("n_selinv", ctypes.c_int64),
        ("nnz_cond", ctypes.c_int64),
        ("n_tiles", ctypes.c_int64),
        ("n_tile_rows", ctypes.c_int64),
        ("factor_flops", ctypes.c_int64),
        ("selinv_flops", ctypes.c_int64),
        ("solve_bytes", ctypes.c_int64),
        ("assemble_bytes", ctypes.c_int64),
        ("device_bytes", ctypes.c_int64),
        ("analyze_s", ctypes.c_double),
        ("kernel_launches", ctypes.c_int64),
        ("factor_launches", ctypes.c_int64),
        ("factor_slot_runs", ctypes.c_int64),
        ("solve_slot_runs", ctypes.c_int64),
        ("factor_ms", ctypes.c_double),
        ("solve_ms", ctypes.c_double),
        ("assemble_ms", ctypes.c_double),
        ("selinv_ms", ctypes.c_double),
        ("last_call_ms", ctypes.c_double),
        ("factor_flops_limited", ctypes.c_int64),
        ("slots", ctypes.c_int64),
        ("solve_kernel_ms", ctypes.c_double),
        ("assemble_bytes_done", ctypes.c_int64),
        ("selinv_launches", ctypes.c_int64),
    ]


EXPORTS = (
    "pinla_create", "pinla_destroy", "pinla_eval_batch", "pinla_eval_batch_warm", "pinla_mode",
    "pinla_selinv_diag",
    "pinla_factor_logdet", "pinla_cond_pattern", "pinla_stats", "pinla_reset_stats",
    "pinla_phase_times", "pinla_last_error", "pinla_version", "pinla_solve_resident",
    "pinla_selinv_resident", "pinla_analyze_pattern", "pinla_nd_order", "pinla_scalar_pattern",
    "pinla_tile_entries", "pinla_cond_values", "pinla_factor_lmul",
)


class PinlaAnalysisInfo(ctypes.Structure):
    _fields_ = [
        ("n_tile_rows", ctypes.c_int64),
        ("n_tiles", ctypes.c_int64),
        ("n_update_pairs", ctypes.c_int64),
        ("factor_flops", ctypes.c_int64),
        ("selinv_flops", ctypes.c_int64),
        ("solve_bytes", ctypes.c_int64),
        ("depth_forward", ctypes.c_int64),
        ("depth_backward", ctypes.c_int64),
        ("factor_flops_limited", ctypes.c_int64),
    ]

_lib = None


def load(path: str = LIB_PATH):
    """Load libpinla.so (raises EngineError when it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise EngineError(
            f"{path} is missing: build it with `make -C paper_2204_04678_b200/csrc` "
            "(there is no CPU fallback)"
        )
    L = ctypes.CDLL(path)
    P = ctypes.c_void_p
    L.pinla_create.argtypes = [ctypes.POINTER(PinlaModel), ctypes.POINTER(PinlaOptions),
                               ctypes.POINTER(P)]
    L.pinla_destroy.argtypes = [P]
    L.pinla_destroy.restype = None
    L.pinla_eval_batch.argtypes = [P, ctypes.c_int32, c_dp, c_dp, c_dp, c_dp, c_i32p, c_i64p,
                                   c_i32p, c_dp, c_dp]
    L.pinla_eval_batch_warm.argtypes = [P, ctypes.c_int32, c_dp, c_dp, c_dp, c_dp, c_i32p, c_i64p,
                                        c_i32p, c_dp, c_dp]
    L.pinla_mode.argtypes = [P, c_dp, c_dp, c_dp, c_i32p, c_i32p, c_i64p, c_dp]
    L.pinla_selinv_diag.argtypes = [P, c_dp, c_dp, c_dp, c_dp, c_i32p, c_i64p]
    L.pinla_factor_logdet.argtypes = [P, c_dp, c_dp, c_i32p, c_i64p]
    L.pinla_solve_resident.argtypes = [P, c_dp, c_dp]
    L.pinla_selinv_resident.argtypes = [P, c_dp]
    L.pinla_analyze_pattern.argtypes = [ctypes.c_int64, c_i64p, c_i64p, c_i64p, ctypes.c_int64,
                                        c_i64p, ctypes.c_int64,
                                        ctypes.POINTER(PinlaAnalysisInfo), c_i32p, c_i32p]
    L.pinla_nd_order.argtypes = [ctypes.c_int64, c_i64p, c_i64p, ctypes.c_int64, ctypes.c_int64,
                                 c_i64p, c_i64p, c_i64p, c_i64p, c_i64p, c_i64p, c_i64p, c_i64p]
    L.pinla_scalar_pattern.argtypes = [ctypes.c_int64, c_i64p, c_i64p, c_i64p, c_i64p, c_i64p,
                                       c_i64p]
    L.pinla_tile_entries.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, c_i64p,
                                     c_i64p, c_dp]
    L.pinla_cond_values.argtypes = [P, ctypes.c_int32, c_dp]
    L.pinla_factor_lmul.argtypes = [P, ctypes.c_int32, c_dp, c_dp]
    L.pinla_cond_pattern.argtypes = [P, c_i64p, c_i64p, c_i64p]
    L.pinla_stats.argtypes = [P, ctypes.POINTER(PinlaStats)]
    L.pinla_reset_stats.argtypes = [P]
    L.pinla_reset_stats.restype = None
    L.pinla_phase_times.argtypes = [P, c_dp, c_dp, c_dp, c_dp, c_dp]
    L.pinla_last_error.restype = ctypes.c_char_p
    L.pinla_version.restype = ctypes.c_char_p
    _lib = L
    return L


def check(rc: int):
    if rc != 0:
        raise EngineError(load().pinla_last_error().decode())


def ptr(a: np.ndarray | None, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def analyze_pattern(indptr, indices, perm, n_dense=0, tile_bounds=None, want_tiles=False):
    """Host-only tile symbolic analysis (no GPU): dict of structure numbers
    (+ tile coordinates of L when ``want_tiles``)."""
    L = load()
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int64)
    pm = np.ascontiguousarray(perm, dtype=np.int64)
    tb = None if tile_bounds is None else np.ascontiguousarray(tile_bounds, dtype=np.int64)
    info = PinlaAnalysisInfo()
    args = [ctypes.c_int64(ip.size - 1), ptr(ip, ctypes.c_int64), ptr(ix, ctypes.c_int64),
            ptr(pm, ctypes.c_int64), ctypes.c_int64(n_dense), ptr(tb, ctypes.c_int64),
            ctypes.c_int64(0 if tb is None else tb.size), ctypes.byref(info)]
    check(L.pinla_analyze_pattern(*args, None, None))
    out = {name: getattr(info, name) for name, _ in info._fields_}
    if want_tiles:
        r = np.empty(info.n_tiles, dtype=np.int32)
        c = np.empty(info.n_tiles, dtype=np.int32)
        check(L.pinla_analyze_pattern(*args, ptr(r, ctypes.c_int32), ptr(c, ctypes.c_int32)))
        out["tile_rows"], out["tile_cols"] = r, c
    return out


def nd_order(indptr, indices, leaf_cutoff: int = 64, tile_max: int = 64, want_tree: bool = False):
    """Native nested dissection of a lower-CSC pattern (host only, no GPU):
    (perm new -> old, n_dense, separator-aligned tile bounds[, tree]) —
    the reference's nested_dissection_order (ordering.py:206-274)."""
    L = load()
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int64)
    n = ip.size - 1
    perm = np.empty(n, dtype=np.int64)
    bounds = np.empty(n + 2, dtype=np.int64)
    nb = ctypes.c_int64()
    nd = ctypes.c_int64()
    nn = ctypes.c_int64()
    ns = np.empty(n + 1, dtype=np.int64)
    ne = np.empty(n + 1, dtype=np.int64)
    npar = np.empty(n + 1, dtype=np.int64)
    T = ctypes.c_int64
    check(L.pinla_nd_order(T(n), ptr(ip, T), ptr(ix, T), T(leaf_cutoff), T(tile_max),
                           ptr(perm, T), ctypes.byref(nd), ptr(bounds, T), ctypes.byref(nb),
                           ptr(ns, T) if want_tree else None, ptr(ne, T) if want_tree else None,
                           ptr(npar, T) if want_tree else None, ctypes.byref(nn)))
    out = (perm, int(nd.value), bounds[: nb.value].copy())
    if want_tree:
        k = nn.value
        out = out + ((ns[:k].copy(), ne[:k].copy(), npar[:k].copy()),)
    return out


def scalar_pattern(indptr, indices, perm):
    """Scalar L pattern (Lp, Li) of a lower-CSC pattern under perm (host)."""
    L = load()
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int64)
    pm = np.ascontiguousarray(perm, dtype=np.int64)
    n = ip.size - 1
    T = ctypes.c_int64
    nnz = ctypes.c_int64()
    check(L.pinla_scalar_pattern(T(n), ptr(ip, T), ptr(ix, T), ptr(pm, T), ctypes.byref(nnz),
                                 None, None))
    Lp = np.empty(n + 1, dtype=np.int64)
    Li = np.empty(nnz.value, dtype=np.int64)
    check(L.pinla_scalar_pattern(T(n), ptr(ip, T), ptr(ix, T), ptr(pm, T), ctypes.byref(nnz),
                                 ptr(Lp, T), ptr(Li, T)))
    return Lp, Li
