"""Python wrapper around one libpinla handle (device-resident model).

Converts a :class:`~.model.ModelSpec` + data into the plain-pointer
``pinla_model`` struct of include/pinla.h, owns the handle, and exposes the
batched calls as numpy-in / numpy-out methods.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import scipy.sparse as sp

from . import _lib
from .errors import EngineError
from .model import ModelSpec, build_design
from .ordering import choose_order

_GAIN_CODES = {"exp": 0, "spde": 1, "ar1": 2, "st": 3}


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Engine:
    """One device-resident model.  Thread-safe (calls are serialized)."""

    def __init__(self, spec: ModelSpec, y, A=None, ordering: str = "structured",
                 max_slots: int = 8, inner_tol: float = 1e-8, max_inner: int = 50,
                 device: int | None = None, selinv_slots: int = 1,
                 analytic_prior_logdet: bool = True, leaf_cutoff: int = 64):
        self.spec = spec
        self.A = build_design(spec) if A is None else sp.csr_matrix(A)
        self.A.sort_indices()
        plan = spec._prior_plan
        perm, n_dense, bounds = choose_order(spec, self.A, plan.indptr, plan.indices, ordering,
                                             leaf_cutoff=leaf_cutoff)
        self.ordering = ordering
        shapes, rates = spec.hyper_shapes_rates()
        gk = np.array([_GAIN_CODES[g[0]] for g in plan.gain_spec] or [0], dtype=np.int32)
        gt = np.array([g[1] for g in plan.gain_spec] or [0], dtype=np.int32)
        gs = np.array([g[2] for g in plan.gain_spec] or [0], dtype=np.int32)
        arrays = dict(
            p_indptr=_i64(plan.indptr), p_indices=_i64(plan.indices),
            term_entry=_i64(plan.term_entry), term_gain=_i32(plan.term_gain),
            term_coef=_f64(plan.term_coef), p_const=_f64(plan.const),
            gain_kind=gk, gain_theta=gt, gain_sub=gs,
            a_indptr=_i64(self.A.indptr), a_indices=_i64(self.A.indices), a_data=_f64(self.A.data),
            y=_f64(y), offsets=_f64(spec.offsets), exposures=_f64(spec.exposures),
            hyper_shape=_f64(shapes if spec.theta_dim else [1.0]),
            hyper_rate=_f64(rates if spec.theta_dim else [1.0]), perm=_i64(perm),
        )
        if bounds is not None:
            arrays["tile_bounds"] = _i64(bounds)
        terms = spec.prior_logdet_terms() if analytic_prior_logdet else None
        if terms is not None:
            kinds, thetas, dims, values = terms
            arrays["ld_kind"] = _i32(kinds)
            arrays["ld_theta"] = _i32(thetas)
            arrays["ld_dims"] = _i64(np.asarray(dims, dtype=np.int64).ravel())
            arrays["ld_value"] = _f64(values)
        self.analytic_prior_logdet = terms is not None
        scalars = dict(
            n_logdet_terms=0 if terms is None else len(terms[0]),
            n_tile_bounds=0 if bounds is None else int(bounds.size),
            n=spec.latent_dim, m=spec.m, d=spec.theta_dim,
            family=0 if spec.family == "gaussian" else 1,
            noise_theta=-1 if spec.noise_theta is None else int(spec.noise_theta),
            noise_precision=float(spec.noise_precision or 0.0),
            n_terms=int(plan.term_entry.size), n_gains=int(plan.n_gains), n_dense=int(n_dense),
        )
        self._create(arrays, scalars, max_slots, inner_tol, max_inner, device, selinv_slots)

    @classmethod
    def for_matrix(cls, indptr, indices, data, perm, n_dense=0, device=None, tile_bounds=None):
        """Engine over a fixed SPD matrix (lower CSC, original order): the
        generic analyze/factorize/solve/selected_inverse drop-in.  The model
        is Q itself (constant prior values, no hyperparameters, a single
        zero-weight observation)."""
        self = cls.__new__(cls)
        self.spec = None
        n = int(indptr.shape[0] - 1)
        self.A = sp.csr_matrix((np.zeros(1), (np.zeros(1, int), np.zeros(1, int))), shape=(1, n))
        arrays = dict(
            p_indptr=_i64(indptr), p_indices=_i64(indices),
            term_entry=np.zeros(1, np.int64), term_gain=np.zeros(1, np.int32),
            term_coef=np.zeros(1), p_const=_f64(data),
            gain_kind=np.zeros(1, np.int32), gain_theta=np.zeros(1, np.int32),
            gain_sub=np.zeros(1, np.int32),
            a_indptr=_i64([0, 1]), a_indices=_i64([0]), a_data=_f64([0.0]),
            y=_f64([0.0]), offsets=_f64([0.0]), exposures=_f64([1.0]),
            hyper_shape=_f64([1.0]), hyper_rate=_f64([1.0]), perm=_i64(perm),
        )
        if tile_bounds is not None:
            arrays["tile_bounds"] = _i64(tile_bounds)
        scalars = dict(n=n, m=1, d=0, family=0, noise_theta=-1, noise_precision=1.0,
                       n_terms=0, n_gains=0, n_dense=int(n_dense),
                       n_tile_bounds=0 if tile_bounds is None else int(np.size(tile_bounds)),
                       n_logdet_terms=0)
        self._create(arrays, scalars, 1, 1e-8, 50, device, 1)
        return self

    def _create(self, arrays, scalars, max_slots, inner_tol, max_inner, device, selinv_slots):
        L = _lib.load()
        self.n = int(scalars["n"])
        self.d = int(scalars["d"])
        self.perm = arrays["perm"]
        self.n_dense = int(scalars["n_dense"])
        if device is None:
            import torch  # plumbing only: which device this process owns

            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.device = int(device)
        m = _lib.PinlaModel()
        for name, val in scalars.items():
            setattr(m, name, val)
        for name, arr in arrays.items():
            ct = {np.dtype(np.int64): ctypes.c_int64, np.dtype(np.int32): ctypes.c_int32,
                  np.dtype(np.float64): ctypes.c_double}[arr.dtype]
            setattr(m, name, _lib.ptr(arr, ct))
        o = _lib.PinlaOptions()
        o.max_slots = int(max_slots)
        o.max_inner = int(max_inner)
        o.inner_tol = float(inner_tol)
        o.device = self.device
        o.selinv_slots = int(selinv_slots)
        o.analytic_prior_logdet = int(scalars.get("n_logdet_terms", 0) > 0)
        h = ctypes.c_void_p()
        _lib.check(L.pinla_create(ctypes.byref(m), ctypes.byref(o), ctypes.byref(h)))
        self._h = h
        self._L = L
        self._lock = threading.Lock()
        self._arrays = arrays  # keep alive (create copies, but be safe)
        # the library may hold fewer slots than asked (device memory)
        self.max_slots = int(self.stats()["slots"])

    def solve_resident(self, b):
        self._check_open()
        bb = _f64(b)
        x = np.empty(self.n)
        with self._lock:
            _lib.check(self._L.pinla_solve_resident(self._h, _lib.ptr(bb, ctypes.c_double),
                                                    _lib.ptr(x, ctypes.c_double)))
        return x

    def selinv_resident(self):
        self._check_open()
        var = np.empty(self.n)
        with self._lock:
            _lib.check(self._L.pinla_selinv_resident(self._h, _lib.ptr(var, ctypes.c_double)))
        return var

    # ------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._L.pinla_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check_open(self):
        if not self._h:
            raise EngineError("engine handle is closed")

    def eval_batch(self, thetas, warm=None, want_modes: bool = False):
        """f and components for k theta points; per-slot status.  ``warm``:
        None, one start (n,) for every point, or one per point (k, n)."""
        self._check_open()
        th = _f64(np.atleast_2d(np.asarray(thetas, dtype=np.float64)))
        k = th.shape[0]
        if th.shape[1] != self.d:
            raise EngineError(f"theta points must have dimension {self.d}")
        w = None if warm is None else _f64(warm)
        per_point = w is not None and w.ndim == 2
        if per_point and w.shape != (k, self.n):
            raise EngineError("per-point warm starts must be k x n")
        f = np.empty(k)
        comps = np.empty((k, 5))
        status = np.empty(k, dtype=np.int32)
        badcol = np.empty(k, dtype=np.int64)
        iters = np.empty(k, dtype=np.int32)
        lds = np.empty((k, 2))
        modes = np.empty((k, self.n)) if want_modes else None
        P = _lib.ptr
        with self._lock:
            fn = self._L.pinla_eval_batch_warm if per_point else self._L.pinla_eval_batch
            _lib.check(fn(
                self._h, k, P(th, ctypes.c_double), P(w, ctypes.c_double), P(f, ctypes.c_double),
                P(comps, ctypes.c_double), P(status, ctypes.c_int32), P(badcol, ctypes.c_int64),
                P(iters, ctypes.c_int32), P(lds, ctypes.c_double), P(modes, ctypes.c_double)))
        return dict(f=f, comps=comps, status=status, badcol=badcol, iters=iters, logdets=lds,
                    modes=modes)

    def mode(self, theta, warm=None):
        self._check_open()
        th = _f64(theta)
        w = None if warm is None else _f64(warm)
        x = np.empty(self.n)
        it = ctypes.c_int32()
        st = ctypes.c_int32()
        bc = ctypes.c_int64()
        ld = ctypes.c_double()
        P = _lib.ptr
        with self._lock:
            _lib.check(self._L.pinla_mode(self._h, P(th, ctypes.c_double), P(w, ctypes.c_double),
                                          P(x, ctypes.c_double), ctypes.byref(it), ctypes.byref(st),
                                          ctypes.byref(bc), ctypes.byref(ld)))
        return x, int(it.value), int(st.value), int(bc.value), float(ld.value)

    def selinv_diag(self, theta, warm=None):
        self._check_open()
        th = _f64(theta)
        w = None if warm is None else _f64(warm)
        var = np.empty(self.n)
        x = np.empty(self.n)
        st = ctypes.c_int32()
        bc = ctypes.c_int64()
        P = _lib.ptr
        with self._lock:
            _lib.check(self._L.pinla_selinv_diag(self._h, P(th, ctypes.c_double),
                                                 P(w, ctypes.c_double), P(var, ctypes.c_double),
                                                 P(x, ctypes.c_double), ctypes.byref(st),
                                                 ctypes.byref(bc)))
        return var, x, int(st.value), int(bc.value)

    def cond_pattern(self):
        self._check_open()
        nnz = ctypes.c_int64()
        _lib.check(self._L.pinla_cond_pattern(self._h, ctypes.byref(nnz), None, None))
        indptr = np.empty(self.n + 1, dtype=np.int64)
        indices = np.empty(nnz.value, dtype=np.int64)
        _lib.check(self._L.pinla_cond_pattern(self._h, None, _lib.ptr(indptr, ctypes.c_int64),
                                              _lib.ptr(indices, ctypes.c_int64)))
        return indptr, indices

    # drop-in payloads (read from the device on request)
    def tile_entries(self, which: int, slot: int, rows, cols):
        """Entries (rows, cols) (permuted, row >= col) of slot ``slot``'s
        factor L (which 0) or of the last selected inverse (which 1)."""
        self._check_open()
        r = _i64(rows)
        c = _i64(cols)
        out = np.empty(r.size)
        with self._lock:
            _lib.check(self._L.pinla_tile_entries(self._h, int(which), int(slot), r.size,
                                                  _lib.ptr(r, ctypes.c_int64),
                                                  _lib.ptr(c, ctypes.c_int64),
                                                  _lib.ptr(out, ctypes.c_double)))
        return out

    def cond_values(self, slot: int = 0):
        """Q_c values last assembled in ``slot`` on the cond_pattern()."""
        self._check_open()
        nnz = ctypes.c_int64()
        _lib.check(self._L.pinla_cond_pattern(self._h, ctypes.byref(nnz), None, None))
        out = np.empty(nnz.value)
        with self._lock:
            _lib.check(self._L.pinla_cond_values(self._h, int(slot), _lib.ptr(out, ctypes.c_double)))
        return out

    def factor_lmul(self, x, slot: int = 0):
        """L x with slot ``slot``'s factor (permuted order)."""
        self._check_open()
        xx = _f64(x)
        y = np.empty(self.n)
        with self._lock:
            _lib.check(self._L.pinla_factor_lmul(self._h, int(slot), _lib.ptr(xx, ctypes.c_double),
                                                 _lib.ptr(y, ctypes.c_double)))
        return y

    def factor_logdet(self, qvals):
        self._check_open()
        q = _f64(qvals)
        ld = ctypes.c_double()
        st = ctypes.c_int32()
        bc = ctypes.c_int64()
        with self._lock:
            _lib.check(self._L.pinla_factor_logdet(self._h, _lib.ptr(q, ctypes.c_double),
                                                   ctypes.byref(ld), ctypes.byref(st),
                                                   ctypes.byref(bc)))
        return float(ld.value), int(st.value), int(bc.value)

    def stats(self) -> dict:
        self._check_open()
        s = _lib.PinlaStats()
        _lib.check(self._L.pinla_stats(self._h, ctypes.byref(s)))
        return {name: getattr(s, name) for name, _ in s._fields_}

    def reset_stats(self):
        self._L.pinla_reset_stats(self._h)

    def phase_times(self) -> dict:
        v = [ctypes.c_double() for _ in range(5)]
        self._L.pinla_phase_times(self._h, *[ctypes.byref(x) for x in v])
        return dict(zip(("assemble_ms", "factor_ms", "solve_ms", "selinv_ms", "other_ms"),
                        [x.value for x in v]))
