"""ctypes front-end of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs -- never by the product
package ``paper_1701_05936_b200``.  See oracle.c's header for what each
function computes and which PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, ERR_ARG, ERR_DEGENERATE, ERR_CONVERGENCE = 0, 1, 2, 3
_DT = {np.dtype(np.float64): 0, np.dtype(np.float32): 1, np.dtype(np.int8): 2}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"oracle {where} failed with status {code}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain -O2, no fast-math, portable ISA; OpenMP for
    the optional host threads, set_threads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        _lib.or_column_stats.argtypes = [P, I, I64, I64, I64, P, P, P]
        _lib.or_lambda_max.argtypes = [P, I, I64, I64, I64, P, P, D, P, P]
        _lib.or_objective.argtypes = [P, I, I64, I64, I64, P, P, P, D, D, P]
        _lib.or_kkt.argtypes = [P, I, I64, I64, I64, P, P, P, D, D, P, P, P]
        _lib.or_bedpp.argtypes = [P, I, I64, I64, I64, P, P, D, D, P]
        _lib.or_fit_path.argtypes = [P, I, I64, I64, I64, P, P, P, I, D, D, I, I, I64,
                                     P, P, P, P, P, P, P, P]
        _lib.or_folds.argtypes = [I64, I, ctypes.c_uint64, P]
        _lib.or_std_dots.argtypes = [P, I, I64, I64, I64, P, P, P]
        _lib.or_prep.argtypes = [P, I, I64, I64, I64, P, P, D, P, P, P, P]
        _lib.or_cv.argtypes = [P, I, I64, I64, I64, P, P, I, P, I, D, D, I, I, P, P, P, P]
        _lib.or_objective_binomial.argtypes = [P, I, I64, I64, I64, P, P, D, P, D, D, P]
        _lib.or_fit_path_binomial.argtypes = [P, I, I64, I64, I64, P, P, P, I, D, D, I, I, I64,
                                              P, P, P, P, P, P, P, P, P]
        _lib.or_set_threads.argtypes = [I]
        _lib.or_set_threads.restype = None
        _lib.or_get_threads.restype = I
        _lib.or_path_begin.argtypes = [P, I, I64, I64, I64, P, P, D, ctypes.POINTER(P)]
        _lib.or_path_run.argtypes = [P, P, I, D, I, I, I64, P, P, P, P, P, P, P, P]
        _lib.or_path_end.argtypes = [P]
        _lib.or_path_end.restype = None
        _lib.or_path_lambda_max.argtypes = [P]
        _lib.or_path_lambda_max.restype = D
    return _lib


def set_threads(t: int) -> None:
    """Host threads of the oracle (1 = the pure serial oracle).  Results are bitwise
    identical for every t (oracle.c: g_threads)."""
    _L().or_set_threads(int(t))


def get_threads() -> int:
    return _L().or_get_threads()


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _design(X):
    """X: a synth.Instance, a (buf (p, ld) column-major, n) pair, or an (n, p) array.

    Returns (column-major buffer, dtype code, n, p, ld)."""
    if hasattr(X, "host_X"):
        buf, n = X.host_X(), X.n
    elif isinstance(X, tuple):
        buf, n = X
    else:
        A = np.asarray(X)
        n = A.shape[0]
        buf = np.ascontiguousarray(A.T)
    buf = np.ascontiguousarray(buf)
    if buf.dtype not in _DT:
        raise TypeError(f"unsupported dtype {buf.dtype}")
    p, ld = buf.shape
    return buf, _DT[buf.dtype], n, p, ld


def _mask(train, n):
    if train is None:
        return None
    m = np.ascontiguousarray(np.asarray(train, dtype=np.uint8))
    assert m.shape == (n,)
    return m


def column_stats(X, train=None):
    """Column means c and population SDs s over the (optional) training rows."""
    buf, dt, n, p, ld = _design(X)
    c = np.empty(p); s = np.empty(p)
    m = _mask(train, n)
    rc = _L().or_column_stats(_p(buf), dt, n, p, ld, _p(m), _p(c), _p(s))
    if rc:
        raise OracleError(rc, "column_stats")
    return c, s


def lambda_max(X, y, alpha=1.0, train=None):
    buf, dt, n, p, ld = _design(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    m = _mask(train, n)
    lm = ctypes.c_double(); js = ctypes.c_int64()
    rc = _L().or_lambda_max(_p(buf), dt, n, p, ld, _p(y), _p(m), alpha,
                            ctypes.byref(lm), ctypes.byref(js))
    if rc:
        raise OracleError(rc, "lambda_max")
    return lm.value, js.value


def std_dots(X, v, train=None):
    """z_j = x~_j' v / n_t for every column, explicit standardisation."""
    buf, dt, n, p, ld = _design(X)
    v = np.ascontiguousarray(v, dtype=np.float64)
    m = _mask(train, n)
    z = np.empty(p)
    rc = _L().or_std_dots(_p(buf), dt, n, p, ld, _p(m), _p(v), _p(z))
    if rc:
        raise OracleError(rc, "std_dots")
    return z


def prep(X, y, alpha=1.0, train=None):
    """a_j = x~_j'y~, b_j = x~_j'x~_*, j*, lambda_max (explicit)."""
    buf, dt, n, p, ld = _design(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    m = _mask(train, n)
    a = np.empty(p); b = np.empty(p)
    js = ctypes.c_int64(); lm = ctypes.c_double()
    rc = _L().or_prep(_p(buf), dt, n, p, ld, _p(y), _p(m), alpha, _p(a), _p(b), ctypes.byref(js),
                      ctypes.byref(lm))
    if rc:
        raise OracleError(rc, "prep")
    return dict(a=a, b=b, jstar=js.value, lambda_max=lm.value)


def objective(X, y, beta, lam, alpha=1.0, train=None):
    buf, dt, n, p, ld = _design(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    b = np.ascontiguousarray(beta, dtype=np.float64)
    m = _mask(train, n)
    q = ctypes.c_double()
    rc = _L().or_objective(_p(buf), dt, n, p, ld, _p(y), _p(m), _p(b), lam, alpha, ctypes.byref(q))
    if rc:
        raise OracleError(rc, "objective")
    return q.value


def kkt(X, y, beta, lam, alpha=1.0, train=None, want_z=False):
    buf, dt, n, p, ld = _design(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    b = np.ascontiguousarray(beta, dtype=np.float64)
    m = _mask(train, n)
    zv = ctypes.c_double(); nv = ctypes.c_double()
    z = np.empty(p) if want_z else None
    rc = _L().or_kkt(_p(buf), dt, n, p, ld, _p(y), _p(m), _p(b), lam, alpha,
                     ctypes.byref(zv), ctypes.byref(nv), _p(z))
    if rc:
        raise OracleError(rc, "kkt")
    return (zv.value, nv.value, z) if want_z else (zv.value, nv.value)


def bedpp_discard(X, y, alpha, lam, train=None):
    buf, dt, n, p, ld = _design(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    m = _mask(train, n)
    d = np.empty(p, dtype=np.uint8)
    rc = _L().or_bedpp(_p(buf), dt, n, p, ld, _p(y), _p(m), alpha, lam, _p(d))
    if rc:
        raise OracleError(rc, "bedpp")
    return d.astype(bool)


class PathResult:
    """Dense view of an oracle path: beta is (p, nlam) on the standardised scale."""

    def __init__(self, lam, beta, a0, obj, passes, resid, n_converged, status):
        self.lam, self.beta, self.a0, self.obj = lam, beta, a0, obj
        self.passes, self.resid, self.n_converged, self.status = passes, resid, n_converged, status


def fit_path(X, y, lam, alpha=1.0, tol=1e-10, max_iter=100000, cycle_active=True,
             train=None, want_resid=False, nnz_cap=None, raise_on_error=True):
    buf, dt, n, p, ld = _design(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    K = lam.size
    m = _mask(train, n)
    cap = nnz_cap or min(p * K, max(1, min(n, p) * K * 2 + 16))
    col_ptr = np.zeros(K + 1, dtype=np.int64)
    idx = np.empty(cap, dtype=np.int64); val = np.empty(cap)
    a0 = np.empty(K); obj = np.empty(K); passes = np.empty(K, dtype=np.int32)
    resid = np.empty((K, n)) if want_resid else None
    nc = ctypes.c_int()
    rc = _L().or_fit_path(_p(buf), dt, n, p, ld, _p(y), _p(m), _p(lam), K, alpha, tol, max_iter,
                          int(cycle_active), cap, _p(col_ptr), _p(idx), _p(val), _p(a0), _p(obj),
                          _p(passes), _p(resid), ctypes.byref(nc))
    if rc and raise_on_error:
        raise OracleError(rc, "fit_path")
    beta = np.zeros((p, K))
    for k in range(nc.value):
        sl = slice(col_ptr[k], col_ptr[k + 1])
        beta[idx[sl], k] = val[sl]
    return PathResult(lam, beta, a0, obj, passes, resid, nc.value, rc)


class PathSession:
    """A pathwise solve run in consecutive chunks of the lambda grid with warm starts
    (or_path_begin / or_path_run / or_path_end): the chunks together are exactly
    fit_path over the concatenated grid."""

    def __init__(self, X, y, alpha=1.0, train=None):
        buf, dt, n, p, ld = _design(X)
        self._buf = buf                       # the C side reads X in place
        self.n, self.p = n, p
        y = np.ascontiguousarray(y, dtype=np.float64)
        m = _mask(train, n)
        h = ctypes.c_void_p()
        rc = _L().or_path_begin(_p(buf), dt, n, p, ld, _p(y), _p(m), alpha, ctypes.byref(h))
        if rc:
            raise OracleError(rc, "path_begin")
        self.h = h
        self.lambda_max = _L().or_path_lambda_max(h)   # max_j |x~_j'y~| / (n alpha) (Q3)

    def run(self, lam, tol=1e-10, max_iter=100000, cycle_active=True, nnz_cap=None):
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        K = lam.size
        cap = nnz_cap or min(self.p * K, max(1, min(self.n, self.p) * K * 2 + 16))
        col_ptr = np.zeros(K + 1, dtype=np.int64)
        idx = np.empty(cap, dtype=np.int64); val = np.empty(cap)
        a0 = np.empty(K); obj = np.empty(K); passes = np.empty(K, dtype=np.int32)
        nc = ctypes.c_int()
        rc = _L().or_path_run(self.h, _p(lam), K, tol, max_iter, int(cycle_active), cap, _p(col_ptr), _p(idx),
                              _p(val), _p(a0), _p(obj), _p(passes), None, ctypes.byref(nc))
        if rc:
            raise OracleError(rc, "path_run")
        beta = np.zeros((self.p, K))
        for k in range(nc.value):
            sl = slice(col_ptr[k], col_ptr[k + 1])
            beta[idx[sl], k] = val[sl]
        return PathResult(lam, beta, a0, obj, passes, None, nc.value, rc)

    def close(self):
        if getattr(self, "h", None):
            _L().or_path_end(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def folds(n, K, seed):
    f = np.empty(n, dtype=np.int32)
    rc = _L().or_folds(n, K, seed, _p(f))
    if rc:
        raise OracleError(rc, "folds")
    return f


def cv(X, y, fold_id, K, lam, alpha=1.0, tol=1e-10, max_iter=100000, cycle_active=True):
    buf, dt, n, p, ld = _design(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    f = np.ascontiguousarray(fold_id, dtype=np.int32)
    nl = lam.size
    E = np.zeros((nl, n)); cve = np.empty(nl); cvse = np.empty(nl)
    lmin = ctypes.c_int()
    rc = _L().or_cv(_p(buf), dt, n, p, ld, _p(y), _p(f), K, _p(lam), nl, alpha, tol, max_iter,
                    int(cycle_active), _p(E), _p(cve), _p(cvse), ctypes.byref(lmin))
    if rc:
        raise OracleError(rc, "cv")
    return E, cve, cvse, lmin.value


# ------------------------------------------------------------ NEXT-3: logistic path

def objective_binomial(X, y, b0, beta, lam, alpha=1.0, train=None):
    """Q(b0, b) = mean_i [log(1 + e^eta_i) - y_i eta_i] + lambda (alpha |b|_1 + (1-alpha)/2 |b|^2) (QL1)."""
    buf, dt, n, p, ld = _design(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    b = np.ascontiguousarray(beta, dtype=np.float64)
    m = _mask(train, n)
    q = ctypes.c_double()
    rc = _L().or_objective_binomial(_p(buf), dt, n, p, ld, _p(y), _p(m), float(b0), _p(b), lam, alpha,
                                    ctypes.byref(q))
    if rc:
        raise OracleError(rc, "objective_binomial")
    return q.value


class BinomialPathResult(PathResult):
    def __init__(self, lam, beta, b0, a0, obj, passes, outer, n_converged, status):
        super().__init__(lam, beta, a0, obj, passes, None, n_converged, status)
        self.b0, self.outer = b0, outer


def fit_path_binomial(X, y, lam, alpha=1.0, tol=1e-10, max_iter=100000, cycle_active=True,
                      train=None, nnz_cap=None, raise_on_error=True):
    """Penalised logistic path by IRLS + cyclic weighted CD, no screening (oracle.c NEXT-3)."""
    buf, dt, n, p, ld = _design(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    K = lam.size
    m = _mask(train, n)
    cap = nnz_cap or min(p * K, max(1, min(n, p) * K * 2 + 16))
    col_ptr = np.zeros(K + 1, dtype=np.int64)
    idx = np.empty(cap, dtype=np.int64); val = np.empty(cap)
    b0 = np.empty(K); a0 = np.empty(K); obj = np.empty(K)
    passes = np.empty(K, dtype=np.int32); outer = np.empty(K, dtype=np.int32)
    nc = ctypes.c_int()
    rc = _L().or_fit_path_binomial(_p(buf), dt, n, p, ld, _p(y), _p(m), _p(lam), K, alpha, tol, max_iter,
                                   int(cycle_active), cap, _p(col_ptr), _p(idx), _p(val), _p(b0), _p(a0),
                                   _p(obj), _p(passes), _p(outer), ctypes.byref(nc))
    if rc and raise_on_error:
        raise OracleError(rc, "fit_path_binomial")
    beta = np.zeros((p, K))
    for k in range(nc.value):
        sl = slice(col_ptr[k], col_ptr[k + 1])
        beta[idx[sl], k] = val[sl]
    return BinomialPathResult(lam, beta, b0, a0, obj, passes, outer, nc.value, rc)
