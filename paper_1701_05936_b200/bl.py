"""Thin ctypes binding of libbl.so (include/bl.h) -- argument marshalling only.

Every step of the path runs in the sm_100a kernels behind the C ABI; this
module only converts numpy / torch buffers to pointers and result buffers back
to numpy.  There is no fallback: if libbl.so is missing or no sm_100a device is
present the calls raise.

Functions carry the C names (bl_load_design, bl_fit_path, bl_cv, bl_free, ...);
`Design`, `Path`, `CvResult`, `Prep` are small owners that free their handle.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libbl.so")

BL_OK, BL_ERR_ARG, BL_ERR_DEGENERATE, BL_ERR_CONVERGENCE, BL_ERR_CUDA, BL_ERR_NCCL, BL_ERR_OOM = range(7)
BL_F64, BL_F32, BL_I8 = 0, 1, 2
SCREEN = {"none": 0, "ssr": 1, "hybrid": 2}
CD_MODE = {"auto": 0, "residual": 1, "gram": 2}
_DT = {np.dtype(np.float64): BL_F64, np.dtype(np.float32): BL_F32, np.dtype(np.int8): BL_I8}
_ITEM = {BL_F64: 8, BL_F32: 4, BL_I8: 1}


class BLError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[bl status {code}] {msg}")
        self.code = code


_ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)
_BCAST = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int)
_ALLREDUCE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)


class bl_host_coll(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("allgather", _ALLGATHER), ("bcast", _BCAST),
                ("allreduce_sum_f64", _ALLREDUCE)]


class bl_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("device", ctypes.c_int),
                ("nccl_unique_id", ctypes.c_void_p), ("col_offset", ctypes.c_int64),
                ("p_global", ctypes.c_int64), ("backend", ctypes.c_int),
                ("host_coll", ctypes.POINTER(bl_host_coll)), ("timeout_ms", ctypes.c_int)]


class bl_opts(ctypes.Structure):
    _fields_ = [("stream", ctypes.c_void_p), ("profile", ctypes.c_int), ("max_kkt_rounds", ctypes.c_int),
                ("cd_mode", ctypes.c_int), ("cv_mode", ctypes.c_int), ("cd_cluster", ctypes.c_int),
                ("stream_chunk_bytes", ctypes.c_int64), ("fault_strong_drop", ctypes.c_int),
                ("cd_accel", ctypes.c_int)]


CV_MODE = {"batched": 0, "batched_fma": 1, "independent": 2, "batched_dmma": 3}


def _opts(stream=None, profile=False, max_kkt_rounds=0, cd="auto", cv_mode="batched", cd_cluster=0,
          stream_chunk_bytes=0, fault_strong_drop=0, cd_accel="newton"):
    return bl_opts(stream, int(profile), int(max_kkt_rounds), CD_MODE[cd], CV_MODE[cv_mode], int(cd_cluster),
                   int(stream_chunk_bytes), int(fault_strong_drop), {"newton": 0, "none": 1}[cd_accel])


class bl_perf(ctypes.Structure):
    _fields_ = [("scan_ms", ctypes.c_double), ("scan_bytes", ctypes.c_double),
                ("scan_launches", ctypes.c_int64), ("cd_ms", ctypes.c_double),
                ("cd_launches", ctypes.c_int64), ("prep_ms", ctypes.c_double),
                ("prep_bytes", ctypes.c_double), ("kernel_launches", ctypes.c_int64),
                ("wall_ms", ctypes.c_double), ("cd_visits", ctypes.c_int64), ("cd_updates", ctypes.c_int64),
                ("cd_kernel_cycles", ctypes.c_int64), ("cd_prof", ctypes.c_int64 * 4),
                ("full_scan_ms", ctypes.c_double), ("full_scan_bytes", ctypes.c_double),
                ("full_scan_launches", ctypes.c_int64), ("cd_events", ctypes.c_int64 * 8),
                ("cd_sub", ctypes.c_int64 * 8)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["cd_prof"] = list(self.cd_prof)
        d["cd_events"] = list(self.cd_events)
        d["cd_sub"] = list(self.cd_sub)
        return d



_lib = None
EXPORTS = ["bl_load_design", "bl_nccl_unique_id", "bl_lambda_max", "bl_fit_path", "bl_cv", "bl_path_info",
           "bl_path_copy", "bl_path_perf", "bl_path_screen", "bl_fit_path_binomial", "bl_path_irls", "bl_cv_copy", "bl_cv_errors", "bl_cv_perf", "bl_prepare", "bl_prep_copy",
           "bl_bedpp", "bl_scan", "bl_scan_batch", "bl_free", "bl_last_error", "bl_trim"]


def lib():
    """Load libbl.so (raises if it was not built -- no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1701_05936_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    P, I, I64, D, U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64
    PP = ctypes.POINTER(ctypes.c_void_p)
    L.bl_load_design.argtypes = [P, I, I64, I64, I64, I, P, PP]
    L.bl_nccl_unique_id.argtypes = [P]
    L.bl_lambda_max.argtypes = [P, P, D, P]
    L.bl_fit_path.argtypes = [P, P, P, I, D, D, I, I, P, PP]
    L.bl_cv.argtypes = [P, P, P, I, D, D, I, I, P, U64, P, PP]
    L.bl_path_info.argtypes = [P, P, P, P]
    L.bl_path_copy.argtypes = [P] + [P] * 10
    L.bl_path_perf.argtypes = [P, P]
    L.bl_path_screen.argtypes = [P, P, P, P]
    L.bl_fit_path_binomial.argtypes = [P, P, P, I, D, D, I, I, P, PP]
    L.bl_path_irls.argtypes = [P, P]
    L.bl_cv_copy.argtypes = [P, P, P, P, P, PP]
    L.bl_cv_errors.argtypes = [P, P]
    L.bl_cv_perf.argtypes = [P, P]
    L.bl_prepare.argtypes = [P, P, P, D, PP]
    L.bl_prep_copy.argtypes = [P, P, P, P, P, P, P]
    L.bl_bedpp.argtypes = [P, D, P, P]
    L.bl_scan.argtypes = [P, P, D, D, P, P, P, P, P, P]
    L.bl_scan_batch.argtypes = [P, ctypes.c_int, P, D, D, ctypes.c_int, P, P, P]
    L.bl_free.argtypes = [P]
    L.bl_free.restype = None
    L.bl_last_error.restype = ctypes.c_char_p
    L.bl_trim.restype = None
    for f in EXPORTS:
        if f not in ("bl_free", "bl_last_error", "bl_trim"):
            getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _check(rc, allow=()):
    if rc != BL_OK and rc not in allow:
        raise BLError(rc, lib().bl_last_error().decode())
    return rc


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ C-named calls

def bl_load_design(X, n, dist=None, host_resident=False):
    """X: (p, ld) column-major buffer -- numpy (host: copied to the device, or with
    host_resident=True borrowed and streamed over PCIe, NEXT-4) or a CUDA torch
    tensor (device, borrowed: keep it alive).  Returns a raw handle."""
    h = ctypes.c_void_p()
    if isinstance(X, np.ndarray):
        if host_resident and not X.flags.c_contiguous:
            raise ValueError("host-resident X must be C-contiguous (p, ld)")
        X = np.ascontiguousarray(X)
        dt = _DT[X.dtype]
        p, ld = X.shape
        rc = lib().bl_load_design(_p(X), dt, n, p, ld, 2 if host_resident else 0,
                                  ctypes.byref(dist) if dist else None, ctypes.byref(h))
    else:  # torch tensor on the device
        import torch
        dt = {torch.float64: BL_F64, torch.float32: BL_F32, torch.int8: BL_I8}[X.dtype]
        assert X.is_cuda and X.is_contiguous()
        p, ld = X.shape
        rc = lib().bl_load_design(ctypes.c_void_p(X.data_ptr()), dt, n, p, ld, 1,
                                  ctypes.byref(dist) if dist else None, ctypes.byref(h))
    _check(rc)
    return h


def bl_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().bl_nccl_unique_id(buf))
    return buf.raw


def bl_free(h):
    if h:
        lib().bl_free(h)


# ------------------------------------------------------------------ owners

class Path:
    """Read-out of a bl_path (standardised and original-scale sparse beta)."""

    def __init__(self, handle, status):
        L = lib()
        self.status = status
        K = ctypes.c_int(); nnz = ctypes.c_int64(); nc = ctypes.c_int()
        _check(L.bl_path_info(handle, ctypes.byref(K), ctypes.byref(nnz), ctypes.byref(nc)))
        K, nnz = K.value, nnz.value
        self.n_converged = nc.value
        self.lam = np.empty(K); self.a0 = np.empty(K); self.obj = np.empty(K)
        self.col_ptr = np.empty(K + 1, np.int64); self.feat = np.empty(nnz, np.int64)
        self.beta_std = np.empty(nnz); self.beta_orig = np.empty(nnz)
        self.passes = np.empty(K, np.int32); self.kkt_rounds = np.empty(K, np.int32)
        self.cols_scanned = np.empty(K, np.int64)
        _check(L.bl_path_copy(handle, _p(self.lam), _p(self.a0), _p(self.obj), _p(self.col_ptr), _p(self.feat),
                              _p(self.beta_std), _p(self.beta_orig), _p(self.passes), _p(self.kkt_rounds),
                              _p(self.cols_scanned)))
        pf = bl_perf()
        _check(L.bl_path_perf(handle, ctypes.byref(pf)))
        self.perf = pf.as_dict()
        # screening diagnostics per lambda: |S_k| (BEDPP-safe), |strong_k|, |W| (Fig 1 analog)
        self.n_safe = np.zeros(K, np.int64); self.n_strong = np.zeros(K, np.int64)
        self.n_working = np.zeros(K, np.int64)
        _check(L.bl_path_screen(handle, _p(self.n_safe), _p(self.n_strong), _p(self.n_working)))

    def dense(self, p, which="std"):
        """(p, n_lambda) dense coefficient matrix."""
        B = np.zeros((p, len(self.lam)))
        v = self.beta_std if which == "std" else self.beta_orig
        for k in range(self.n_converged):
            sl = slice(self.col_ptr[k], self.col_ptr[k + 1])
            B[self.feat[sl], k] = v[sl]
        return B


class Prep:
    def __init__(self, design, y, train=None, alpha=1.0):
        self.design = design
        self.p = design.p
        y = _f64(y)
        m = None if train is None else np.ascontiguousarray(train, dtype=np.uint8)
        h = ctypes.c_void_p()
        _check(lib().bl_prepare(design.h, _p(y), _p(m), alpha, ctypes.byref(h)))
        self.h = h

    def copy(self):
        p = self.p
        c, s, a, b = np.empty(p), np.empty(p), np.empty(p), np.empty(p)
        js = ctypes.c_int64(); lm = ctypes.c_double()
        _check(lib().bl_prep_copy(self.h, _p(c), _p(s), _p(a), _p(b), ctypes.byref(js), ctypes.byref(lm)))
        return dict(c=c, s=s, a=a, b=b, jstar=js.value, lambda_max=lm.value)

    def bedpp(self, lam):
        keep = np.empty(self.p, np.uint8)
        cnt = ctypes.c_int64()
        _check(lib().bl_bedpp(self.h, lam, _p(keep), ctypes.byref(cnt)))
        return keep.astype(bool), cnt.value

    def scan(self, r, lam, lam_next=-1.0, in_w=None):
        r = _f64(r)
        w = None if in_w is None else np.ascontiguousarray(in_w, dtype=np.uint8)
        z = np.empty(self.p)
        viol = np.empty(self.p, np.int32); strong = np.empty(self.p, np.int32)
        nv = ctypes.c_int64(); ns = ctypes.c_int64()
        _check(lib().bl_scan(self.h, _p(r), lam, lam_next, _p(w), _p(z), _p(viol), ctypes.byref(nv),
                             _p(strong), ctypes.byref(ns)))
        return z, viol[: nv.value].copy(), strong[: ns.value].copy()

    def __del__(self):
        if getattr(self, "h", None):
            lib().bl_free(self.h)
            self.h = None


def trim():
    """bl_trim: hand the library's cached device / pinned-host blocks back to the driver."""
    lib().bl_trim()


def scan_batch(preps, rs, lam, lam_next=-1.0, cv_mode="batched"):
    """bl_scan_batch: the fused scans of several fits of one design in one fold-batched pass.
    Returns z (nf, p) and the violator / strong counts per fit."""
    nf = len(preps)
    rs = [_f64(r) for r in rs]
    hs = (ctypes.c_void_p * nf)(*[pr.h.value for pr in preps])
    rp = (ctypes.c_void_p * nf)(*[r.ctypes.data for r in rs])
    p = preps[0].p
    z = np.empty((nf, p))
    nv = np.empty(nf, np.int64); ns = np.empty(nf, np.int64)
    _check(lib().bl_scan_batch(ctypes.cast(hs, ctypes.c_void_p), nf, ctypes.cast(rp, ctypes.c_void_p), lam, lam_next,
                               CV_MODE[cv_mode], _p(z), _p(nv), _p(ns)))
    return z, nv, ns


class Design:
    """Owner of a bl_design.  X is a (p, ld) column-major buffer (see synth)."""

    def __init__(self, X, n, dist=None, host_resident=False):
        self._keep = X  # borrowed device / host-resident buffers must outlive the design
        self._dist = dist   # host-collective callbacks (backend 2) must outlive the design
        self.n = int(n)
        self.p = int(X.shape[0])
        self.h = bl_load_design(X, self.n, dist, host_resident)

    def lambda_max(self, y, alpha=1.0):
        out = ctypes.c_double()
        _check(lib().bl_lambda_max(self.h, _p(_f64(y)), alpha, ctypes.byref(out)))
        return out.value

    def fit_path(self, y, lam, alpha=1.0, tol=1e-7, max_iter=10000, screen="hybrid", stream=None,
                 profile=False, max_kkt_rounds=0, raise_on_error=True, cd="auto", **opts):
        """opts: cd_cluster, stream_chunk_bytes, fault_strong_drop (bl_opts, include/bl.h)."""
        lam = _f64(lam)
        o = _opts(stream, profile, max_kkt_rounds, cd, **opts)
        h = ctypes.c_void_p()
        rc = lib().bl_fit_path(self.h, _p(_f64(y)), _p(lam), lam.size, alpha, tol, max_iter,
                               SCREEN.get(screen, screen), ctypes.byref(o), ctypes.byref(h))
        _check(rc, allow=() if raise_on_error else (BL_ERR_CONVERGENCE,))
        try:
            return Path(h, rc)
        finally:
            lib().bl_free(h)

    def fit_path_binomial(self, y, lam, alpha=1.0, tol=1e-7, max_iter=10000, screen="ssr", stream=None,
                          profile=False, max_kkt_rounds=0, raise_on_error=True, cd="auto", **opts):
        """Penalised logistic path (NEXT-3, bl_fit_path_binomial); y in {0, 1}.
        cd: "auto" (covariance form while |W| < 2048) or "residual"."""
        lam = _f64(lam)
        o = _opts(stream, profile, max_kkt_rounds, cd, **opts)
        h = ctypes.c_void_p()
        rc = lib().bl_fit_path_binomial(self.h, _p(_f64(y)), _p(lam), lam.size, alpha, tol, max_iter,
                                        SCREEN.get(screen, screen), ctypes.byref(o), ctypes.byref(h))
        _check(rc, allow=() if raise_on_error else (BL_ERR_CONVERGENCE,))
        try:
            path = Path(h, rc)
            path.outer = np.zeros(lam.size, np.int32)
            _check(lib().bl_path_irls(h, _p(path.outer)))
            return path
        finally:
            lib().bl_free(h)

    def cv(self, y, lam, K=10, alpha=1.0, tol=1e-7, max_iter=10000, fold_id=None, seed=0, stream=None,
           profile=False, cd="auto", cv_mode="batched", max_kkt_rounds=0, **opts):
        """cv_mode: "batched" (lockstep fits, one fold-batched pass over X per round on the tensor
        cores; default), "batched_fma", "independent" (bl_opts.cv_mode)."""
        lam = _f64(lam)
        f = None if fold_id is None else np.ascontiguousarray(fold_id, dtype=np.int32)
        o = _opts(stream, profile, max_kkt_rounds, cd, cv_mode, **opts)
        h = ctypes.c_void_p()
        _check(lib().bl_cv(self.h, _p(_f64(y)), _p(lam), lam.size, alpha, tol, max_iter, K, _p(f), seed,
                           ctypes.byref(o), ctypes.byref(h)))
        try:
            return CvResult(h, lam.size, self.n)
        finally:
            lib().bl_free(h)

    def prepare(self, y, train=None, alpha=1.0):
        return Prep(self, y, train, alpha)

    def free(self):
        if getattr(self, "h", None):
            lib().bl_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:      # interpreter shutdown: the module globals may already be gone
            pass


class CvResult:
    def __init__(self, handle, K_lam, n):
        L = lib()
        self.cve = np.empty(K_lam); self.cvse = np.empty(K_lam)
        lmin = ctypes.c_int()
        self.fold_id = np.empty(n, np.int32)
        full = ctypes.c_void_p()
        _check(L.bl_cv_copy(handle, _p(self.cve), _p(self.cvse), ctypes.byref(lmin), _p(self.fold_id),
                            ctypes.byref(full)))
        self.lambda_min_index = lmin.value
        self.E = np.empty((K_lam, n))
        _check(L.bl_cv_errors(handle, _p(self.E)))
        pf = bl_perf()
        _check(L.bl_cv_perf(handle, ctypes.byref(pf)))
        self.perf = pf.as_dict()
        self.full = Path(full, BL_OK) if full.value else None


# ------------------------------------------------------------------ multi-GPU plumbing

def shard_range(p, world, rank, block=1):
    """Rank's contiguous column shard [j0, j1) of p columns: balanced whole
    `block`-column blocks, in rank order (the layout bl_dist requires)."""
    nb = (p + block - 1) // block
    b0, b1 = nb * rank // world, nb * (rank + 1) // world
    return min(p, b0 * block), min(p, b1 * block)


def make_dist(rank, world, col_range, p_global, device=0, group=None, timeout_ms=0):
    """bl_dist of a torch.distributed job (NCCL backend): rank 0 draws the NCCL
    unique id, every rank receives it with torch.distributed.broadcast_object_list.
    p_global == col_range width => replicated design."""
    import torch.distributed as tdist
    uid = [bl_nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(uid, src=0, group=group)
    return _dist(rank, world, device, uid[0], col_range, p_global, 0, timeout_ms)


def loopback_dist(rank, world, col_range, p_global, key, device=0):
    """bl_dist of the in-process loopback backend (testing: ranks = threads of
    one process on one device); `key` = 128-byte group key shared by the ranks."""
    return _dist(rank, world, device, key, col_range, p_global, 1)


def _dist(rank, world, device, key, col_range, p_global, backend, timeout_ms=0):
    key = bytes(key)
    assert len(key) == 128
    buf = ctypes.create_string_buffer(key, 128)
    d = bl_dist(rank, world, device, ctypes.cast(buf, ctypes.c_void_p), int(col_range[0]), int(p_global), backend,
                None, int(timeout_ms))
    d._key_buf = buf          # keep the id alive with the struct
    return d


def host_coll_dist(rank, world, col_range, p_global, allgather, bcast, allreduce_sum, device=0):
    """bl_dist of the host-collective backend (bl_dist.backend = 2): the library stages each
    collective in host memory and calls back into Python --
      allgather(send: bytes) -> bytes (world x len(send), rank order)
      bcast(buf: bytearray, root) -> None (in place)
      allreduce_sum(v: np.ndarray float64) -> None (in place)
    e.g. implemented with torch.distributed over gloo between processes (marshalling only)."""
    def ag(ctx, send, recv, nbytes):
        try:
            out = allgather(ctypes.string_at(send, nbytes) if nbytes else b"")
            assert len(out) == world * nbytes
            if nbytes:
                ctypes.memmove(recv, out, world * nbytes)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
            return 1

    def bc(ctx, buf, nbytes, root):
        try:
            b = bytearray(ctypes.string_at(buf, nbytes)) if nbytes else bytearray()
            bcast(b, root)
            if nbytes:
                ctypes.memmove(buf, bytes(b), nbytes)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def ar(ctx, buf, count):
        try:
            v = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ctypes.c_double)), shape=(int(count),))
            allreduce_sum(v)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    hc = bl_host_coll(None, _ALLGATHER(ag), _BCAST(bc), _ALLREDUCE(ar))
    d = bl_dist(rank, world, device, None, int(col_range[0]), int(p_global), 2, ctypes.pointer(hc), 0)
    d._hc = hc                # the callbacks must outlive every call on the design
    return d
