"""NEXT-4: out-of-core (host-resident) designs.  X stays in host memory, mapped into
the device address space (bl_load_design x_is_device_ptr = 2); full passes stream it
over the host link and the working-set columns live in a device store.  The
arithmetic is the device-resident path's, so results must be BITWISE identical, and
oracle parity follows from tests/test_gpu_parity.py."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

bl = pytest.importorskip("paper_1701_05936_b200.bl")


def same_path(a, b):
    assert a.n_converged == b.n_converged
    for f in ("col_ptr", "feat", "beta_std", "beta_orig", "a0", "obj", "kkt_rounds", "cols_scanned", "passes"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)


@pytest.mark.parametrize("dtype,alpha,cd", [
    (np.float32, 1.0, "auto"), (np.float64, 0.5, "auto"), (np.int8, 1.0, "auto"),
    (np.float32, 0.5, "residual"), (np.int8, 0.5, "residual")])
def test_host_resident_path_is_bitwise_equal(dtype, alpha, cd):
    kind = "geno" if dtype == np.int8 else "corr"
    inst = synth.random_instance(211, 1500, dtype=dtype, seed=41, kind=kind, n_true=12, const_cols=2)
    Xh = np.ascontiguousarray(inst.host_X())
    dd = bl.Design(Xh, inst.n)
    dh = bl.Design(Xh, inst.n, host_resident=True)
    lm = dd.lambda_max(inst.y, alpha)
    assert dh.lambda_max(inst.y, alpha) == lm
    lams = synth.lambda_grid(lm, 40, 0.05)
    a = dd.fit_path(inst.y, lams, alpha=alpha, tol=1e-9, cd=cd)
    b = dh.fit_path(inst.y, lams, alpha=alpha, tol=1e-9, cd=cd)
    same_path(a, b)
    op = oracle.fit_path(inst, inst.y, lams, alpha=alpha, tol=1e-11)
    B = b.dense(inst.p)
    for k in range(len(lams)):
        sc = np.abs(op.beta[:, k]).max()
        assert np.abs(B[:, k] - op.beta[:, k]).max() <= 1e-5 * sc or sc == 0.0


@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.int8])
def test_streamed_chunks_cross_boundaries(dtype):
    """The streamed dense scans with a small bl_opts.stream_chunk_bytes: >= 3 chunks per pass
    with a short last chunk (buffer flips, shifted virtual bases, the copied / used event
    waits) give the device-resident path bitwise."""
    kind = "geno" if dtype == np.int8 else "corr"
    inst = synth.random_instance(203, 2101, dtype=dtype, seed=42, kind=kind, n_true=12, const_cols=2)
    Xh = np.ascontiguousarray(inst.host_X())
    colb = Xh.shape[1] * Xh.itemsize
    chunk = 500 * colb                                    # 2101 columns -> 500, 500, 500, 500, 101
    assert -(-inst.p // 500) >= 3 and inst.p % 500 != 0
    dd = bl.Design(Xh, inst.n)
    dh = bl.Design(Xh, inst.n, host_resident=True)
    lm = dd.lambda_max(inst.y, 1.0)
    lams = synth.lambda_grid(lm, 30, 0.05)
    a = dd.fit_path(inst.y, lams, tol=1e-9)
    b = dh.fit_path(inst.y, lams, tol=1e-9, stream_chunk_bytes=chunk)
    same_path(a, b)
    c = dh.fit_path(inst.y, lams, tol=1e-9, stream_chunk_bytes=chunk + 7 * colb)   # re-sized buffers on reuse
    same_path(a, c)


def test_host_resident_cv_and_logistic():
    inst = synth.random_instance(150, 800, dtype=np.float32, seed=43, kind="corr", n_true=8)
    Xh = np.ascontiguousarray(inst.host_X())
    dd, dh = bl.Design(Xh, inst.n), bl.Design(Xh, inst.n, host_resident=True)
    lams = synth.lambda_grid(dd.lambda_max(inst.y, 0.5), 20, 0.1)
    ca = dd.cv(inst.y, lams, K=5, alpha=0.5, tol=1e-9, seed=3)
    cb = dh.cv(inst.y, lams, K=5, alpha=0.5, tol=1e-9, seed=3)
    np.testing.assert_array_equal(ca.cve, cb.cve)
    np.testing.assert_array_equal(ca.cvse, cb.cvse)
    li = synth.logistic_instance(150, 800, dtype=np.float32, seed=44, n_true=8, scale=1.5)
    Lh = np.ascontiguousarray(li.host_X())
    ld_, lh_ = bl.Design(Lh, li.n), bl.Design(Lh, li.n, host_resident=True)
    ll = synth.lambda_grid(ld_.lambda_max(li.y), 15, 0.2)
    same_path(ld_.fit_path_binomial(li.y, ll, tol=1e-10), lh_.fit_path_binomial(li.y, ll, tol=1e-10))


def test_host_resident_pinned_by_caller_and_alignment():
    import torch
    inst = synth.random_instance(120, 300, dtype=np.float32, seed=45, n_true=5)
    t = torch.from_numpy(np.ascontiguousarray(inst.host_X())).pin_memory()
    d = bl.Design(t.numpy(), inst.n, host_resident=True)      # already registered: mapped, not owned
    lams = synth.lambda_grid(d.lambda_max(inst.y), 10, 0.2)
    ref = bl.Design(inst.host_X(), inst.n).fit_path(inst.y, lams, tol=1e-9)
    same_path(d.fit_path(inst.y, lams, tol=1e-9), ref)
    d.free()
    assert t.is_pinned()                                      # the caller's registration survives
    X = np.zeros((10, 121), np.float32)                       # ld * 4 bytes not a multiple of 16
    with pytest.raises(bl.BLError) as e:
        bl.Design(X, 120, host_resident=True)
    assert e.value.code == bl.BL_ERR_ARG


def test_host_resident_sharded_is_G_invariant():
    """Column shards that each stay in host memory (loopback transport, 2 ranks) give the
    single-GPU path bitwise."""
    import os
    import threading
    inst = synth.random_instance(130, 700, dtype=np.float32, seed=47, kind="corr", n_true=10)
    Xh = np.ascontiguousarray(inst.host_X())
    ref_d = bl.Design(Xh, inst.n)
    lams = synth.lambda_grid(ref_d.lambda_max(inst.y), 25, 0.1)
    ref = ref_d.fit_path(inst.y, lams, tol=1e-9)
    G, key = 2, os.urandom(128)
    out, errs = [None] * G, []

    def work(r):
        try:
            j0, j1 = bl.shard_range(inst.p, G, r)
            shard = np.ascontiguousarray(Xh[j0:j1])
            d = bl.Design(shard, inst.n, dist=bl.loopback_dist(r, G, (j0, j1), inst.p, key), host_resident=True)
            out[r] = d.fit_path(inst.y, lams, tol=1e-9)
            d.free()
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))
    th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    [t.start() for t in th]
    [t.join(timeout=600) for t in th]
    assert not errs, errs
    for r in range(G):
        same_path(out[r], ref)
