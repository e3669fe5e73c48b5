"""Column-sharded multi-GPU path (BASELINE north star: features
column-sharded for the scans, strong / violator index lists all-gathered, the
working-set columns broadcast by their owners, CD replicated) on ONE GPU: the
ranks are threads of this process using the library's in-process loopback
backend (bl_dist.backend = 1), so the orchestration, the collectives' payloads
and the global bookkeeping run exactly as with NCCL, only the transport
differs.  The sharded path must be G-invariant: identical coefficients (bitwise)
to the single-GPU path, and to the oracle within the north-star tolerances."""
import os
import threading

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

bl = pytest.importorskip("paper_1701_05936_b200.bl")


def run_ranks(G, fn):
    out, errs = [None] * G, []

    def work(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


def sharded_designs(inst, G):
    key = os.urandom(128)
    Xh = inst.host_X()

    def mk(r):
        j0, j1 = bl.shard_range(inst.p, G, r)
        return bl.Design(np.ascontiguousarray(Xh[j0:j1]), inst.n,
                         dist=bl.loopback_dist(r, G, (j0, j1), inst.p, key))
    return run_ranks(G, mk)


@pytest.mark.parametrize("dtype,alpha,G,cd", [
    (np.float64, 1.0, 2, "gram"), (np.float32, 0.5, 3, "gram"), (np.int8, 1.0, 2, "gram"),
    (np.float32, 1.0, 2, "residual"), (np.float64, 0.5, 4, "residual")])
def test_sharded_path_is_G_invariant(dtype, alpha, G, cd):
    kind = "geno" if dtype == np.int8 else "corr"
    inst = synth.random_instance(150, 700, dtype=dtype, seed=11, kind=kind, n_true=12, alpha=alpha)
    d1 = bl.Design(inst.host_X(), inst.n)
    lm = d1.lambda_max(inst.y, alpha)
    lams = synth.lambda_grid(lm, 30, 0.05)
    ref = d1.fit_path(inst.y, lams, alpha=alpha, tol=1e-9, cd=cd)
    ds = sharded_designs(inst, G)
    lms = run_ranks(G, lambda r: ds[r].lambda_max(inst.y, alpha))
    assert all(v == lm for v in lms)
    paths = run_ranks(G, lambda r: ds[r].fit_path(inst.y, lams, alpha=alpha, tol=1e-9, cd=cd))
    for p in paths:
        assert p.n_converged == ref.n_converged == len(lams)
        assert np.array_equal(p.col_ptr, ref.col_ptr)
        assert np.array_equal(p.feat, ref.feat)
        assert np.array_equal(p.beta_std, ref.beta_std)
        assert np.array_equal(p.beta_orig, ref.beta_orig)
        assert np.array_equal(p.a0, ref.a0)
        assert np.array_equal(p.kkt_rounds, ref.kkt_rounds)
        assert np.array_equal(p.cols_scanned, ref.cols_scanned)
    op = oracle.fit_path(inst, inst.y, lams, alpha=alpha, tol=1e-11)
    B, Bo = paths[0].dense(inst.p), op.beta
    for k in range(len(lams)):
        sc = np.abs(Bo[:, k]).max()
        assert np.abs(B[:, k] - Bo[:, k]).max() <= 1e-5 * sc or sc == 0.0


def test_sharded_screening_policies_and_cv():
    inst = synth.random_instance(120, 400, dtype=np.float32, seed=5, kind="corr", n_true=8)
    G = 3
    d1 = bl.Design(inst.host_X(), inst.n)
    lams = synth.lambda_grid(d1.lambda_max(inst.y), 20, 0.1)
    ds = sharded_designs(inst, G)
    for screen in ("none", "ssr", "hybrid"):
        ref = d1.fit_path(inst.y, lams, tol=1e-9, screen=screen)
        paths = run_ranks(G, lambda r: ds[r].fit_path(inst.y, lams, tol=1e-9, screen=screen))
        for p in paths:
            assert np.array_equal(p.feat, ref.feat) and np.array_equal(p.beta_std, ref.beta_std), screen
    ref = d1.cv(inst.y, lams, K=4, seed=3, tol=1e-9)
    cvs = run_ranks(G, lambda r: ds[r].cv(inst.y, lams, K=4, seed=3, tol=1e-9))
    for c in cvs:
        assert np.array_equal(c.fold_id, ref.fold_id)
        assert np.array_equal(c.cve, ref.cve) and np.array_equal(c.cvse, ref.cvse)
        assert c.lambda_min_index == ref.lambda_min_index


def test_sharded_rejects_bad_layout():
    inst = synth.random_instance(60, 50, seed=2)
    key = os.urandom(128)
    Xh = inst.host_X()

    def mk(r):   # rank 1 claims an offset that leaves a gap
        j0, j1 = (0, 20) if r == 0 else (25, 50)
        try:
            bl.Design(np.ascontiguousarray(Xh[j0:j1]), inst.n, dist=bl.loopback_dist(r, 2, (j0, j1), 50, key))
        except bl.BLError as e:
            return e.code
        return 0
    codes = run_ranks(2, mk)
    assert all(c == bl.BL_ERR_ARG for c in codes)


@pytest.mark.parametrize("dtype,cv_mode", [(np.int8, "batched"), (np.float64, "independent"),
                                           (np.float32, "batched_fma")])
def test_sharded_cv_modes_are_G_invariant(dtype, cv_mode):
    """Lockstep CV on a column-sharded design (every fit's round exchanged in one collective,
    SURVEY 8(e)) and the independent-fits mode: bitwise the single-GPU CV."""
    kind = "geno" if dtype == np.int8 else "corr"
    inst = synth.random_instance(110, 500, dtype=dtype, seed=6, kind=kind, n_true=8)
    G = 2
    d1 = bl.Design(inst.host_X(), inst.n)
    lams = synth.lambda_grid(d1.lambda_max(inst.y, 0.5), 15, 0.1)
    ref = d1.cv(inst.y, lams, K=5, alpha=0.5, seed=4, tol=1e-9, cv_mode=cv_mode)
    ds = sharded_designs(inst, G)
    cvs = run_ranks(G, lambda r: ds[r].cv(inst.y, lams, K=5, alpha=0.5, seed=4, tol=1e-9, cv_mode=cv_mode))
    for c in cvs:
        assert np.array_equal(c.cve, ref.cve) and np.array_equal(c.cvse, ref.cvse)
        assert np.array_equal(c.full.beta_std, ref.full.beta_std)


def test_sharded_design_rejects_a_concurrent_call():
    """A multi-rank design accepts one call at a time (include/bl.h): while rank 0 waits in a
    collective of one fit, a second fit on the same rank's design returns BL_ERR_ARG at once."""
    import time
    inst = synth.random_instance(100, 300, dtype=np.float32, seed=8, kind="corr", n_true=6)
    ds = sharded_designs(inst, 2)
    lams = synth.lambda_grid(bl.Design(inst.host_X(), inst.n).lambda_max(inst.y), 10, 0.2)
    out = {}

    def first():
        out["a"] = ds[0].fit_path(inst.y, lams, tol=1e-9)

    t = threading.Thread(target=first)
    t.start()
    time.sleep(1.0)                      # rank 0 is now blocked in its first collective
    with pytest.raises(bl.BLError) as e:
        ds[0].fit_path(inst.y, lams, tol=1e-9)
    assert e.value.code == bl.BL_ERR_ARG
    ds[1].fit_path(inst.y, lams, tol=1e-9)   # rank 1 joins: the first fit completes
    t.join(timeout=300)
    assert "a" in out and out["a"].n_converged == len(lams)
