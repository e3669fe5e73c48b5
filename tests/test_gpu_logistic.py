"""NEXT-3: the penalised logistic path (bl_fit_path_binomial) against the fp64 oracle
(oracle.fit_path_binomial, pinned in test_oracle_pins.py).

Tolerances as the linear path (BASELINE north star):
  * per lambda  max|beta_gpu - beta_oracle| <= 1e-5 max|beta_oracle|
  * relative objective difference <= 1e-7 (both evaluated by the oracle, QL1)
  * identical active sets {|beta| >= 1e-8}, KKT-tight mismatches excused (Q20)
  * intercept on the original scale within 1e-6 (absolute, log-odds units)
"""
import math
import os
import threading

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

bl = pytest.importorskip("paper_1701_05936_b200.bl")


def _std(inst):
    Xf = inst.host_X()[:, :inst.n].T.astype(np.float64)
    c, s = oracle.column_stats(inst)
    return c, s


def _logit_z(inst, b0, beta):
    """z_j = x~_j'(y - p^)/n at (b0, beta) -- the logistic KKT quantity (QL1), numpy, explicit
    standardisation (population SD) -- for the Q20 active-set rule."""
    X = inst.dense()
    sd = X.std(0)
    live = np.ptp(X, axis=0) > 0
    Xs = np.zeros_like(X)
    Xs[:, live] = (X[:, live] - X[:, live].mean(0)) / sd[live]
    eta = b0 + Xs @ beta
    return Xs.T @ (inst.y - 1.0 / (1.0 + np.exp(-eta))) / inst.n


def compare(inst, gp, op, alpha, lams):
    c, s = oracle.column_stats(inst)
    Bg = gp.dense(inst.p)
    assert gp.n_converged == op.n_converged == len(lams)
    for k, lam in enumerate(lams):
        bo, bg = op.beta[:, k], Bg[:, k]
        scale = np.abs(bo).max()
        if scale == 0.0:
            assert np.all(bg == 0.0), k
        else:
            err = np.abs(bg - bo).max() / scale
            assert err <= 1e-5, f"lambda {k}: rel beta err {err:.3e}"
        live = s > 0
        b0g = gp.a0[k] + np.sum(bg[live] * c[live] / s[live])      # back to the standardised intercept
        assert abs(b0g - op.b0[k]) <= 1e-6, (k, b0g, op.b0[k])
        assert abs(gp.a0[k] - op.a0[k]) <= 1e-6 * max(1.0, abs(op.a0[k]))
        qo = oracle.objective_binomial(inst, inst.y, op.b0[k], bo, lam, alpha)
        qg = oracle.objective_binomial(inst, inst.y, b0g, bg, lam, alpha)
        assert abs(qg - qo) / qo <= 1e-7, f"lambda {k}: RD {(qg - qo) / qo:.3e}"
        assert abs(gp.obj[k] - qg) <= 1e-9 * qg
        ao, ag = np.abs(bo) >= 1e-8, np.abs(bg) >= 1e-8
        if not np.array_equal(ao, ag):          # Q20: excused only for a KKT-tight feature
            z = _logit_z(inst, op.b0[k], bo)
            bad = np.flatnonzero(ao != ag)
            slack = np.abs(np.abs(z[bad]) - alpha * lam)
            assert np.all(slack <= 1e-9), (k, bad, slack)


@pytest.mark.parametrize("dtype,alpha,screen,cd", [
    (np.float64, 1.0, "ssr", "auto"), (np.float32, 1.0, "ssr", "auto"), (np.int8, 1.0, "ssr", "auto"),
    (np.float32, 0.5, "ssr", "auto"), (np.float64, 0.5, "none", "auto"), (np.int8, 0.3, "hybrid", "auto"),
    (np.float64, 1.0, "ssr", "residual"), (np.int8, 0.5, "ssr", "residual"), (np.float32, 1.0, "none", "residual")])
def test_logistic_path_parity(dtype, alpha, screen, cd):
    kind = "geno" if dtype == np.int8 else "corr"
    inst = synth.logistic_instance(157, 613, dtype=dtype, seed=7, kind=kind, n_true=10, scale=1.5, const_cols=3)
    d = bl.Design(inst.host_X(), inst.n)
    lm = d.lambda_max(inst.y, alpha)
    lams = synth.lambda_grid(lm, 30, 0.15)
    op = oracle.fit_path_binomial(inst, inst.y, lams, alpha=alpha, tol=1e-12)
    gp = d.fit_path_binomial(inst.y, lams, alpha=alpha, tol=1e-10, screen=screen, cd=cd)
    compare(inst, gp, op, alpha, lams)
    assert np.all(gp.outer[1:] >= 1)


@pytest.mark.parametrize("n,cd", [(1500, "residual"), (5000, "residual"), (9000, "residual"), (9000, "auto")])
def test_logistic_row_layouts(n, cd):
    """n spans the 4 / 8 / 16 rows-per-thread variants of the CD kernel with ragged tails."""
    inst = synth.logistic_instance(n, 120, dtype=np.float32, seed=n, n_true=8, scale=1.0)
    d = bl.Design(inst.host_X(), inst.n)
    lm = d.lambda_max(inst.y)
    lams = synth.lambda_grid(lm, 12, 0.1)
    op = oracle.fit_path_binomial(inst, inst.y, lams, tol=1e-12)
    gp = d.fit_path_binomial(inst.y, lams, tol=1e-10, cd=cd)
    compare(inst, gp, op, 1.0, lams)


def test_logistic_null_model_and_screening():
    inst = synth.logistic_instance(200, 3000, dtype=np.float32, seed=3, n_true=10, scale=2.0)
    d = bl.Design(inst.host_X(), inst.n)
    lm = d.lambda_max(inst.y)
    lams = synth.lambda_grid(lm, 25, 0.2)
    ss = d.fit_path_binomial(inst.y, lams, tol=1e-10, screen="ssr")
    hy = d.fit_path_binomial(inst.y, lams, tol=1e-10, screen="hybrid")
    no = d.fit_path_binomial(inst.y, lams, tol=1e-10, screen="none")
    yb = inst.y.mean()
    assert ss.col_ptr[1] == 0 and abs(ss.a0[0] - math.log(yb / (1 - yb))) <= 1e-14
    np.testing.assert_array_equal(ss.dense(inst.p), hy.dense(inst.p))     # QL3: hybrid runs as SSR
    assert np.abs(ss.dense(inst.p) - no.dense(inst.p)).max() <= 1e-7 * max(1.0, np.abs(no.dense(inst.p)).max())
    # KKT on the full design at every lambda (gradient recomputed in numpy)
    Xf = inst.host_X()[:, :inst.n].T.astype(np.float64)
    Xs = (Xf - Xf.mean(0)) / Xf.std(0)
    B = ss.dense(inst.p)
    c, s = Xf.mean(0), Xf.std(0)
    for k, lam in enumerate(lams):
        b = B[:, k]
        eta = ss.a0[k] + np.sum(b * c / s) + Xs @ b
        g = Xs.T @ (inst.y - 0.5 * (1 + np.tanh(0.5 * eta))) / inst.n
        nz = b != 0
        assert np.all(np.abs(g[~nz]) <= lam + 1e-6)
        assert np.all(np.abs(g[nz] - lam * np.sign(b[nz])) <= 1e-6)


def test_logistic_input_errors():
    inst = synth.logistic_instance(50, 20, seed=1)
    d = bl.Design(inst.host_X(), inst.n)
    lams = np.array([0.1, 0.05])
    y = inst.y.copy(); y[3] = 2.0
    with pytest.raises(bl.BLError) as e:
        d.fit_path_binomial(y, lams)
    assert e.value.code == bl.BL_ERR_ARG
    with pytest.raises(bl.BLError) as e:
        d.fit_path_binomial(np.zeros(inst.n), lams)
    assert e.value.code == bl.BL_ERR_DEGENERATE


def test_logistic_sharded_is_G_invariant():
    """Column-sharded logistic path (loopback transport): bitwise equal to one GPU."""
    inst = synth.logistic_instance(140, 500, dtype=np.float32, seed=9, kind="corr", n_true=8, scale=1.5)
    d1 = bl.Design(inst.host_X(), inst.n)
    lm = d1.lambda_max(inst.y)
    lams = synth.lambda_grid(lm, 20, 0.15)
    ref = d1.fit_path_binomial(inst.y, lams, tol=1e-10)
    G = 2
    key = os.urandom(128)
    Xh = inst.host_X()
    out, errs = [None] * G, []

    def work(r):
        try:
            j0, j1 = bl.shard_range(inst.p, G, r)
            d = bl.Design(np.ascontiguousarray(Xh[j0:j1]), inst.n, dist=bl.loopback_dist(r, G, (j0, j1), inst.p, key))
            out[r] = d.fit_path_binomial(inst.y, lams, tol=1e-10)
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))
    th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    [t.start() for t in th]
    [t.join(timeout=600) for t in th]
    assert not errs, errs
    for r in range(G):
        np.testing.assert_array_equal(out[r].dense(inst.p), ref.dense(inst.p))
        np.testing.assert_array_equal(out[r].a0, ref.a0)


def test_logistic_single_cta_covariance_form():
    """The single-CTA covariance-form kernel (k_cd_logit_gram, selected with BL_LOGIT_G7=0,
    read once per process) against the oracle, in a child process."""
    import subprocess
    import sys
    code = (
        "import numpy as np, oracle, synth\n"
        "from paper_1701_05936_b200 import bl\n"
        "inst = synth.logistic_instance(157, 613, dtype=np.float32, seed=7, kind='corr', n_true=10, scale=1.5)\n"
        "d = bl.Design(inst.host_X(), inst.n)\n"
        "for alpha in (1.0, 0.5):\n"
        "    lams = synth.lambda_grid(d.lambda_max(inst.y, alpha), 20, 0.15)\n"
        "    op = oracle.fit_path_binomial(inst, inst.y, lams, alpha=alpha, tol=1e-12)\n"
        "    B = d.fit_path_binomial(inst.y, lams, alpha=alpha, tol=1e-10).dense(inst.p)\n"
        "    for k in range(len(lams)):\n"
        "        sc = np.abs(op.beta[:, k]).max()\n"
        "        assert np.abs(B[:, k] - op.beta[:, k]).max() <= 1e-5 * sc or sc == 0.0, (alpha, k)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BL_LOGIT_G7="0", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
