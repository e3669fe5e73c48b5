"""Pins for the fp64 CPU oracle (oracle/oracle.c), against things other than itself:
printed worked examples (tests/golden, SPEC/PAPER cited), closed forms, brute
force on tiny inputs, a library routine (scikit-learn enet_path) that minimises
the identical objective, textbook limits, and the independent vector form of
the EDPP safe rule.  CPU only."""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def std_cols(X):
    """numpy standardisation used ONLY to build pins (population SD)."""
    X = np.asarray(X, dtype=np.float64)
    return (X - X.mean(0)) / X.std(0)


# ------------------------------------------------------------------ worked examples

@pytest.mark.parametrize("ex", GOLD["column_stats"])
def test_stats_worked_examples(ex):
    x = np.array(ex["x"], dtype=np.float64)[:, None]
    c, s = oracle.column_stats(x)
    assert c[0] == pytest.approx(ex["c"], abs=1e-15)
    assert s[0] ** 2 == pytest.approx(ex["s2"], abs=1e-15)


def test_lambda_max_worked_example():
    ex = GOLD["lambda_max"][0]
    x = np.array(ex["x"])[:, None]
    lm, js = oracle.lambda_max(x, np.array(ex["y"]), ex["alpha"])
    assert lm == pytest.approx(ex["value"], rel=1e-15) and js == 0


@pytest.mark.parametrize("ex", GOLD["lambda_grid_linear"])
def test_lambda_grid_worked_examples(ex):
    g = synth.lambda_grid(ex["lambda_max"], ex["K"], ex["ratio"], "linear")
    np.testing.assert_allclose(g, ex["value"], rtol=1e-14)


@pytest.mark.parametrize("ex", GOLD["cd_update"])
def test_cd_update_worked_examples(ex):
    # p = 1, n = 2: x = (-1, 1) -> x~ = x, y = (-z, z) -> x~'y~/n = z exactly.
    z = ex["z"]
    x = np.array([[-1.0], [1.0]])
    y = np.array([-z, z])
    res = oracle.fit_path(x, y, [ex["lambda"]], alpha=ex["alpha"], tol=1e-14)
    assert res.beta[0, 0] == pytest.approx(ex["value"], abs=1e-14)


def test_folds_worked_example_and_properties():
    ex = GOLD["folds"][0]
    f = oracle.folds(ex["n"], ex["K"], 1234)
    assert sorted(np.bincount(f, minlength=ex["K"]).tolist()) == ex["fold_sizes"]
    for n, K in [(10, 3), (103, 10), (2898, 10)]:
        f1, f2 = oracle.folds(n, K, 7), oracle.folds(n, K, 7)
        assert np.array_equal(f1, f2)                       # deterministic under the seed
        cnt = np.bincount(f1, minlength=K)
        assert cnt.min() >= 1 and cnt.max() - cnt.min() <= 1  # partition, balanced, nonempty
        assert not np.array_equal(f1, oracle.folds(n, K, 8))


# ------------------------------------------------------------------ closed forms

def test_lambda_max_is_the_kink_of_the_path():
    """At lambda_max the solution is 0; just below it exactly j* enters."""
    inst = synth.random_instance(40, 30, seed=3)
    for alpha in (1.0, 0.5):
        lm, js = oracle.lambda_max(inst, inst.y, alpha)
        Xs = std_cols(inst.dense())
        yt = inst.y - inst.y.mean()
        assert lm == pytest.approx(np.abs(Xs.T @ yt).max() / (inst.n * alpha), rel=1e-12)
        res = oracle.fit_path(inst, inst.y, [lm, lm * (1 - 1e-6)], alpha=alpha, tol=1e-12)
        assert np.all(res.beta[:, 0] == 0)
        assert np.flatnonzero(res.beta[:, 1]).tolist() == [js]
        assert res.a0[0] == pytest.approx(inst.y.mean(), rel=1e-14)   # null model


@pytest.mark.parametrize("alpha", [1.0, 0.5, 0.1])
def test_single_feature_closed_form(alpha):
    """p = 1: beta(lambda) = S(x~'y~/n, lambda alpha)/(1 + lambda(1-alpha))."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((25, 1)) * 3 + 1
    y = 2 * x[:, 0] + rng.standard_normal(25)
    xs = std_cols(x)[:, 0]
    z = xs @ (y - y.mean()) / 25
    lams = np.abs(z) / alpha * np.array([1.5, 1.0, 0.7, 0.3, 0.01])
    res = oracle.fit_path(x, y, lams, alpha=alpha, tol=1e-14)
    expect = np.sign(z) * np.maximum(np.abs(z) - lams * alpha, 0) / (1 + lams * (1 - alpha))
    np.testing.assert_allclose(res.beta[0], expect, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_orthogonal_design_closed_form(alpha):
    """X~'X~ = n I: beta_j = S(x~_j'y~/n, lambda alpha)/(1+lambda(1-alpha)) (BASELINE)."""
    n, p = 64, 12
    rng = np.random.default_rng(11)
    Q, _ = np.linalg.qr(np.column_stack([np.ones(n), rng.standard_normal((n, p))]))
    X = math.sqrt(n) * Q[:, 1:]          # centred, population SD 1, orthogonal
    y = X @ rng.standard_normal(p) + rng.standard_normal(n) + 3.0
    z = X.T @ (y - y.mean()) / n
    lm, _ = oracle.lambda_max(X, y, alpha)
    lams = synth.lambda_grid(lm, 20, 0.01)
    res = oracle.fit_path(X, y, lams, alpha=alpha, tol=1e-14)
    expect = np.sign(z)[:, None] * np.maximum(np.abs(z)[:, None] - lams[None] * alpha, 0) \
        / (1 + lams[None] * (1 - alpha))
    np.testing.assert_allclose(res.beta, expect, atol=1e-12)


def brute_force(Xs, yt, lam, alpha):
    """Enumerate support A and signs s (3^p candidates): solve the stationarity
    system (X_A'X_A/n + lam(1-alpha) I) b = X_A'y/n - lam alpha s, keep
    sign-consistent candidates, return the min-objective one (BASELINE)."""
    n, p = Xs.shape
    best, bq = np.zeros(p), 0.5 * yt @ yt / n
    for A in itertools.chain.from_iterable(itertools.combinations(range(p), k) for k in range(1, p + 1)):
        A = list(A)
        XA = Xs[:, A]
        G = XA.T @ XA / n + lam * (1 - alpha) * np.eye(len(A))
        for s in itertools.product((-1.0, 1.0), repeat=len(A)):
            s = np.array(s)
            try:
                b = np.linalg.solve(G, XA.T @ yt / n - lam * alpha * s)
            except np.linalg.LinAlgError:
                continue
            if np.any(np.sign(b) != s):
                continue
            r = yt - XA @ b
            q = 0.5 * r @ r / n + lam * (alpha * np.abs(b).sum() + 0.5 * (1 - alpha) * b @ b)
            if q < bq:
                bq, best = q, np.zeros(p)
                best[A] = b
    return best, bq


@pytest.mark.parametrize("seed,alpha", [(0, 1.0), (1, 0.5), (2, 1.0)])
def test_brute_force_small_p(seed, alpha):
    inst = synth.random_instance(15, 7, seed=seed, kind="corr", n_true=3)
    Xs = std_cols(inst.dense())
    yt = inst.y - inst.y.mean()
    lm, _ = oracle.lambda_max(inst, inst.y, alpha)
    lams = synth.lambda_grid(lm, 6, 0.05)
    res = oracle.fit_path(inst, inst.y, lams, alpha=alpha, tol=1e-13)
    for k, lam in enumerate(lams):
        b, q = brute_force(Xs, yt, lam, alpha)
        np.testing.assert_allclose(res.beta[:, k], b, atol=1e-9)
        assert res.obj[k] == pytest.approx(q, rel=1e-10, abs=1e-14)


@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_matches_sklearn_enet_path(alpha):
    """scikit-learn's enet_path minimises 1/(2n)|y - Xw|^2 + a l1|w|_1 + a(1-l1)/2 |w|^2,
    i.e. Q with a = lambda, l1_ratio = alpha, on X~, y~ (Q2)."""
    from sklearn.linear_model import enet_path
    inst = synth.random_instance(60, 150, seed=21, kind="corr", n_true=8)
    Xs = std_cols(inst.dense())
    yt = inst.y - inst.y.mean()
    lm, _ = oracle.lambda_max(inst, inst.y, alpha)
    lams = synth.lambda_grid(lm, 30, 0.05)
    res = oracle.fit_path(inst, inst.y, lams, alpha=alpha, tol=1e-12)
    _, coefs, _ = enet_path(Xs, yt, l1_ratio=alpha, alphas=lams, tol=1e-14, max_iter=100000)
    for k in range(len(lams)):
        scale = max(1e-12, np.abs(coefs[:, k]).max())
        assert np.abs(res.beta[:, k] - coefs[:, k]).max() <= 1e-6 * scale


def test_small_lambda_limit_is_least_squares():
    inst = synth.random_instance(80, 10, seed=4)
    Xs = std_cols(inst.dense())
    yt = inst.y - inst.y.mean()
    ls = np.linalg.lstsq(Xs, yt, rcond=None)[0]
    lm, _ = oracle.lambda_max(inst, inst.y)
    res = oracle.fit_path(inst, inst.y, synth.lambda_grid(lm, 40, 1e-9), tol=1e-14)
    np.testing.assert_allclose(res.beta[:, -1], ls, rtol=1e-6, atol=1e-8)


def test_objective_pins():
    inst = synth.random_instance(30, 20, seed=8)
    yt = inst.y - inst.y.mean()
    # beta = 0: Q = |y~|^2 / (2n)
    assert oracle.objective(inst, inst.y, np.zeros(20), 0.3, 0.7) == pytest.approx(yt @ yt / 60, rel=1e-14)
    # the oracle's solution is a minimiser: random perturbations never decrease Q
    lm, _ = oracle.lambda_max(inst, inst.y, 0.7)
    res = oracle.fit_path(inst, inst.y, [0.3 * lm], alpha=0.7, tol=1e-14)
    b = res.beta[:, 0]
    q0 = oracle.objective(inst, inst.y, b, 0.3 * lm, 0.7)
    assert q0 == pytest.approx(res.obj[0], rel=1e-12)
    rng = np.random.default_rng(0)
    for _ in range(20):
        assert oracle.objective(inst, inst.y, b + 1e-4 * rng.standard_normal(20), 0.3 * lm, 0.7) >= q0


# ------------------------------------------------------------------ invariants

@pytest.mark.parametrize("kind,dtype,alpha", [("iid", np.float64, 1.0), ("corr", np.float32, 0.5),
                                              ("geno", np.int8, 1.0)])
def test_kkt_holds_along_path(kind, dtype, alpha):
    inst = synth.random_instance(50, 120, dtype=dtype, seed=9, kind=kind, const_cols=2)
    lm, _ = oracle.lambda_max(inst, inst.y, alpha)
    lams = synth.lambda_grid(lm, 25, 0.05)
    res = oracle.fit_path(inst, inst.y, lams, alpha=alpha, tol=1e-12)
    for k, lam in enumerate(lams):
        zv, nv = oracle.kkt(inst, inst.y, res.beta[:, k], lam, alpha)
        assert zv <= 1e-9 and nv <= 1e-9


def test_plain_and_cycle_active_agree():
    inst = synth.random_instance(40, 60, seed=12, kind="corr")
    lm, _ = oracle.lambda_max(inst, inst.y)
    lams = synth.lambda_grid(lm, 15, 0.1)
    a = oracle.fit_path(inst, inst.y, lams, tol=1e-13, cycle_active=False)
    b = oracle.fit_path(inst, inst.y, lams, tol=1e-13, cycle_active=True)
    np.testing.assert_allclose(a.beta, b.beta, atol=1e-10)


def test_int8_equals_widened_copy():
    inst = synth.random_instance(30, 40, dtype=np.int8, seed=2, kind="geno")
    Xd = inst.dense().astype(np.float64)
    lm, _ = oracle.lambda_max(inst, inst.y)
    lams = synth.lambda_grid(lm, 10, 0.1)
    a = oracle.fit_path(inst, inst.y, lams, tol=1e-12)
    b = oracle.fit_path(Xd, inst.y, lams, tol=1e-12)
    assert np.array_equal(a.beta, b.beta)


def test_row_subset_equals_submatrix():
    """Mask rows (P:278 row-index vectors) == fitting the row-subset matrix."""
    inst = synth.random_instance(40, 25, seed=13)
    train = np.ones(40, dtype=bool)
    train[[1, 5, 6, 17, 30, 39]] = False
    X = inst.dense()
    lm, _ = oracle.lambda_max(X[train], inst.y[train])
    lams = synth.lambda_grid(lm, 10, 0.1)
    a = oracle.fit_path(inst, inst.y, lams, tol=1e-12, train=train, want_resid=True)
    b = oracle.fit_path(X[train], inst.y[train], lams, tol=1e-12, want_resid=True)
    np.testing.assert_allclose(a.beta, b.beta, atol=1e-13)
    np.testing.assert_allclose(a.resid[:, train], b.resid, atol=1e-12)
    np.testing.assert_allclose(a.obj, b.obj, rtol=1e-13)


def test_intercept_unstandardisation():
    """y - resid == a0 + X beta_orig with beta_orig = beta/s (Q4)."""
    inst = synth.random_instance(30, 15, seed=14, mean_shift=2.0)
    X = inst.dense()
    lm, _ = oracle.lambda_max(inst, inst.y)
    lams = synth.lambda_grid(lm, 8, 0.1)
    res = oracle.fit_path(inst, inst.y, lams, tol=1e-13, want_resid=True)
    s = X.std(0)
    for k in range(len(lams)):
        fit = res.a0[k] + X @ (res.beta[:, k] / s)
        np.testing.assert_allclose(inst.y - res.resid[k], fit, atol=1e-11)


def test_cv_null_model_closed_form():
    """At lambda >= lambda_max of every fold the fit is the training mean, so
    E_i = (y_i - mean(y[train of fold(i)]))^2 exactly."""
    inst = synth.random_instance(30, 12, seed=15)
    f = oracle.folds(30, 5, 1234)
    lm, _ = oracle.lambda_max(inst, inst.y)
    lams = np.array([100 * lm, 50 * lm])
    E, cve, cvse, lmin = oracle.cv(inst, inst.y, f, 5, lams)
    for i in range(30):
        tr = f != f[i]
        assert E[0, i] == pytest.approx((inst.y[i] - inst.y[tr].mean()) ** 2, rel=1e-13)
    assert cve[0] == pytest.approx(E[0].mean(), rel=1e-14)
    assert cvse[0] == pytest.approx(E[0].std(ddof=1) / math.sqrt(30), rel=1e-12)


def test_degenerate_inputs():
    X = np.random.default_rng(0).standard_normal((10, 4))
    with pytest.raises(oracle.OracleError) as e:
        oracle.lambda_max(X, np.ones(10))
    assert e.value.code == oracle.ERR_DEGENERATE
    with pytest.raises(oracle.OracleError) as e:
        oracle.fit_path(X, np.arange(10.0), [1.0, 2.0])     # not decreasing
    assert e.value.code == oracle.ERR_ARG
    with pytest.raises(oracle.OracleError) as e:
        oracle.fit_path(X, np.arange(10.0), [1.0], alpha=0.0)
    assert e.value.code == oracle.ERR_ARG


# ------------------------------------------------------------------ BEDPP

def edpp_vector_discard(Xs, yt, lam, alpha):
    """Independent vector form of the basic EDPP test (the rule of
    P:211's 'JMLR:v16:wang15a'), on the augmented design for alpha < 1:
    theta0 = y/lam'max, v1 = sign(x*'y) x*, v2 = y/lam' - theta0,
    v2perp = v2 - <v1,v2>/|v1|^2 v1; discard iff |x_j'(theta0 + v2perp/2)| < 1 - |v2perp| |x_j| / 2."""
    n, p = Xs.shape
    nu = math.sqrt(n * lam * (1 - alpha))
    Xa = np.vstack([Xs, nu * np.eye(p)])
    ya = np.concatenate([yt, np.zeros(p)])
    a = Xa.T @ ya
    js = int(np.argmax(np.abs(a)))
    lmax_p = abs(a[js])
    lp = n * alpha * lam
    th0 = ya / lmax_p
    v1 = np.sign(a[js]) * Xa[:, js]
    v2 = ya / lp - th0
    v2p = v2 - (v1 @ v2) / (v1 @ v1) * v1
    lhs = np.abs(Xa.T @ (th0 + 0.5 * v2p))
    rhs = 1 - 0.5 * np.linalg.norm(v2p) * np.linalg.norm(Xa, axis=0)
    d = lhs < rhs
    d[js] = False
    return d, lhs, rhs


@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_bedpp_scalar_form_equals_vector_form(alpha):
    disagree = 0
    total = 0
    for seed in range(12):
        inst = synth.random_instance(30 + seed, 60 + 5 * seed, seed=100 + seed, kind="corr" if seed % 2 else "iid")
        Xs = std_cols(inst.dense())
        yt = inst.y - inst.y.mean()
        lm, _ = oracle.lambda_max(inst, inst.y, alpha)
        for lam in synth.lambda_grid(lm, 12, 0.2)[1:]:
            d_or = oracle.bedpp_discard(inst, inst.y, alpha, lam)
            d_vec, lhs, rhs = edpp_vector_discard(Xs, yt, lam, alpha)
            tight = np.abs(lhs - rhs) <= 1e-9 * (1 + np.abs(rhs))
            bad = (d_or != d_vec) & ~tight
            disagree += int(bad.sum())
            total += d_or.size
            assert not np.any(d_or & ~d_vec & ~tight)   # never more aggressive than the vector form
    assert disagree == 0, f"{disagree}/{total}"


def test_bedpp_at_lambda_max_discards_all_but_star():
    inst = synth.random_instance(40, 50, seed=31)
    for alpha in (1.0, 0.5):
        lm, js = oracle.lambda_max(inst, inst.y, alpha)
        d = oracle.bedpp_discard(inst, inst.y, alpha, lm)
        assert not d[js] and d.sum() == 49


@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_bedpp_is_safe(alpha):
    """Zero tolerance: never discards a feature whose oracle coefficient is
    nonzero (P:211 'guaranteed to never incorrectly screen')."""
    for seed in range(100):
        kinds = ["iid", "corr", "geno"]
        inst = synth.random_instance(20 + seed % 30, 40 + 3 * seed, seed=1000 + seed,
                                     kind=kinds[seed % 3], dtype=np.int8 if seed % 3 == 2 else np.float64)
        lm, _ = oracle.lambda_max(inst, inst.y, alpha)
        lams = synth.lambda_grid(lm, 10, 0.3)
        res = oracle.fit_path(inst, inst.y, lams, alpha=alpha, tol=1e-12)
        for k, lam in enumerate(lams):
            d = oracle.bedpp_discard(inst, inst.y, alpha, lam)
            assert not np.any(d & (res.beta[:, k] != 0)), (seed, k)


def test_bedpp_power_shape():
    """Qualitative P:211: strong discarding near lambda_max, ~none far below 0.45."""
    inst = synth.random_instance(200, 1000, seed=3)
    lm, _ = oracle.lambda_max(inst, inst.y)
    assert oracle.bedpp_discard(inst, inst.y, 1.0, 0.97 * lm).mean() > 0.9
    assert oracle.bedpp_discard(inst, inst.y, 1.0, 0.2 * lm).mean() < 0.05


# ------------------------------------------------------------ NEXT-3: logistic path
# Pins for oracle.fit_path_binomial (QL1-QL6): the null model and lambda_max closed
# forms, the KKT conditions recomputed here in numpy, an independent minimiser
# (scipy L-BFGS-B on the split-variable form of QL1), label-flip symmetry and the
# input errors.

def _logit_fixture(n=80, p=10, seed=3, kind="iid", dtype=np.float64, const_cols=0):
    return synth.logistic_instance(n, p, dtype=dtype, seed=seed, kind=kind, n_true=4, scale=2.0,
                                   const_cols=const_cols)


def _np_std(inst):
    Xf = inst.host_X()[:, :inst.n].T.astype(np.float64)
    sd = Xf.std(0)
    return np.where(sd > 0, (Xf - Xf.mean(0)) / np.where(sd > 0, sd, 1.0), 0.0), sd > 0


def _sig(t):
    return 0.5 * (1.0 + np.tanh(0.5 * t))


def test_binomial_null_model_and_lambda_max():
    inst = _logit_fixture()
    Xs, live = _np_std(inst)
    y = inst.y
    ybar = y.mean()
    lmax = np.abs(Xs.T @ (y - ybar)).max() / inst.n            # QL2, alpha = 1
    lm_or, _ = oracle.lambda_max(inst, y, 1.0)                 # same closed form as the linear model
    assert abs(lm_or - lmax) <= 1e-12 * lmax
    lams = lmax * np.array([1.0, 0.999, 0.9])
    op = oracle.fit_path_binomial(inst, y, lams, tol=1e-12)
    assert np.all(op.beta[:, 0] == 0.0)
    assert abs(op.b0[0] - math.log(ybar / (1 - ybar))) <= 1e-14
    assert abs(op.a0[0] - math.log(ybar / (1 - ybar))) <= 1e-14
    # just below lambda_max only the argmax feature enters
    jstar = int(np.argmax(np.abs(Xs.T @ (y - ybar))))
    assert set(np.flatnonzero(op.beta[:, 1])) == {jstar}


@pytest.mark.parametrize("alpha", [1.0, 0.5])
@pytest.mark.parametrize("kind,dtype", [("iid", np.float64), ("corr", np.float32), ("geno", np.int8)])
def test_binomial_kkt_along_path(alpha, kind, dtype):
    inst = _logit_fixture(n=120, p=30, seed=5, kind=kind, dtype=dtype, const_cols=2)
    Xs, live = _np_std(inst)
    y = inst.y
    lmax = np.abs(Xs.T @ (y - y.mean())).max() / (inst.n * alpha)
    lams = synth.lambda_grid(lmax, 25, 0.05)
    op = oracle.fit_path_binomial(inst, y, lams, alpha=alpha, tol=1e-12)
    assert op.n_converged == len(lams)
    for k, lam in enumerate(lams):
        b = op.beta[:, k]
        assert np.all(b[~live] == 0.0)
        eta = op.b0[k] + Xs @ b
        g = Xs.T @ (y - _sig(eta)) / inst.n                     # gradient of the mean log-likelihood
        assert abs(np.sum(y - _sig(eta))) / inst.n <= 1e-9     # unpenalised intercept
        nz = b != 0
        assert np.all(np.abs(g[~nz & live]) <= alpha * lam + 1e-9)
        assert np.all(np.abs(g[nz] - alpha * lam * np.sign(b[nz]) - lam * (1 - alpha) * b[nz]) <= 1e-9)
        # objective evaluator = the QL1 formula
        q = np.mean(np.logaddexp(0.0, eta) - y * eta) + lam * (alpha * np.abs(b).sum() + 0.5 * (1 - alpha) * b @ b)
        assert abs(oracle.objective_binomial(inst, y, op.b0[k], b, lam, alpha) - q) <= 1e-12 * abs(q)
        assert abs(op.obj[k] - q) <= 1e-10 * abs(q)


@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_binomial_matches_lbfgsb(alpha):
    """Independent minimiser of QL1: L-BFGS-B over (b0, b+, b-) with b+, b- >= 0."""
    from scipy.optimize import minimize
    inst = _logit_fixture(n=90, p=8, seed=11)
    Xs, _ = _np_std(inst)
    y, n, p = inst.y, inst.n, Xs.shape[1]
    lmax = np.abs(Xs.T @ (y - y.mean())).max() / (n * alpha)
    lams = lmax * np.array([0.8, 0.5, 0.25, 0.1])
    op = oracle.fit_path_binomial(inst, y, lams, alpha=alpha, tol=1e-13)
    for k, lam in enumerate(lams):
        def f(t):
            b0, bp, bm = t[0], t[1:p + 1], t[p + 1:]
            b = bp - bm
            eta = b0 + Xs @ b
            mu = _sig(eta)
            val = np.mean(np.logaddexp(0.0, eta) - y * eta) + lam * (alpha * (bp + bm).sum() + 0.5 * (1 - alpha) * b @ b)
            gb = Xs.T @ (mu - y) / n + lam * (1 - alpha) * b
            return val, np.concatenate([[np.mean(mu - y)], gb + lam * alpha, -gb + lam * alpha])
        res = minimize(f, np.zeros(2 * p + 1), jac=True, method="L-BFGS-B",
                       bounds=[(None, None)] + [(0, None)] * (2 * p),
                       options=dict(ftol=1e-15, gtol=1e-12, maxiter=20000))
        b_ref = res.x[1:p + 1] - res.x[p + 1:]
        scale = max(np.abs(b_ref).max(), 1e-3)
        assert np.abs(op.beta[:, k] - b_ref).max() <= 1e-5 * scale, (k, op.beta[:, k], b_ref)
        assert abs(op.b0[k] - res.x[0]) <= 1e-5
        assert op.obj[k] <= res.fun + 1e-12


def test_binomial_label_flip_symmetry():
    """y -> 1 - y maps the solution (b0, b) to (-b0, -b) (the loss is odd in eta <-> y)."""
    inst = _logit_fixture(n=70, p=12, seed=21)
    lm, _ = oracle.lambda_max(inst, inst.y, 1.0)
    lams = synth.lambda_grid(lm, 12, 0.1)
    a = oracle.fit_path_binomial(inst, inst.y, lams, tol=1e-13)
    b = oracle.fit_path_binomial(inst, 1.0 - inst.y, lams, tol=1e-13)
    np.testing.assert_allclose(a.beta, -b.beta, rtol=0, atol=1e-9)
    np.testing.assert_allclose(a.b0, -b.b0, rtol=0, atol=1e-9)
    np.testing.assert_allclose(a.obj, b.obj, rtol=1e-12)


def test_binomial_plain_and_cycle_active_agree():
    inst = _logit_fixture(n=60, p=15, seed=8, kind="corr")
    lm, _ = oracle.lambda_max(inst, inst.y, 1.0)
    lams = synth.lambda_grid(lm, 10, 0.1)
    a = oracle.fit_path_binomial(inst, inst.y, lams, tol=1e-13, cycle_active=True)
    b = oracle.fit_path_binomial(inst, inst.y, lams, tol=1e-13, cycle_active=False)
    np.testing.assert_allclose(a.beta, b.beta, rtol=0, atol=1e-9)


def test_binomial_input_errors():
    inst = _logit_fixture(n=40, p=5, seed=2)
    lams = np.array([0.1, 0.05])
    y = inst.y.copy(); y[0] = 0.5
    with pytest.raises(oracle.OracleError) as e:
        oracle.fit_path_binomial(inst, y, lams)
    assert e.value.code == oracle.ERR_ARG
    with pytest.raises(oracle.OracleError) as e:
        oracle.fit_path_binomial(inst, np.ones(inst.n), lams)
    assert e.value.code == oracle.ERR_DEGENERATE


# ------------------------------------------------------------------ identities (1)-(3)
# or_std_dots / or_prep form every standardised value explicitly, element by element;
# these pins check them against the paper's identity arithmetic (a different formula,
# evaluated here in numpy) and against SPEC's printed identity examples.

def _identity_stats(X, m):
    """Column mean and population SD over the rows m (numpy; pins only)."""
    Xm = X[m]
    return Xm.mean(0), Xm.std(0)


def test_identity_worked_examples():
    """S:132-142 (identity (1) P:261, identity (2) P:262): x = (1,2,3), x' = (3,2,1):
    x~'x~' = -3, x~'x~ = n; x~'y for y = x: 2 sqrt(3/2); y == 1: 0; r = 0: 0."""
    xx = GOLD["identity_xx"][0]
    xy, x1 = GOLD["identity_xy"]
    X = np.column_stack([xx["xj"], xx["xk"]]).astype(np.float64)
    y = np.array(xy["y"], dtype=np.float64)
    o = oracle.prep(X, y)                          # a_0 = +2.449, a_1 = -2.449: tie -> j* = 0 (lowest)
    assert o["jstar"] == 0
    assert o["a"][0] == pytest.approx(xy["value"], rel=1e-15)
    assert o["a"][1] == pytest.approx(-xy["value"], rel=1e-15)
    assert o["b"][1] == pytest.approx(xx["value"], rel=1e-15)     # x~_1' x~_*  = -3
    assert o["b"][0] == pytest.approx(3.0, rel=1e-15)             # x~_*' x~_*  = n
    # or_std_dots returns x~'v / n_t
    z = oracle.std_dots(X[:, :1], np.array(xy["y"], dtype=np.float64))
    assert 3 * z[0] == pytest.approx(xy["value"], rel=1e-15)
    z1 = oracle.std_dots(X[:, :1], np.array(x1["y"], dtype=np.float64))
    assert abs(z1[0]) <= 1e-15 and x1["value"] == 0.0
    assert np.all(oracle.std_dots(X, np.zeros(3)) == 0.0)


def test_std_dots_and_prep_match_identities():
    """over >= 1000 random small instances (fp64 / fp32 / int8, with and without a
    row mask, with constant columns), the explicit standardisation of or_std_dots and
    or_prep agrees to 1e-12 with the identities of P:261-263:
      (3)  x~_j'v = (x_j'v - c_j sum v) / s_j            (v zero outside the rows)
      (2)  a_j = x~_j'y~ = x_j'y~ / s_j                   (sum y~ = 0)
      (1)  b_j = x~_j'x~_* = (x_j'x_* - n_t c_j c_*) / (s_j s_*),  b_j* = n_t
    A dropped centring term, a missing 1/n_t under a mask or a sign slip fails here."""
    rng = np.random.default_rng(2024)
    count = 0
    for it in range(1000):
        n = int(rng.integers(3, 40))
        p = int(rng.integers(1, 9))
        dt = [np.float64, np.float32, np.int8][it % 3]
        if dt == np.int8:
            X = rng.integers(0, 3, (n, p)).astype(np.int8)
        else:
            X = (rng.standard_normal((n, p)) * rng.uniform(0.2, 5, p) + rng.uniform(-3, 3, p)).astype(dt)
        if it % 7 == 0:
            X[:, 0] = X[0, 0]                      # a constant column
        m = np.ones(n, bool)
        if it % 2:
            m[rng.choice(n, int(rng.integers(0, n - 2)), replace=False)] = False
        train = None if m.all() else m
        Xd = X.astype(np.float64)
        c, s = _identity_stats(Xd, m)
        live = np.ptp(Xd[m], axis=0) > 0          # Q13: constant on the rows <=> s_j = 0 exactly
        s = np.where(live, s, 0.0)
        # identity (3) for a random v (zero outside the rows)
        v = rng.standard_normal(n) * m
        nt = m.sum()
        z = oracle.std_dots(X, v, train)
        zi = np.zeros(p)
        zi[live] = (Xd[:, live].T @ v - c[live] * v.sum()) / (s[live] * nt)
        scale = (np.abs(Xd - c) / np.where(live, s, 1.0)).T @ np.abs(v) / nt
        assert np.all(np.abs(z - zi) <= 1e-12 * np.maximum(scale, 1e-300)), (it, z, zi)
        assert np.all(z[~live] == 0.0)
        # identities (2) and (1) through or_prep
        y = rng.standard_normal(n) + 0.5 * Xd[:, -1]
        yt = (y - y[m].mean()) * m
        if not live.any() or not np.any(np.abs(Xd[:, live].T @ yt) > 0):
            continue
        o = oracle.prep(X, y, 1.0, train)
        a = np.zeros(p)
        a[live] = Xd[:, live].T @ yt / s[live]
        sa = (np.abs(Xd - c) / np.where(live, s, 1.0)).T @ np.abs(yt)
        assert np.all(np.abs(o["a"] - a) <= 1e-12 * np.maximum(sa, 1e-300)), (it, o["a"], a)
        js = o["jstar"]
        assert live[js] and np.abs(a[js]) >= np.abs(a[live]).max() * (1 - 1e-12)
        b = np.zeros(p)
        xs = Xd[m][:, js]
        b[live] = (Xd[m][:, live].T @ xs - nt * c[live] * c[js]) / (s[live] * s[js])
        assert np.all(np.abs(o["b"] - b) <= 1e-12 * nt * (1 + np.abs(c) / np.where(live, s, 1.0)) *
                      (1 + abs(c[js]) / s[js])), (it, o["b"], b)
        assert o["b"][js] == pytest.approx(nt, rel=1e-12)
        assert o["lambda_max"] == pytest.approx(abs(a[js]) / nt, rel=1e-12)
        count += 1
    assert count >= 900


# ------------------------------------------------------------------ KKT audit

@pytest.mark.parametrize("alpha,masked", [(1.0, False), (0.5, True)])
def test_kkt_audit_pins(alpha, masked):
    """or_kkt against closed forms and a numpy recomputation:
      * the null solution at lambda_max has no violation (zv = 0 up to rounding, nv = 0),
        and at 1.25 lambda_max zv = -0.25 alpha lambda_max exactly;
      * at a converged solution zv, nv ~ 0; zeroing one active coordinate j0 (a
        constructed violation) gives, in closed form,
        |z_j0| - alpha lam = |b_j0| (1 + lam (1 - alpha))   (x~_j0'x~_j0 = n_t),
        and zv / nv equal a numpy recomputation from r = y~ - X~ b (explicit) to 1e-12.
    A stale residual, a missing 1/n_t or a sign slip in the nonzero test fails."""
    inst = synth.random_instance(60, 25, seed=71, kind="corr", n_true=6)
    n, p = inst.n, inst.p
    m = np.ones(n, bool)
    if masked:
        m[::5] = False
    train = None if not masked else m
    lm, _ = oracle.lambda_max(inst, inst.y, alpha, train)
    zv, nv = oracle.kkt(inst, inst.y, np.zeros(p), lm, alpha, train)
    assert abs(zv) <= 1e-12 * alpha * lm and nv == 0.0
    zv, nv = oracle.kkt(inst, inst.y, np.zeros(p), 1.25 * lm, alpha, train)
    assert zv == pytest.approx(-0.25 * alpha * lm, rel=1e-11)
    lam = 0.3 * lm
    fit = oracle.fit_path(inst, inst.y, synth.lambda_grid(lm, 12, 0.3), alpha=alpha, tol=1e-13, train=train)
    b = fit.beta[:, -1].copy()
    zv, nv = oracle.kkt(inst, inst.y, b, lam, alpha, train)
    assert zv <= 1e-10 and nv <= 1e-10
    act = np.flatnonzero(b)
    assert act.size >= 2
    j0 = act[np.argmax(np.abs(b[act]))]
    bp = b.copy()
    bp[j0] = 0.0
    zv2, nv2, z2 = oracle.kkt(inst, inst.y, bp, lam, alpha, train, want_z=True)
    assert abs(z2[j0]) - alpha * lam == pytest.approx(abs(b[j0]) * (1 + lam * (1 - alpha)), rel=1e-8)
    # numpy recomputation (explicit standardisation over the rows, population SD)
    Xd = inst.dense()
    Xs = (Xd - Xd[m].mean(0)) / Xd[m].std(0)
    yt = (inst.y - inst.y[m].mean()) * m
    r = (yt - Xs @ bp) * m
    z = Xs.T @ r / m.sum()
    zero = bp == 0
    zv_np = np.max(np.abs(z[zero]) - alpha * lam)
    nz = ~zero
    nv_np = np.max(np.abs(z[nz] - alpha * lam * np.sign(bp[nz]) - lam * (1 - alpha) * bp[nz]))
    assert zv2 == pytest.approx(zv_np, rel=1e-12, abs=1e-14)
    assert nv2 == pytest.approx(nv_np, rel=1e-12, abs=1e-14)
    np.testing.assert_allclose(z2, z, rtol=0, atol=1e-13)


# ------------------------------------------------------------------ host threads

@pytest.mark.parametrize("kind,dtype,alpha", [("corr", np.float32, 1.0), ("iid", np.float64, 0.5),
                                              ("geno", np.int8, 1.0)])
def test_threaded_oracle_is_bitwise_serial(kind, dtype, alpha):
    """The block-speculative threaded pass reproduces the serial iterates bitwise (beta,
    passes, objective), and the chunked session (warm starts across calls) equals one
    call over the whole grid."""
    inst = synth.random_instance(90, 2500, dtype=dtype, seed=81, kind=kind, n_true=10, const_cols=3)
    lm, _ = oracle.lambda_max(inst, inst.y, alpha)
    lams = synth.lambda_grid(lm, 25, 0.05)
    r = np.random.default_rng(3).standard_normal(inst.n)

    def per_column():
        return (oracle.column_stats(inst), oracle.std_dots(inst, r), oracle.prep(inst, inst.y, alpha),
                oracle.lambda_max(inst, inst.y, alpha), oracle.bedpp_discard(inst, inst.y, alpha, 0.7 * lm),
                oracle.kkt(inst, inst.y, np.zeros(inst.p), 0.5 * lm, alpha, want_z=True))
    try:
        oracle.set_threads(1)
        a = oracle.fit_path(inst, inst.y, lams, alpha=alpha, tol=1e-10)
        one = per_column()
        oracle.set_threads(4)
        b = oracle.fit_path(inst, inst.y, lams, alpha=alpha, tol=1e-10)
        four = per_column()
        s = oracle.PathSession(inst, inst.y, alpha)
        parts = [s.run(lams[i:i + 6], tol=1e-10) for i in range(0, len(lams), 6)]
        s.close()
    finally:
        oracle.set_threads(1)
    assert np.array_equal(a.beta, b.beta) and np.array_equal(a.passes, b.passes) and np.array_equal(a.obj, b.obj)
    assert np.array_equal(np.concatenate([q.beta for q in parts], axis=1), a.beta)
    assert np.array_equal(np.concatenate([q.passes for q in parts]), a.passes)
    flat = lambda t: [np.asarray(u) for v in t for u in (v.values() if isinstance(v, dict) else v if isinstance(v, tuple) else (v,))]
    for u, v in zip(flat(one), flat(four)):
        assert np.array_equal(u, v)
