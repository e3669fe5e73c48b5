"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no standardisation used by the
solver, no screening, no CD): it only draws designs X, responses y and builds
the caller-side lambda grid.  Both sides receive the same bytes.

Recipes follow SURVEY.md 8(d) / BASELINE.json configs (stated again in
DESIGN.md section 4).  Layout: a design is stored column-major as an array of
shape (p, ld) -- row j of the array is column j of X -- with ld >= n padded so
every column starts on a 16-byte boundary; padding rows are zero.

Small instances (cfg1, test instances) are drawn with numpy's default_rng.
Large configs (cfg2-cfg5) are drawn in 1000-column blocks with torch generators
seeded by (seed, block), on the GPU when one is present (else on the CPU), so a
column shard is the union of whole blocks and independent of the shard count.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

BLOCK = 1000
_ITEM = {np.dtype(np.float64): 8, np.dtype(np.float32): 4, np.dtype(np.int8): 1}


def padded_ld(n: int, dtype) -> int:
    """Smallest ld >= n with ld * itemsize a multiple of 16 bytes."""
    q = 16 // _ITEM[np.dtype(dtype)]
    return (n + q - 1) // q * q


@dataclasses.dataclass
class Instance:
    name: str
    X: object          # (p, ld) column-major buffer: np.ndarray or torch.Tensor
    n: int
    y: np.ndarray      # (n,) float64
    alpha: float = 1.0
    ratio: float = 0.1
    nlam: int = 100
    tol: float = 1e-7
    spacing: str = "log"
    beta_true: np.ndarray | None = None
    seed: int = 0

    @property
    def p(self) -> int:
        return int(self.X.shape[0])

    @property
    def ld(self) -> int:
        return int(self.X.shape[1])

    @property
    def dtype(self):
        X = self.X
        if isinstance(X, np.ndarray):
            return X.dtype
        import torch
        return {torch.float64: np.dtype(np.float64), torch.float32: np.dtype(np.float32),
                torch.int8: np.dtype(np.int8)}[X.dtype]

    def host_X(self) -> np.ndarray:
        X = self.X
        if isinstance(X, np.ndarray):
            return X
        return X.cpu().numpy()

    def dense(self) -> np.ndarray:
        """(n, p) view of the design (for small instances / numpy pins)."""
        return self.host_X()[:, : self.n].T


def to_colmajor(Xnp: np.ndarray, dtype=None) -> np.ndarray:
    """(n, p) array -> (p, ld) padded column-major buffer."""
    Xnp = np.asarray(Xnp)
    dtype = np.dtype(dtype or Xnp.dtype)
    n, p = Xnp.shape
    ld = padded_ld(n, dtype)
    buf = np.zeros((p, ld), dtype=dtype)
    buf[:, :n] = Xnp.T
    return buf


def lambda_grid(lambda_max: float, nlam: int = 100, ratio: float = 0.1, spacing: str = "log"):
    """Caller-side grid from lambda_max down to ratio*lambda_max (Q5).

    "equally spaced on the scale of lambda/lambda_max":
    log spacing for the BASELINE configs (cfg1 states it), linear kept for
    paper-shaped runs."""
    if nlam == 1:
        return np.array([lambda_max])
    t = np.arange(nlam) / (nlam - 1)
    if spacing == "log":
        return lambda_max * np.exp(t * math.log(ratio))
    return lambda_max * (1.0 - t * (1.0 - ratio))


# ---------------------------------------------------------------- small instances

def random_instance(n, p, dtype=np.float64, seed=0, kind="iid", n_true=None, noise=1.0,
                    const_cols=0, alpha=1.0, mean_shift=0.0):
    """Small seeded instance for parity/pin tests.

    kind: iid N(0,1) | "corr" (shared factor) | "geno" (int8 codes 0/1/2)."""
    rng = np.random.default_rng(seed)
    if kind == "geno":
        maf = rng.uniform(0.05, 0.5, size=p)
        X = (rng.random((n, p)) < maf).astype(np.int8) + (rng.random((n, p)) < maf).astype(np.int8)
        Xf = X.astype(np.float64)
    else:
        Xf = rng.standard_normal((n, p))
        if kind == "corr":
            Xf = 0.6 * rng.standard_normal((n, 1)) + 0.8 * Xf
        Xf = Xf + mean_shift
        X = Xf.astype(dtype)
        Xf = X.astype(np.float64)
    if const_cols:
        cols = rng.choice(p, size=const_cols, replace=False)
        X[:, cols] = X[0:1, cols]
        Xf = X.astype(np.float64)
    k = n_true if n_true is not None else max(1, min(10, p // 4))
    beta = np.zeros(p)
    idx = rng.choice(p, size=k, replace=False)
    beta[idx] = rng.choice([-1.0, 1.0], size=k) * rng.uniform(0.5, 1.5, size=k)
    y = (Xf - Xf.mean(0)) @ beta + noise * rng.standard_normal(n)
    return Instance(name=f"rand_{kind}_{n}x{p}", X=to_colmajor(X, X.dtype), n=n, y=y,
                    alpha=alpha, beta_true=beta, seed=seed)


# ---------------------------------------------------------------- BASELINE configs

def cfg1(seed=0, n=200, p=1000):
    """BASELINE cfg1: fp64 iid N(0,1), columns standardised before storage; 10
    nonzeros +-1; y = X beta + N(0,1); 100 log lambdas to 0.05; alpha 1."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, p))
    X = (X - X.mean(0)) / X.std(0)
    beta = np.zeros(p)
    idx = rng.choice(p, size=10, replace=False)
    beta[idx] = rng.choice([-1.0, 1.0], size=10)
    y = X @ beta + rng.standard_normal(n)
    return Instance("cfg1", to_colmajor(X), n, y, alpha=1.0, ratio=0.05, tol=1e-7,
                    beta_true=beta, seed=seed)


def _torch_dev(device):
    import torch
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    return torch.device(device)


def _gen(device, seed, block):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed * 1_000_003 + int(block) * 7919 + 17) & 0x7FFF_FFFF_FFFF_FFFF)
    return g


def cfg2(seed=0, n=1000, p=100_000, device=None):
    """BASELINE cfg2: rows N(0, Sigma), Sigma_jk = 0.5^|j-k| (exact stationary
    AR(1) across columns: x_1 = e_1, x_j = 0.5 x_{j-1} + sqrt(.75) e_j), fp32;
    20 nonzeros u + 0.5 sign(u), u ~ U(-1,1); sigma^2 = beta' Sigma beta / 3."""
    import torch
    dev = _torch_dev(device)
    ld = padded_ld(n, np.float32)
    X = torch.zeros((p, ld), dtype=torch.float32, device=dev)
    prev = None
    t_ = torch.arange(BLOCK, device=dev, dtype=torch.float64)
    # x_{j0+t} = 0.5^(t+1) x_{j0-1} + sum_{s<=t} 0.5^(t-s) c_s e_s  (the AR(1) recursion unrolled
    # over a block as one triangular matmul; c_s = sqrt(.75), except c = 1 for global column 0)
    L = torch.tril(0.5 ** (t_[:, None] - t_[None, :]).clamp(min=0)) * math.sqrt(0.75)
    for b in range((p + BLOCK - 1) // BLOCK):
        j0, j1 = b * BLOCK, min(p, (b + 1) * BLOCK)
        m = j1 - j0
        e = torch.randn((m, n), generator=_gen(dev, seed, b), device=dev, dtype=torch.float64)
        Lb = L[:m, :m].clone()
        if b == 0:
            Lb[:, 0] /= math.sqrt(0.75)
        blk = Lb @ e
        if prev is not None:
            blk += (0.5 ** (t_[:m] + 1))[:, None] * prev[None, :]
        prev = blk[m - 1].clone()
        X[j0:j1, :n] = blk.to(torch.float32)
    rng = np.random.default_rng(seed + 1)
    idx = np.sort(rng.choice(p, size=20, replace=False))
    u = rng.uniform(-1, 1, size=20)
    bv = u + 0.5 * np.sign(u)
    beta = np.zeros(p); beta[idx] = bv
    Sig = 0.5 ** np.abs(idx[:, None] - idx[None, :])
    sigma = math.sqrt(bv @ Sig @ bv / 3.0)
    Xb = (X[torch.as_tensor(idx, device=dev), :n].double().T @ torch.as_tensor(bv, device=dev)).cpu().numpy()
    y = Xb + sigma * rng.standard_normal(n)
    return Instance("cfg2", X, n, y, alpha=1.0, ratio=0.1, tol=1e-7, beta_true=beta, seed=seed)


def cfg3(seed=0, n=1000, p=1_000_000, device=None):
    """BASELINE cfg3: x_ij = 0.3 f_{i, j//1000} + sqrt(0.91) e_ij, fp32; 50
    nonzeros +-0.5; y = X beta + N(0,1); alpha 0.5; 100 log lambdas to 0.1."""
    import torch
    dev = _torch_dev(device)
    ld = padded_ld(n, np.float32)
    X = torch.zeros((p, ld), dtype=torch.float32, device=dev)
    for b in range((p + BLOCK - 1) // BLOCK):
        j0, j1 = b * BLOCK, min(p, (b + 1) * BLOCK)
        g = _gen(dev, seed, b)
        f = torch.randn((1, n), generator=g, device=dev, dtype=torch.float32)
        e = torch.randn((j1 - j0, n), generator=g, device=dev, dtype=torch.float32)
        X[j0:j1, :n] = 0.3 * f + math.sqrt(0.91) * e
    rng = np.random.default_rng(seed + 1)
    idx = np.sort(rng.choice(p, size=50, replace=False))
    bv = 0.5 * rng.choice([-1.0, 1.0], size=50)
    beta = np.zeros(p); beta[idx] = bv
    Xb = (X[torch.as_tensor(idx, device=dev), :n].double().T @ torch.as_tensor(bv, device=dev)).cpu().numpy()
    y = Xb + rng.standard_normal(n)
    return Instance("cfg3", X, n, y, alpha=0.5, ratio=0.1, tol=1e-7, beta_true=beta, seed=seed)


def cfg4(seed=0, n=2898, p=1_339_511, device=None):
    """BASELINE cfg4 (GWAS-shaped): int8 codes x_ij ~ Binomial(2, MAF_j), MAF_j ~
    U(0.05, 0.5), no LD; 100 nonzeros N(0, 0.25) on the standardised scale,
    standardised with the GENERATING MAF: y = sum_j beta_j (x_j - 2 MAF_j) /
    sqrt(2 MAF_j (1 - MAF_j)) + N(0,1); alpha 1; 100 log lambdas to 0.1."""
    import torch
    dev = _torch_dev(device)
    ld = padded_ld(n, np.int8)
    X = torch.zeros((p, ld), dtype=torch.int8, device=dev)
    mafs = torch.empty(p, dtype=torch.float64)
    for b in range((p + BLOCK - 1) // BLOCK):
        j0, j1 = b * BLOCK, min(p, (b + 1) * BLOCK)
        g = _gen(dev, seed, b)
        maf = 0.05 + 0.45 * torch.rand((j1 - j0, 1), generator=g, device=dev, dtype=torch.float64)
        u = torch.rand((2, j1 - j0, n), generator=g, device=dev, dtype=torch.float32)
        X[j0:j1, :n] = ((u[0] < maf).to(torch.int8) + (u[1] < maf).to(torch.int8))
        mafs[j0:j1] = maf[:, 0].cpu()
    rng = np.random.default_rng(seed + 1)
    idx = np.sort(rng.choice(p, size=100, replace=False))
    bv = rng.normal(0.0, 0.5, size=100)
    beta = np.zeros(p); beta[idx] = bv
    m = mafs.numpy()[idx]
    Xs = X[torch.as_tensor(idx, device=dev), :n].double().cpu().numpy().T
    y = ((Xs - 2 * m) / np.sqrt(2 * m * (1 - m))) @ bv + rng.standard_normal(n)
    return Instance("cfg4", X, n, y, alpha=1.0, ratio=0.1, tol=1e-7, beta_true=beta, seed=seed)


def cfg5(seed=0, n=10_000, p=2_000_000, device=None, col_range=None):
    """BASELINE cfg5: iid N(0,1) fp32 (80 GB at full size); 200 nonzeros
    0.3 N(0,1); y = X beta + N(0,1); alpha 0.5; 100 log lambdas to 0.05;
    10-fold CV.  col_range=(j0, j1) draws only a shard (whole blocks)."""
    import torch
    dev = _torch_dev(device)
    ld = padded_ld(n, np.float32)
    j0g, j1g = col_range or (0, p)
    X = torch.zeros((j1g - j0g, ld), dtype=torch.float32, device=dev)
    for b in range(j0g // BLOCK, (j1g + BLOCK - 1) // BLOCK):
        j0, j1 = max(j0g, b * BLOCK), min(j1g, (b + 1) * BLOCK)
        g = _gen(dev, seed, b)
        e = torch.randn((min(p, (b + 1) * BLOCK) - b * BLOCK, n), generator=g, device=dev)
        X[j0 - j0g:j1 - j0g, :n] = e[j0 - b * BLOCK:j1 - b * BLOCK]
    rng = np.random.default_rng(seed + 1)
    idx = np.sort(rng.choice(p, size=200, replace=False))
    bv = 0.3 * rng.standard_normal(200)
    beta = np.zeros(p); beta[idx] = bv
    # X beta: regenerate the needed columns' blocks (shard independent)
    xb = np.zeros(n)
    for j, v in zip(idx, bv):
        b = j // BLOCK
        e = torch.randn((min(p, (b + 1) * BLOCK) - b * BLOCK, n), generator=_gen(dev, seed, b), device=dev)
        xb += v * e[j - b * BLOCK].double().cpu().numpy()
    y = xb + rng.standard_normal(n)
    return Instance("cfg5", X, n, y, alpha=0.5, ratio=0.05, tol=1e-7, beta_true=beta, seed=seed)


# ------------------------------------------------ NEXT-3: logistic (binomial) inputs

def logistic_instance(n, p, dtype=np.float64, seed=0, kind="iid", n_true=None, scale=1.0, const_cols=0,
                      alpha=1.0):
    """Small seeded binary-response instance: X as random_instance; y_i ~ Bernoulli(sigmoid(eta_i))
    with eta = x beta - mean (raw columns), beta_true on n_true random
    columns ~ scale * U(-1, 1) (the P:383 simulation's coefficient law)."""
    rng = np.random.default_rng(seed)
    if kind == "geno":
        maf = rng.uniform(0.05, 0.5, size=p)
        X = (rng.random((n, p)) < maf).astype(np.int8) + (rng.random((n, p)) < maf).astype(np.int8)
    else:
        X = rng.standard_normal((n, p))
        if kind == "corr":
            X = 0.6 * rng.standard_normal((n, 1)) + 0.8 * X
        X = X.astype(dtype)
    if const_cols:
        cols = rng.choice(p, size=const_cols, replace=False)
        X[:, cols] = X[0:1, cols]
    Xf = X.astype(np.float64)
    k = n_true if n_true is not None else max(1, min(20, p // 4))
    beta = np.zeros(p)
    idx = rng.choice(p, size=k, replace=False)
    beta[idx] = scale * rng.uniform(-1.0, 1.0, size=k)
    eta = Xf @ beta                          # logit(prob) = x_i' beta (raw x), centred
    eta -= eta.mean()
    y = (rng.random(n) < 1.0 / (1.0 + np.exp(-eta))).astype(np.float64)
    return Instance(name=f"logit_{kind}_{n}x{p}", X=to_colmajor(X, X.dtype), n=n, y=y,
                    alpha=alpha, beta_true=beta, seed=seed)


def logit_sim(seed=0, n=1000, p=100_000, device=None):
    """Bench workload for the logistic path (NEXT-3), shaped like the P:383 simulation:
    x_ij iid N(0,1) stored fp32, 20 true features with coefficients U(-1, 1),
    y_i ~ Bin(1, sigmoid(x_i' beta)); 100 log-spaced lambdas to 0.1 lambda_max."""
    import torch
    dev = _torch_dev(device)
    ld = padded_ld(n, np.float32)
    X = torch.zeros((p, ld), dtype=torch.float32, device=dev)
    for b in range((p + BLOCK - 1) // BLOCK):
        j0, j1 = b * BLOCK, min(p, (b + 1) * BLOCK)
        X[j0:j1, :n] = torch.randn((j1 - j0, n), generator=_gen(dev, seed + 77, b), device=dev,
                                   dtype=torch.float32)
    rng = np.random.default_rng(seed + 5)
    idx = np.sort(rng.choice(p, size=20, replace=False))
    bv = rng.uniform(-1.0, 1.0, size=20)
    beta = np.zeros(p); beta[idx] = bv
    eta = (X[torch.as_tensor(idx, device=dev), :n].double().T @ torch.as_tensor(bv, device=dev)).cpu().numpy()
    y = (rng.random(n) < 1.0 / (1.0 + np.exp(-eta))).astype(np.float64)
    return Instance("logit", X, n, y, alpha=1.0, ratio=0.1, tol=1e-7, beta_true=beta, seed=seed)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}
