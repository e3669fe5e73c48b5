"""cfg5 full-size duality-gap certificate of the full-data path vs the CD tolerance and the
Newton (CG) acceleration (tests/test_gpu_parity.py::cfg5_certify).  GPU only.
    python scripts/cert_probe.py [tol ...]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1701_05936_b200 import bl  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from test_gpu_parity import cfg5_certify  # noqa: E402


def main():
    tols = [float(t) for t in sys.argv[1:]] or [1e-10, 1e-11, 1e-12]
    inst = synth.cfg5(device="cuda")
    X, n, a = inst.X, inst.n, inst.alpha
    d = bl.Design(X, n)
    lams = synth.lambda_grid(d.lambda_max(inst.y, a), 100, inst.ratio)
    y = torch.as_tensor(inst.y, device="cuda", dtype=torch.float64)
    yt = y - y.mean()
    p = X.shape[0]
    c = torch.empty(p, dtype=torch.float64, device="cuda")
    s = torch.empty_like(c)
    CH = 50_000
    for j0 in range(0, p, CH):
        B = X[j0:j0 + CH, :n].double()
        c[j0:j0 + CH] = B.mean(1)
        s[j0:j0 + CH] = (B - c[j0:j0 + CH, None]).pow(2).mean(1).sqrt()
    for accel in ("newton", "none"):
        for tol in tols:
            path = d.fit_path(inst.y, lams, alpha=a, tol=tol, cd_accel=accel, profile=True)
            out = []
            for k in (40, 70, 99):
                bound, bmax = cfg5_certify(X, n, a, lams, c, s, yt, path, k, CH)
                out.append(f"k={k} {bound / bmax:.2e}")
            print(f"accel={accel:6s} tol={tol:.0e} conv={path.n_converged} passes={int(path.passes.sum())}"
                  f" cd_ms={path.perf["cd_ms"]:.1f}  bound/max|beta|: " + "  ".join(out), flush=True)


if __name__ == "__main__":
    main()
