"""Small fits for compute-sanitizer (memcheck / synccheck / racecheck) over the Gram-CD
cluster protocol (mbarrier rings, bulk-copy hand-off, Newton CG barriers): cfg1-sized
paths at cluster sizes 4 / 8 / 16, lasso and elastic net, with and without Newton steps,
the residual CD, a lockstep CV and a logistic path.  Prints one line per fit."""
import sys
sys.path.insert(0, ".")
import numpy as np
import synth
from paper_1701_05936_b200 import bl

inst = synth.random_instance(200, 1000, dtype=np.float64, seed=0, kind="corr", n_true=10)
d = bl.Design(inst.host_X(), inst.n)
for alpha in (1.0, 0.5):
    lams = synth.lambda_grid(d.lambda_max(inst.y, alpha), 30, 0.05)
    for R in (4, 8, 16):
        for accel in ("newton", "none"):
            p = d.fit_path(inst.y, lams, alpha=alpha, tol=1e-9, cd_cluster=R, cd_accel=accel)
            print(f"gram alpha={alpha} R={R} {accel}: nnz(last)={int(p.col_ptr[-1] - p.col_ptr[-2])}", flush=True)
    p = d.fit_path(inst.y, lams, alpha=alpha, tol=1e-9, cd="residual")
    print(f"residual alpha={alpha}: nnz(last)={int(p.col_ptr[-1] - p.col_ptr[-2])}", flush=True)
c = d.cv(inst.y, synth.lambda_grid(d.lambda_max(inst.y, 0.5), 15, 0.1), K=4, alpha=0.5, tol=1e-9, seed=1)
print("cv lambda_min", c.lambda_min_index, flush=True)
li = synth.logistic_instance(160, 300, dtype=np.float32, seed=4, n_true=6, scale=1.5)
dl = bl.Design(li.host_X(), li.n)
pl = dl.fit_path_binomial(li.y, synth.lambda_grid(dl.lambda_max(li.y), 10, 0.2), tol=1e-10)
print("logistic nnz(last)", int(pl.col_ptr[-1] - pl.col_ptr[-2]), flush=True)
