"""Time ONE full-data cfg5 path (fit_path, no CV) to separate per-fit cost from CV contention."""
import json, sys, time
sys.path.insert(0, ".")
import torch
import synth
from paper_1701_05936_b200 import bl
inst = synth.cfg5(device="cuda")
d = bl.Design(inst.X, inst.n)
lm = d.lambda_max(inst.y, inst.alpha)
lams = synth.lambda_grid(lm, 100, inst.ratio)
d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol)
torch.cuda.synchronize()
t0 = time.perf_counter()
p = d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, profile=True)
torch.cuda.synchronize()
t = time.perf_counter() - t0
pf = p.perf
print(json.dumps({"path_s": t, "scan_ms": pf["scan_ms"], "scan_GBps": pf["scan_bytes"] / pf["scan_ms"] / 1e6,
                  "cd_ms": pf["cd_ms"], "cd_visits": pf["cd_visits"], "cd_kernel_ms": pf["cd_kernel_cycles"] / 1.965e6,
                  "prof": pf["cd_prof"], "launches": pf["kernel_launches"], "nnz_last": int(p.col_ptr[-1] - p.col_ptr[-2]),
                  "passes": int(p.passes.sum()), "cols_scanned": int(p.cols_scanned.sum())}))
t0 = time.perf_counter()
cv = d.cv(inst.y, lams, K=10, alpha=inst.alpha, tol=inst.tol, seed=0, profile=True)
torch.cuda.synchronize()
print(json.dumps({"cv_s": time.perf_counter() - t0, "sum_scan_ms": cv.perf["scan_ms"], "sum_cd_ms": cv.perf["cd_ms"],
                  "sum_visits": cv.perf["cd_visits"], "sum_cd_kernel_ms": cv.perf["cd_kernel_cycles"] / 1.965e6}))
