"""Per-lambda CD structure of the bench configs (passes, |W|, nnz) -- diagnostics for the CD work."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
from paper_1701_05936_b200 import bl

out = {}
for cfg in sys.argv[1:]:
    inst = synth.CONFIGS[cfg](device="cuda")
    d = bl.Design(inst.X, inst.n)
    lm = d.lambda_max(inst.y, inst.alpha)
    lams = synth.lambda_grid(lm, inst.nlam, inst.ratio)
    d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol)
    t0 = time.perf_counter()
    gp = d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, profile=True)
    t1 = time.perf_counter()
    nnz = np.diff(gp.col_ptr)
    out[cfg] = dict(wall=t1 - t0, perf=gp.perf, passes=gp.passes.tolist(), nnz=nnz.tolist(),
                    W=gp.n_working.tolist(), kkt=gp.kkt_rounds.tolist())
    print(cfg, t1 - t0, gp.perf["cd_ms"], gp.perf["scan_ms"], int(gp.passes.sum()), flush=True)
json.dump(out, open("gpurun_out/cd_structure.json", "w"))
