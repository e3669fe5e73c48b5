"""Where the end-to-end time of one path goes (host X pinned -> design -> lambda_max -> path -> free).
   python scripts/e2e_breakdown.py [cfg2|cfg3]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1701_05936_b200 import bl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
inst = synth.CONFIGS[cfg](device="cuda:0")
Xd = inst.X
Xh_t = torch.empty(Xd.shape, dtype=Xd.dtype, pin_memory=True)
Xh_t.copy_(Xd)
Xh = Xh_t.numpy()
d0 = bl.Design(Xd, inst.n)
lm = d0.lambda_max(inst.y, inst.alpha)
lams = synth.lambda_grid(lm, 100, inst.ratio)
for _ in range(2):
    d0.fit_path(inst.y, lams, alpha=inst.alpha, tol=1e-7)
torch.cuda.synchronize()
for rep in range(5):
    t = [time.perf_counter()]
    dh = bl.Design(Xh, inst.n); torch.cuda.synchronize(); t.append(time.perf_counter())
    lmh = dh.lambda_max(inst.y, inst.alpha); torch.cuda.synchronize(); t.append(time.perf_counter())
    lh = synth.lambda_grid(lmh, 100, inst.ratio)
    ph = dh.fit_path(inst.y, lh, alpha=inst.alpha, tol=1e-7); torch.cuda.synchronize(); t.append(time.perf_counter())
    ph2 = dh.fit_path(inst.y, lh, alpha=inst.alpha, tol=1e-7); torch.cuda.synchronize(); t.append(time.perf_counter())
    dh.free(); torch.cuda.synchronize(); t.append(time.perf_counter())
    dt = np.diff(t) * 1e3
    print(json.dumps({"design_ms": dt[0], "lambda_max_ms": dt[1], "first_path_ms": dt[2], "second_path_ms": dt[3],
                      "free_ms": dt[4]}), flush=True)
