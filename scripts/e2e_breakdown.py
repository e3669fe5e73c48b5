"""Where the end-to-end time of one cfg2 path goes (host X pinned -> design -> lambda_max -> path -> free)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1701_05936_b200 import bl  # noqa: E402

inst = synth.cfg2(device="cuda:0")
Xd = inst.X
Xh_t = torch.empty(Xd.shape, dtype=Xd.dtype, pin_memory=True)
Xh_t.copy_(Xd)
Xh = Xh_t.numpy()
d0 = bl.Design(Xd, inst.n)
lm = d0.lambda_max(inst.y, 1.0)
lams = synth.lambda_grid(lm, 100, 0.1)
for _ in range(2):
    d0.fit_path(inst.y, lams, tol=1e-7)
torch.cuda.synchronize()
for rep in range(3):
    t = [time.perf_counter()]
    dh = bl.Design(Xh, inst.n); torch.cuda.synchronize(); t.append(time.perf_counter())
    lmh = dh.lambda_max(inst.y, 1.0); torch.cuda.synchronize(); t.append(time.perf_counter())
    ph = dh.fit_path(inst.y, synth.lambda_grid(lmh, 100, 0.1), tol=1e-7); torch.cuda.synchronize(); t.append(time.perf_counter())
    ph2 = dh.fit_path(inst.y, synth.lambda_grid(lmh, 100, 0.1), tol=1e-7); torch.cuda.synchronize(); t.append(time.perf_counter())
    dh.free(); torch.cuda.synchronize(); t.append(time.perf_counter())
    dt = np.diff(t) * 1e3
    print(json.dumps({"design_ms": dt[0], "lambda_max_ms": dt[1], "first_path_ms": dt[2], "second_path_ms": dt[3],
                      "free_ms": dt[4]}), flush=True)
