"""A small logistic path (p = 20,000, n = 1000, fp32) for profiling k_cd_logit under ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1701_05936_b200 import bl  # noqa: E402

inst = synth.logit_sim(p=20_000, device="cuda:0")
d = bl.Design(inst.X, inst.n)
lm = d.lambda_max(inst.y)
lams = synth.lambda_grid(lm, 100, 0.1)
path = d.fit_path_binomial(inst.y, lams, tol=1e-7, profile=True)
torch.cuda.synchronize()
print("cd_ms", path.perf["cd_ms"], "visits", path.perf["cd_visits"], "nnz", int(path.col_ptr[-1] - path.col_ptr[-2]))
