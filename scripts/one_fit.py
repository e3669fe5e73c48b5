"""One path fit of a bench config (for ncu captures): python scripts/one_fit.py cfg3 [reps]."""
import sys
sys.path.insert(0, ".")
import synth
from paper_1701_05936_b200 import bl

cfg = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
inst = synth.CONFIGS[cfg](device="cuda")
d = bl.Design(inst.X, inst.n)
lams = synth.lambda_grid(d.lambda_max(inst.y, inst.alpha), inst.nlam, inst.ratio)
for _ in range(reps):
    gp = d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol)
print(cfg, "nnz(last)", int(gp.col_ptr[-1] - gp.col_ptr[-2]))
