"""One 10-fold CV of cfg5's generator at reduced p (for ncu captures of the fold-batched scan):
python scripts/one_cv.py [p]"""
import sys
sys.path.insert(0, ".")
import synth
from paper_1701_05936_b200 import bl

p = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
inst = synth.cfg5(device="cuda", p=p)
d = bl.Design(inst.X, inst.n)
lams = synth.lambda_grid(d.lambda_max(inst.y, inst.alpha), inst.nlam, inst.ratio)
cv = d.cv(inst.y, lams, K=10, alpha=inst.alpha, tol=inst.tol, seed=0)
print("cfg5 p", p, "lambda_min", cv.lambda_min_index)
