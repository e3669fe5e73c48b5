"""Fold-batched CV scan throughput on cfg5's generator at reduced p:
python scripts/cv_scan_time.py [p] -- prints the batched scans' time, X GB/s and fp64 TFLOP/s."""
import os
import sys
sys.path.insert(0, ".")
import synth
from paper_1701_05936_b200 import bl

if os.environ.get("CV_LIB"):
    bl.LIB_PATH = os.environ["CV_LIB"]
p = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
inst = synth.cfg5(device="cuda", p=p)
d = bl.Design(inst.X, inst.n)
lams = synth.lambda_grid(d.lambda_max(inst.y, inst.alpha), 40, inst.ratio)
d.cv(inst.y, lams, K=K, alpha=inst.alpha, tol=inst.tol, seed=0)
cv = d.cv(inst.y, lams, K=K, alpha=inst.alpha, tol=inst.tol, seed=0, profile=True)
pf = cv.perf
gbs = pf["scan_bytes"] / (pf["scan_ms"] / 1e3) / 1e9
tfl = 2 * (K + 1) * pf["scan_bytes"] / 4 / (pf["scan_ms"] / 1e3) / 1e12
print(f"p={p} K={K} scan_ms={pf['scan_ms']:.1f} launches={pf['scan_launches']} X={gbs:.0f} GB/s fp64={tfl:.2f} TFLOP/s "
      f"({tfl / 36.3:.3f} of 36.3) wall={pf['wall_ms']:.1f} ms")
