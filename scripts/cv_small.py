"""cfg5-shaped CV at reduced p (profiling target for the batched scan)."""
import sys, time, json
sys.path.insert(0, ".")
import torch
import synth
from paper_1701_05936_b200 import bl
p = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
inst = synth.cfg5(device="cuda", p=p)
d = bl.Design(inst.X, inst.n)
lm = d.lambda_max(inst.y, inst.alpha)
lams = synth.lambda_grid(lm, 100, inst.ratio)
t0 = time.perf_counter()
cv = d.cv(inst.y, lams, K=10, alpha=inst.alpha, tol=inst.tol, seed=0, profile=True)
torch.cuda.synchronize()
pf = cv.perf
print(json.dumps({"p": p, "cv_s": time.perf_counter() - t0, "scan_ms": pf["scan_ms"], "scan_launches": pf["scan_launches"],
                  "scan_GBps": pf["scan_bytes"] / max(pf["scan_ms"], 1e-9) / 1e6, "cd_ms": pf["cd_ms"]}))
