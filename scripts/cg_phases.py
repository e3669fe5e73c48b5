import sys, os
sys.path.insert(0, ".")
import synth
from paper_1701_05936_b200 import bl
bl.LIB_PATH = "paper_1701_05936_b200/libcgphases.so"   # build.build_variant("cgphases", ["-DBL_CG_PHASES=1"])
for cfg in ("cfg3",):
    inst = synth.CONFIGS[cfg](device="cuda")
    d = bl.Design(inst.X, inst.n)
    lams = synth.lambda_grid(d.lambda_max(inst.y, inst.alpha), inst.nlam, inst.ratio)
    gp = d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, profile=True)
    pf = gp.perf
    it = pf["cd_events"][5]
    print(cfg, "cg iters", it, "newton cycles/iter", pf["cd_events"][6] / max(it, 1))
    print("  per-iteration cycles (owner 1): r-publish barrier, load r, matvec, dots+cta sum, cluster reduce:",
          [round(x / max(it, 1)) for x in pf["cd_sub"][:5]])
