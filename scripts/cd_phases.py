"""Gram CD leader-warp sub-phase breakdown (bl_perf.cd_sub / cd_events) per config."""
import sys
import numpy as np
sys.path.insert(0, ".")
import synth
from paper_1701_05936_b200 import bl
import os
if os.environ.get("CD_PHASES_LIB"):        # the -DBL_G7_SUBPHASES=1 build (build.build_variant)
    bl.LIB_PATH = os.environ["CD_PHASES_LIB"]

accel = os.environ.get("CD_ACCEL", "newton")
R = int(os.environ.get("CD_CLUSTER", "0"))
ref = {}
for cfg in sys.argv[1:]:
    inst = synth.CONFIGS[cfg](device="cuda")
    d = bl.Design(inst.X, inst.n)
    lams = synth.lambda_grid(d.lambda_max(inst.y, inst.alpha), inst.nlam, inst.ratio)
    d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, cd_accel=accel, cd_cluster=R)
    gp = d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, profile=True, cd_accel=accel, cd_cluster=R)
    if accel != "none":                    # against the sweeps-only solution of the same path
        g0 = d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, cd_accel="none")
        B, B0 = gp.dense(inst.p), g0.dense(inst.p)
        sc = np.abs(B0).max(0)
        rel = np.abs(B - B0).max(0) / np.where(sc > 0, sc, 1)
        print(cfg, "max rel diff vs sweeps-only per lambda:", float(rel.max()), "passes", int(gp.passes.sum()), "vs", int(g0.passes.sum()))
    pf = gp.perf
    v = pf["cd_visits"]
    blocks = v / 32
    names = ["prologue", "active_matvec", "fwd_subst", "publish", "wait_stage+snap", "wait_next_stage", "link", "w_checks(count)"]
    print(cfg, "cluster", R or 8, "cd_ms", round(pf["cd_ms"], 2), "path_ms", round(pf["wall_ms"], 2), "visits", v, "cycles/visit", round(pf["cd_kernel_cycles"] / v, 1))
    print("  events (retries, builds, catchups, full sweeps, newton, cg iters, newton cycles, partial):", pf["cd_events"])
    print("  phases per visit (lead, bulk, build, catch):", [round(x / v, 1) for x in pf["cd_prof"]])
    print("  leader sub-phases per BLOCK:", {n: round(x / blocks, 1) for n, x in zip(names[:7], pf["cd_sub"][:7])},
          "W checks:", pf["cd_sub"][7])
