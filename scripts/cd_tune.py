"""Gram CD tunables sweep: builds library variants (build.build_variant) and times cfg3 / cfg2 paths.
   build:  python scripts/cd_tune.py build      (CPU; parallel nvcc)
   run:    python scripts/cd_tune.py run cfg3 cfg2   (GPU)"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
VARIANTS = {
    "base": [],
    "rho01": ["-DBL_NEWTON_RHO=0.1"],
    "rho06": ["-DBL_NEWTON_RHO=0.6"],
    "nmax4": ["-DBL_NEWTON_MAX=4"],
    "rtol005": ["-DBL_CG_RTOL=0.05"],
    "rtol05": ["-DBL_CG_RTOL=0.5"],
    "sw2": ["-DBL_NEWTON_SWEEPS=2"],
}


def build():
    from concurrent.futures import ThreadPoolExecutor
    from paper_1701_05936_b200 import build as b
    with ThreadPoolExecutor(len(VARIANTS)) as ex:
        for name, out in zip(VARIANTS, ex.map(lambda kv: b.build_variant("tune_" + kv[0], kv[1]), VARIANTS.items())):
            print(name, out)


def run(cfgs):
    for name in VARIANTS:
        lib = f"paper_1701_05936_b200/libtune_{name}.so"
        out = subprocess.run([sys.executable, __file__, "one", lib, *cfgs], capture_output=True, text=True)
        print(name, out.stdout.strip(), out.stderr.strip()[-300:], flush=True)


def one(lib, cfgs):
    import numpy as np
    import synth
    from paper_1701_05936_b200 import bl
    bl.LIB_PATH = lib
    res = []
    for cfg in cfgs:
        inst = synth.CONFIGS[cfg](device="cuda")
        d = bl.Design(inst.X, inst.n)
        lams = synth.lambda_grid(d.lambda_max(inst.y, inst.alpha), inst.nlam, inst.ratio)
        d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol)
        best = None
        for _ in range(3):
            gp = d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, profile=True)
            pf = gp.perf
            t = (pf["wall_ms"], pf["cd_ms"])
            best = t if best is None or t[0] < best[0] else best
        g0 = d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, cd_accel="none")
        B, B0 = gp.dense(inst.p), g0.dense(inst.p)
        sc = np.abs(B0).max(0)
        rel = float((np.abs(B - B0).max(0) / np.where(sc > 0, sc, 1)).max())
        res.append(f"{cfg}: path {best[0]:.1f} ms cd {best[1]:.1f} ms passes {int(gp.passes.sum())} "
                   f"newton {pf['cd_events'][4]} cg {pf['cd_events'][5]} rel-vs-sweeps {rel:.1e}")
        del d
    print(" | ".join(res))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    elif sys.argv[1] == "run":
        run(sys.argv[2:])
    else:
        one(sys.argv[2], sys.argv[3:])
