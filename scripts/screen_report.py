"""Screening report (SURVEY 8(d) secondary reports).

1. Fig 1 analog: per lambda, the fraction of live columns the BEDPP
   safe rule keeps (|S_k| / p), the strong set entering lambda_k and |W|, for the
   BASELINE cfg2/cfg3/cfg4 paths (hybrid SSR-BEDPP).
2. Table 6 shape: hybrid vs SSR-only on cfg4 with lambda_min/lambda_max
   in {0.1, 0.5}: path time (CUDA events), columns scanned, scan GB/s.

Writes one JSON object per line to stdout.  Usage: python scripts/screen_report.py [cfg ...]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1701_05936_b200 import bl  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts, out = [], None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), out


def main(cfgs):
    for name in cfgs:
        inst = synth.CONFIGS[name](device="cuda:0")
        X = inst.X if not isinstance(inst.X, np.ndarray) else torch.from_numpy(inst.X).cuda()
        d = bl.Design(X, inst.n)
        lm = d.lambda_max(inst.y, inst.alpha)
        ratios = [inst.ratio] + ([0.5] if name == "cfg4" else [])
        for ratio in ratios:
            lams = synth.lambda_grid(lm, inst.nlam, ratio)
            for screen in (["hybrid", "ssr"] if name == "cfg4" else ["hybrid"]):
                ms, path = timed(lambda: d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, screen=screen,
                                                    profile=True))
                pf = path.perf
                rec = {"config": name, "screen": screen, "lambda_min_ratio": ratio, "path_ms": ms,
                       "cols_scanned": int(path.cols_scanned.sum()),
                       "full_scan_equivalents": float(path.cols_scanned.sum() / inst.p),
                       "scan_ms": pf["scan_ms"],
                       "scan_GBps": pf["scan_bytes"] / (pf["scan_ms"] / 1e3) / 1e9 if pf["scan_ms"] else None,
                       "kkt_rounds": int(path.kkt_rounds.sum()), "nnz_last": int(path.col_ptr[-1] - path.col_ptr[-2])}
                if screen == "hybrid" and ratio == inst.ratio:
                    rec["per_lambda"] = {"lambda_over_max": [round(float(v), 5) for v in lams / lm],
                                         "bedpp_kept_frac": [round(float(v) / inst.p, 6) for v in path.n_safe],
                                         "strong": path.n_strong.tolist(), "working": path.n_working.tolist(),
                                         "cols_scanned": path.cols_scanned.tolist()}
                print(json.dumps(rec), flush=True)
        d.free()
        del X, inst
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg3", "cfg4"])
