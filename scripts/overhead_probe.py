"""Per-lambda overhead of a path outside the scan and CD launches: the same fit timed with and
without the library's per-launch CUDA events (profile), and the remainder path - scan - CD.
    python scripts/overhead_probe.py cfg3 cfg2
"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch
import synth
from paper_1701_05936_b200 import bl

for cfg in sys.argv[1:] or ["cfg3"]:
    inst = synth.CONFIGS[cfg](device="cuda")
    d = bl.Design(inst.X, inst.n)
    lams = synth.lambda_grid(d.lambda_max(inst.y, inst.alpha), inst.nlam, inst.ratio)
    sh = torch.cuda.current_stream().cuda_stream
    row = {"config": cfg}
    for prof in (False, True, False, True):
        for _ in range(2):
            d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, stream=sh, profile=prof)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps, ms, perf = 5, [], None
        for _ in range(reps):
            e0.record()
            t0 = time.perf_counter()
            gp = d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, stream=sh, profile=prof)
            e1.record()
            torch.cuda.synchronize()
            ms.append((e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)))
            perf = gp.perf
        ms.sort()
        key = "profile" if prof else "plain"
        row[key] = {"path_ms": ms[len(ms) // 2][0], "host_ms": ms[len(ms) // 2][1]}
        if prof:
            row[key].update(scan_ms=perf["scan_ms"], cd_ms=perf["cd_ms"],
                            rest_ms=ms[len(ms) // 2][0] - perf["scan_ms"] - perf["cd_ms"],
                            scan_launches=perf["scan_launches"], cd_launches=perf["cd_launches"],
                            launches=perf["kernel_launches"])
    print(json.dumps(row))
    d.free()
