"""Path time vs Gram-CD cluster size (bl_opts.cd_cluster): python scripts/cluster_sweep.py logit cfg2"""
import json
import sys

sys.path.insert(0, ".")
import torch
import synth
from paper_1701_05936_b200 import bl

for cfg in sys.argv[1:] or ["logit"]:
    inst = synth.logit_sim(device="cuda") if cfg == "logit" else synth.CONFIGS[cfg](device="cuda")
    d = bl.Design(inst.X, inst.n)
    lams = synth.lambda_grid(d.lambda_max(inst.y, inst.alpha), inst.nlam, inst.ratio)
    sh = torch.cuda.current_stream().cuda_stream
    row = {"config": cfg}
    for cc in (16, 8, 4, 16):
        fit = (lambda: d.fit_path_binomial(inst.y, lams, alpha=inst.alpha, tol=inst.tol, stream=sh, cd_cluster=cc)) \
            if cfg == "logit" else \
            (lambda: d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, stream=sh, cd_cluster=cc))
        fit()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(3):
            e0.record()
            fit()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        row[str(cc)] = sorted(ms)[1]
    print(json.dumps(row), flush=True)
    d.free()
