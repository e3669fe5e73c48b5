#!/usr/bin/env python
"""Benchmark: 100-lambda lasso / elastic-net path wall time and fused-scan HBM
throughput (BASELINE.json metric) on a B200.

    python bench.py [--gpus N --steps K --warmup W] [--config cfg2] [--impl ours|reference]

A step = one full 100-lambda path (all SURVEY 8(a) rows: preprocessing, BEDPP,
strong rule, CD, fused KKT/strong scans) over the config's synthetic design,
through the C ABI (libbl.so).  Default workload = BASELINE cfg3, the largest
single-GPU configuration: n = 1000, p = 1,000,000, fp32 block-factor design,
elastic net alpha = 0.5, lambda to 0.1 lambda_max.  X (4.0 GB) is far larger than
L2 (126 MB), so no flush is needed between steps.

N > 1 (torchrun): the design is column-sharded over the ranks (whole
1000-column blocks, BASELINE north star): scans, BEDPP and the strong rule run
per shard, the small index lists are all-gathered and the working-set columns
broadcast by their owners over NCCL, the CD runs replicated (DESIGN.md section
7).  The same path is solved at every N (strong scaling); the time is the max
over ranks.

`--impl reference` times the fp64 CPU oracle (oracle/, naive CD, no screening)
on this box's host cores on the same full-size workload: the K steps run the
100-lambda grid in K chunks, so their summed time is the measured path time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "100-λ lasso path wall-time (s) and feature-scan HBM GB/s vs B200 peak, 1/2/4/8 GPU"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_instance(name, device=None):
    import synth
    if name == "logit":
        return synth.logit_sim(device=device)
    return synth.CONFIGS[name](device=device) if name != "cfg1" else synth.cfg1()


# ---------------------------------------------------------------- oracle legs

def host_cpu():
    """(threads the oracle may use, CPU model) of this host."""
    try:
        T = len(os.sched_getaffinity(0))
    except Exception:
        T = os.cpu_count() or 1
    model = "unknown"
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return T, model


def oracle_prefix(inst, lams, budget_s, threads, binomial=False):
    """cpu_baseline leg: the oracle as it stands (naive cyclic CD, no screening, fp64) on the
    FULL design of the workload, T host threads (block-speculative passes: bitwise the serial
    oracle), over the first m lambdas of the SAME grid: column statistics and lambda_max, then
    one lambda at a time with warm starts until the time budget is spent.  Nothing is scaled.
    Returns (seconds, m)."""
    import oracle
    oracle.set_threads(threads)
    try:
        Xh = inst.host_X()
        if binomial:                                   # the logistic oracle has no session API: whole prefixes
            m, t = 1, 0.0
            while True:
                t0 = time.perf_counter()
                oracle.fit_path_binomial((Xh, inst.n), inst.y, lams[:m], alpha=inst.alpha, tol=inst.tol,
                                         raise_on_error=False)
                t = time.perf_counter() - t0
                if t >= budget_s / 3 or m >= len(lams):
                    return t, m
                m = min(len(lams), 2 * m)
        t0 = time.perf_counter()
        sess = oracle.PathSession((Xh, inst.n), inst.y, inst.alpha)
        m = 0
        while m < len(lams) and time.perf_counter() - t0 < budget_s:
            sess.run(lams[m:m + 1], tol=inst.tol, cycle_active=True)
            m += 1
        dt = time.perf_counter() - t0
        sess.close()
        return dt, m
    finally:
        oracle.set_threads(1)


def run_reference(args, rank, world):
    """--impl reference: the oracle (as it stands) on this box's host cores, on the same
    workload bytes, lambda grid rule, alpha and tol as our arm.  The K timed steps run the
    WHOLE 100-lambda path in K consecutive chunks of the grid (warm starts carry across
    chunks; step 0 also computes the column statistics and lambda_max), so the summed step
    time is the measured path wall time -- nothing is extrapolated.  W warm-up steps are
    untimed passes over X (page-in).  N > 1: rank 0 alone runs it."""
    if rank != 0:
        return
    import oracle
    import synth
    inst = make_instance(args.config)
    T, model = host_cpu()
    Xh = inst.host_X()
    oracle.set_threads(T)
    try:
        for _ in range(args.warmup):
            oracle.column_stats((Xh, inst.n))
        nl = inst.nlam
        K = max(1, min(args.steps, nl))
        chunk = -(-nl // K)
        times, sess, lams = [], None, None
        for s in range(K):
            t0 = time.perf_counter()
            if sess is None:
                sess = oracle.PathSession((Xh, inst.n), inst.y, inst.alpha)
                lams = synth.lambda_grid(sess.lambda_max, nl, inst.ratio)
            part = lams[s * chunk:(s + 1) * chunk]
            if len(part):
                sess.run(part, tol=inst.tol, cycle_active=True)
            times.append(time.perf_counter() - t0)
        sess.close()
    finally:
        oracle.set_threads(1)
    total = sum(times)
    sample = (f"oracle (naive cyclic CD with active cycling, fp64, tol {inst.tol:g}, no screening) on the full "
              f"{args.config} design (n={inst.n}, p={inst.p}), the whole {nl}-lambda grid run in {K} chunks of "
              f"{chunk} lambdas (warm starts across chunks), {T} threads (block-speculative passes, bitwise the "
              f"serial oracle); value = summed step time = the path wall time")
    line = {"impl": "reference", "metric": METRIC, "value": total, "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / max(1, len(times)),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n": inst.n, "p": inst.p, "alpha": inst.alpha,
                       "n_lambda": nl, "lambda_min_ratio": inst.ratio, "tol": inst.tol},
            "cpu_baseline": {"value": total, "unit": "s", "cores": T, "cpu_model": model, "kind": "oracle",
                             "sample": sample, "step_seconds": times},
            "e2e": {"value": total, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1701_05936_b200 import bl
    import synth
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if world > 1 and args.config == "cfg5":
        j0, j1 = bl.shard_range(synth.cfg5.__defaults__[2], world, rank, block=synth.BLOCK)
        inst = synth.cfg5(device=f"cuda:{local_rank}", col_range=(j0, j1))
        p_global = synth.cfg5.__defaults__[2]
    else:
        inst = make_instance(args.config, device=f"cuda:{local_rank}")
        p_global = inst.p
        j0, j1 = bl.shard_range(p_global, world, rank, block=synth.BLOCK)
    X = inst.X if not isinstance(inst.X, np.ndarray) else torch.from_numpy(inst.X).cuda()
    if world > 1 and X.shape[0] != j1 - j0:             # this rank's shard only
        X = X[j0:j1].contiguous()
        inst.X = X
        torch.cuda.empty_cache()
    dist_of = (lambda: bl.make_dist(rank, world, (j0, j1), p_global, device=local_rank)) if world > 1 else (lambda: None)
    host_res = args.resident == "host"    # NEXT-4: X stays in pinned host memory, streamed over PCIe
    link_gbs = None
    if host_res:
        Xpin = torch.empty(X.shape, dtype=X.dtype, pin_memory=True)
        Xpin.copy_(X)
        # the host link's measured copy bandwidth (pinned -> device), the roof of a streamed scan
        probe = torch.empty(min(X.numel(), (1 << 31) // X.element_size()), dtype=X.dtype, device=X.device)
        src = Xpin.view(-1)[:probe.numel()]
        probe.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0_.record()
        for _ in range(3):
            probe.copy_(src, non_blocking=True)
        e1_.record()
        torch.cuda.synchronize()
        link_gbs = 3 * probe.numel() * probe.element_size() / (e0_.elapsed_time(e1_) / 1e3) / 1e9
        del probe, X
        inst.X = Xpin
        torch.cuda.empty_cache()
        X = Xpin
        d = bl.Design(Xpin.numpy(), inst.n, dist=dist_of(), host_resident=True)
    else:
        d = bl.Design(X, inst.n, dist=dist_of())
    lm = d.lambda_max(inst.y, inst.alpha)
    lams = synth.lambda_grid(lm, inst.nlam, inst.ratio)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    is_cv = args.config == "cfg5"        # BASELINE cfg5: 10-fold CV -- a step is the whole CV
    is_logit = args.config == "logit"    # NEXT-3: penalised logistic path (P:379-385 simulation shape)

    def step(profile):
        if is_logit:
            return d.fit_path_binomial(inst.y, lams, alpha=inst.alpha, tol=inst.tol, stream=sh, profile=profile)
        if is_cv:
            return d.cv(inst.y, lams, K=10, alpha=inst.alpha, tol=inst.tol, seed=0, profile=profile, cd=args.cd,
                        cv_mode=args.cv_mode)
        return d.fit_path(inst.y, lams, alpha=inst.alpha, tol=inst.tol, stream=sh, profile=profile, cd=args.cd)

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    perfs = []
    with Clocks(local_rank) as clk:
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            perfs.append(step(True))
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    last = perfs[-1].full if is_cv else perfs[-1]
    scan_ms = sum(p.perf["scan_ms"] for p in perfs)
    scan_bytes = sum(p.perf["scan_bytes"] for p in perfs)
    scan_launches = sum(p.perf["scan_launches"] for p in perfs)
    cd_ms = sum(p.perf["cd_ms"] for p in perfs)
    launches = sum(p.perf["kernel_launches"] for p in perfs)
    visits = sum(p.perf["cd_visits"] for p in perfs) / args.steps
    updates = sum(p.perf["cd_updates"] for p in perfs) / args.steps
    cd_cycles = sum(p.perf["cd_kernel_cycles"] for p in perfs) / args.steps
    cd_prof = [sum(p.perf["cd_prof"][u] for p in perfs) / args.steps / max(visits, 1) for u in range(4)]
    # GB/s over the scan launches that covered every live column (|S_k| = p)
    fs_ms = sum(p.perf["full_scan_ms"] for p in perfs)
    fs_bytes = sum(p.perf["full_scan_bytes"] for p in perfs)
    fs_launches = sum(p.perf["full_scan_launches"] for p in perfs) / args.steps

    # end to end through the C ABI with HOST buffers (H2D of X inside the timed region)
    x_bytes = X.numel() * X.element_size()
    e2e, e2e_load, h2d, d2h = [], [], 0, 0
    if x_bytes <= 40e9:
        Xh_t = X if host_res else torch.empty(X.shape, dtype=X.dtype, pin_memory=True)
        if not host_res:
            Xh_t.copy_(X)
        Xh = Xh_t.numpy()
        for it in range(1 + max(1, min(args.steps, 5))):        # one untimed warm-up, then up to 5 samples
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dh = bl.Design(Xh, inst.n, dist=dist_of(), host_resident=host_res)
            torch.cuda.synchronize()
            t_load = time.perf_counter() - t0
            lm_h = dh.lambda_max(inst.y, inst.alpha)
            lams_h = synth.lambda_grid(lm_h, inst.nlam, inst.ratio)
            if is_logit:
                ph = dh.fit_path_binomial(inst.y, lams_h, alpha=inst.alpha, tol=inst.tol)
            elif is_cv:
                ph = dh.cv(inst.y, lams_h, K=10, alpha=inst.alpha, tol=inst.tol, seed=0).full
            else:
                ph = dh.fit_path(inst.y, lams_h, alpha=inst.alpha, tol=inst.tol)
            dh.free()
            torch.cuda.synchronize()
            if it == 0:
                continue
            e2e.append(time.perf_counter() - t0)
            e2e_load.append(t_load)
        h2d = Xh.nbytes + 8 * inst.n * 2 + 8 * inst.nlam
        d2h = int(ph.beta_std.nbytes * 2 + ph.feat.nbytes + 8 * inst.nlam * 3)

    if rank != 0:
        return
    pk, pk_src = peaks()
    achieved = scan_bytes / (scan_ms / 1e3) / 1e9 if scan_ms > 0 else None
    roof = None
    if host_res:
        roof = {"kernel": "k_scan_fp/k_scan_i8 over host-resident X (zero-copy over PCIe, NEXT-4)", "bound": "host link",
                "achieved": achieved, "peak": link_gbs,
                "peak_source": "measured pinned host -> device copy bandwidth in this run", "unit": "GB/s",
                "frac": achieved / link_gbs if achieved and link_gbs else None, "traffic": None}
    if is_cv:
        fits = 11
        flops = 2.0 * fits * scan_bytes / X.element_size()
        tfl = flops / (scan_ms / 1e3) / 1e12 if scan_ms > 0 else None
        if args.cv_mode == "batched" and X.dtype == torch.float32:
            # the fold-batched scan on the tcgen05 integer tensor cores (exact digit products): one pass
            # over X serves all 11 fits and the int8 MMAs have >100x the needed rate -- bound by reading X
            roof = {"kernel": "k_scan_batch_tc (fold-batched fused scan, tcgen05 kind::i8 on SM pairs, 11 residuals per pass over X)",
                    "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "peak_source": pk_src, "unit": "GB/s",
                    "frac": achieved / pk["hbm_gbs"] if achieved else None, "traffic": None,
                    "useful_fp64_equiv_TFLOPs": tfl}
        else:
            # the fp64 tensor-core / FMA kernels: 11 FMAs per element, at the fp64 ridge
            fpk = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["fp64_tflops"]
            roof = {"kernel": "k_scan_batch_mma (fold-batched fused scan on the fp64 tensor cores, 11 residuals per pass over X)", "bound": "alu",
                    "achieved": tfl, "peak": fpk, "peak_source": "measured fp64 FMA throughput (scripts/fp64_peak.cu, profiles/fp64_peak.json)",
                    "unit": "TFLOP/s", "frac": tfl / fpk if tfl else None, "traffic": None,
                    "x_read_GBps": achieved, "x_read_frac_of_hbm": achieved / pk["hbm_gbs"] if achieved else None}
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("traffic_per_launch")
        except Exception:
            traffic = None
    cpu = {"value": None, "unit": "s", "cores": 1, "kind": "oracle", "sample": "skipped (--no-cpu-baseline)"}
    if world == 1 and not args.no_cpu_baseline and not is_cv:
        T, model = host_cpu()
        v, m = oracle_prefix(inst, lams, args.ref_seconds, T, binomial=is_logit)
        # our path on exactly that sample (the same first m lambdas), for a like-for-like ratio
        gpu_m = []
        for _ in range(3):
            e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0_.record(stream)
            if is_logit:
                d.fit_path_binomial(inst.y, lams[:m], alpha=inst.alpha, tol=inst.tol, stream=sh)
            else:
                d.fit_path(inst.y, lams[:m], alpha=inst.alpha, tol=inst.tol, stream=sh, cd=args.cd)
            e1_.record(stream)
            torch.cuda.synchronize()
            gpu_m.append(e0_.elapsed_time(e1_) / 1e3)
        what = "IRLS + naive cyclic weighted CD" if is_logit else "naive cyclic CD with active cycling"
        cpu = {"value": v, "unit": "s", "cores": T, "cpu_model": model, "kind": "oracle", "lambdas": m,
               "sample": (f"oracle ({what}, fp64, tol {inst.tol:g}, no screening) on the full {args.config} design "
                          f"(n={inst.n}, p={p_global}), column statistics + lambda_max + the first {m} of the "
                          f"{inst.nlam} lambdas of the same grid, {T} threads (block-speculative passes, bitwise "
                          f"the serial oracle); measured, not scaled"),
               "gpu_same_sample_s": statistics.median(gpu_m)}
    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": ("f32-in/i8-digit-exact-scan/f64-accum" if is_cv and args.cv_mode == "batched"
                  else {"cfg1": "f64", "cfg4": "i8"}.get(args.config, "f32") + "-in/f64-accum"),
        "data": "synthetic",
        "config": {"workload": args.config, "n": inst.n, "p": p_global, "alpha": inst.alpha,
                   "n_lambda": inst.nlam, "lambda_min_ratio": inst.ratio, "tol": inst.tol,
                   "screen": "SSR (logistic, QL3)" if is_logit else "hybrid (SSR-BEDPP)",
                   "model": "logistic" if is_logit else "gaussian", "cd": args.cd, "X_bytes": int(x_bytes),
                   "cv_folds": 10 if is_cv else None, "cv_mode": args.cv_mode if is_cv else None,
                   "l2_policy": "X larger than L2 (126 MB); no flush" if X.numel() * X.element_size() > 126e6
                   else "X fits L2 (reported as such)", "resident": args.resident, "parallelism": f"column-sharded x{world}" if world > 1 else "1 GPU",
                   "p_global": p_global},
        "roofline": {**(roof or {"kernel": "k_scan_fp/k_scan_i8 (fused KKT + strong-rule scan)", "bound": "hbm",
                                 "achieved": achieved, "peak": pk["hbm_gbs"], "peak_source": pk_src, "unit": "GB/s",
                                 "frac": achieved / pk["hbm_gbs"] if achieved else None, "traffic": traffic}),
                     "scan_ms_per_step": scan_ms / args.steps, "scan_launches_per_step": scan_launches / args.steps,
                     "cd_ms_per_step": cd_ms / args.steps, "cd_visits_per_step": visits,
                     "cd_updates_per_step": updates,
                     "cd_ns_per_visit": cd_ms / args.steps * 1e6 / max(visits, 1),
                     "cd_kernel_cycles_per_visit": cd_cycles / max(visits, 1),
                     "cd_kernel_ms_per_step": cd_cycles / 1.965e6,
                     "cd_phase_cycles_per_visit": dict(zip(["cd_passes", "weights_v", "eta", "intercept (within cd_passes)"] if is_logit else ["lead", "bulk", "build_A", "catch_up"], cd_prof)),
                     "algorithmic_bytes_per_step": scan_bytes / args.steps,
                     "dominant_kernel_note": ("the fused scan is the method's bandwidth-bound kernel and BASELINE's metric; "
                                              "by time the sequential CD (k_cd_gram7) dominates when cd_ms_per_step > "
                                              "scan_ms_per_step -- it is latency-bound (no roofline), reported as "
                                              "cd_ns_per_visit / cd_kernel_cycles_per_visit"),
                     "full_scan": ({"GBps": fs_bytes / (fs_ms / 1e3) / 1e9,
                                    "frac": fs_bytes / (fs_ms / 1e3) / 1e9 / (link_gbs if host_res else pk["hbm_gbs"]),
                                    "launches_per_step": fs_launches} if fs_ms > 0 else None)},
        "cpu_baseline": cpu,
        "e2e": ({"value": statistics.median(e2e), "unit": "s", "h2d_bytes_per_step": int(h2d),
                 "d2h_bytes_per_step": d2h, "design_load_s": statistics.median(e2e_load),
                 "samples_s": e2e} if e2e else
                {"value": None, "unit": "s", "note": "X > 40 GB: no pinned host copy on this box"}),
        "gpu_launches": int(launches / args.steps),
        "path": {"nnz_last": int(last.col_ptr[-1] - last.col_ptr[-2]), "kkt_rounds": int(last.kkt_rounds.sum()),
                 "cd_passes": int(last.passes.sum()), "cols_scanned": int(last.cols_scanned.sum()),
                 "n_converged": int(last.n_converged),
                 # Fig 1 analog: fraction of live columns BEDPP keeps, by lambda/lambda_max
                 "bedpp_kept_frac": {f"{q:.1f}": float(last.n_safe[int(np.argmin(np.abs(lams / lm - q)))] / p_global)
                                     for q in (0.9, 0.7, 0.5, 0.3)},
                 "max_working_set": int(last.n_working.max()),
                 **({"irls_iterations": int(last.outer.sum())} if hasattr(last, "outer") else {})},
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "logit"],
                    help="BASELINE cfg1-cfg5, or 'logit' (NEXT-3 logistic path, n=1000, p=100,000 fp32)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--resident", default="device", choices=["device", "host"],
                    help="where X lives: HBM (default) or pinned host memory read over PCIe (NEXT-4, out-of-core)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=20.0,
                    help="cpu_baseline time budget: the oracle runs lambdas of the grid until it is spent")
    ap.add_argument("--cv-mode", default="batched", choices=["batched", "batched_dmma", "batched_fma", "independent"],
                    help="cfg5: the fold-batched scan kernel (bl_opts.cv_mode)")
    ap.add_argument("--cd", default="auto", choices=["auto", "residual", "gram"],
                    help="CD flavour: residual updates (r on chip) or covariance updates (NEXT-2)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
