#!/usr/bin/env python
"""Benchmark: train/test scenario evaluations per second of the fused
Tier-2/Tier-3 path (arXiv 1910.07776) on B200, with the roofline of the
dominant kernel and the CPU oracle as a reported baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

One step = one sr_evaluate call over the rank's batch of scenarios: A0 rates,
A1 labels + pairs, A2-A7 fused (three kernel launches).  Default workload =
config C3 (2 programs x 64 variants x 64 counters, 1e6 random train/test
splits per GPU; weak scaling: rank r evaluates splits [r*S, (r+1)*S)).
Under torchrun each rank drives one GPU and evaluates its own scenario
shard with no collective on the data path; each step then gathers the
per-scenario score tables to rank 0 with one NCCL all_gather_into_tensor per
table (inside the timed step, also reported on its own as
`gather`), and the pooled integer totals and the timing are all-reduced.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_FMA_PER_CLK_PER_SM = 64   # inferred from the measured DMMA loop (profiles/fp64_peak.txt)


def fit_flops(n: np.ndarray, t: np.ndarray, d: int, refine: int = 2, predict: bool = True) -> float:
    """Algorithmic FP64 flops of the fits a batch performed:
    per fit with n training pairs, t test cases and d active features,
      dual   (n-1 < d): n(n+1)/2*d + n^3/6 + n^2 + R*(2nd + n^2) + nd + td   FMA
      primal (else)   : n*d(d+1)/2 + d^3/6 + nd + d^2 + R*(2nd + d^2) + td   FMA
    R = refine when the fit's rule asks for it (dual: 2(n-1) >= d, primal:
    n-1 < 2d or n > 64), else 0.  flop = 2 * FMA.  Fits with
    n == 0 or t == 0 do no work.  predict=False drops the t*d prediction term
    (the split LS path predicts in k_pred_rank)."""
    n = n.astype(np.float64)
    t = t.astype(np.float64) if predict else np.zeros_like(n) + (t > 0)
    live = (n > 0) & (t > 0)
    t = t * (1.0 if predict else 0.0)
    dual = (n - 1) < d
    rd = np.where(2 * (n - 1) >= d, refine, 0)
    rp = np.where(((n - 1) < 2 * d) | (n > 64), refine, 0)
    fd = n * (n + 1) / 2 * d + n ** 3 / 6 + n ** 2 + rd * (2 * n * d + n ** 2) + n * d + t * d
    fp = n * d * (d + 1) / 2 + d ** 3 / 6 + n * d + d ** 2 + rp * (2 * n * d + d ** 2) + t * d
    return float(2.0 * np.where(live, np.where(dual, fd, fp), 0.0).sum())


def fit_flops_big(n: np.ndarray, t: np.ndarray, d: int, refine: int = 0) -> float:
    """k_fit_big (C4 path, primal; prediction is in k_rank_big): SURVEY 8(d)'s
    C4 yardstick n*d(d+1)/2 + d^3/6 + nd + d^2 FMA per fit, flop = 2 FMA.  The
    refinement passes (adaptive) are not counted: the yardstick
    says none is needed, they are the kernel's accuracy insurance."""
    n = n.astype(np.float64)
    live = (n > 0) & (t > 0)
    f = n * d * (d + 1) / 2 + d ** 3 / 6 + n * d + d ** 2 + refine * (2 * n * d + d ** 2)
    return float(2.0 * np.where(live, f, 0.0).sum())


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, fl in rows for i, f in enumerate(fl) if f.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def oracle_rate(cfg, first: int, count: int, threads: int, learner: int = 0, stats: dict | None = None):
    """Scenarios/s of the oracle as it stands on `threads` host threads over
    scenarios [first, first+count).  stats (LS learner): filled with the
    sample's kappa^ statistics and the long-double share."""
    import oracle
    t0 = time.perf_counter()
    if learner == 2:    # M5P: the exact-rational Python oracle (oracle/m5.py), one core
        from oracle import m5
        m5.evaluate(cfg.dataset, cfg.scenarios, first, count)
    else:
        r = oracle.evaluate(cfg.dataset, cfg.scenarios, first, count, n_threads=threads, learner=learner,
                            want_kappa=stats is not None and learner == 0)
        if stats is not None and r["kappa"] is not None:
            k = r["kappa"][np.isfinite(r["kappa"])]
            if k.size:
                stats.update(kappa_min=float(k.min()), kappa_median=float(np.median(k)), kappa_max=float(k.max()),
                             fits=int(k.size), long_double_fits=int(r["fit_ld"].sum()),
                             guard_cases=int(r["scn"]["n_guard"].sum()))
    return count / (time.perf_counter() - t0)


def ibk_fit_rate(cfg, threads: int) -> float:
    """C4 under IBK: one scenario is 6 fits of n*t*d ~ 1.7e10 distance terms
    each (minutes of oracle time), so the bounded sample is ONE fit (split 0,
    optimization O0) on one core; scenarios/s = 1 / (6 x its time)."""
    import copy
    import oracle
    sc = copy.copy(cfg.scenarios)
    sc.opt_mask = 1
    t0 = time.perf_counter()
    oracle.evaluate(cfg.dataset, sc, 0, 1, n_threads=1, learner=1)
    return 1.0 / (6.0 * (time.perf_counter() - t0))


# Context (Table 3): the paper's sign accuracies, measured on a
# Tesla K20c (0.7 GHz Kepler, 13 SMX) with nvprof 6.5 profiles of BH/NB and
# Weka's IBK / M5P.  Different data and hardware: context, not a target.
PAPER_TABLE3 = {
    "source": "PAPER.md Table 3 (P:216-224)",
    "profiled_on": "Tesla K20c (Kepler, 0.7 GHz, 13 SMX), nvcc 6.0.1 -O3 -arch=sm_35, nvprof 6.5, Weka",
    "ibk_pct": {"1": 97.3, "2": 96.0, "3": 96.3, "4": 92.0, "5": 83.6, "6": 55.7},
    "m5p_pct": {"1": 86.4, "2": 86.4, "3": 33.3, "4": 81.6, "5": 33.3, "6": 60.1},
    "note": "context only: the paper's K20c data; this run is synthetic data (DESIGN.md 8)",
}


def per_experiment_accuracy(cfg, opt_rows) -> dict | None:
    """Pooled sign accuracy per Table-2 experiment of this run (C2 / BH6)."""
    exp = getattr(cfg.scenarios, "experiment", None)
    if exp is None:
        return None
    out = {}
    for e in sorted(set(int(x) for x in exp)):
        sel = exp[:len(opt_rows)] == e
        t = int(opt_rows["n_test"][sel].astype(np.int64).sum())
        c = int(opt_rows["n_correct"][sel].astype(np.int64).sum())
        out[str(e)] = round(100.0 * c / t, 2) if t else None
    return out


def oracle_cores(threads: int, learner: int) -> int:
    return 1 if learner == 2 else threads


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle (this tier's reference arm) on host cores."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample = args.ref_sample
    for _ in range(args.warmup):
        oracle_rate(cfg, 0, max(threads, sample // 10), threads, LEARNERS[args.learner])
    rates = []
    for k in range(args.steps):
        rates.append(oracle_rate(cfg, (k * sample) % cfg.scenarios.n_splits, sample, threads, LEARNERS[args.learner]))
    v = float(np.mean(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "scenario_evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sample / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64+rational" if args.learner == "m5" else "f64+quad",
        "data": "synthetic", "config": workload_config(cfg, args, sample),
        "cpu_baseline": {"value": v, "unit": "scenario_evals/s", "cores": oracle_cores(threads, LEARNERS[args.learner]),
                         "kind": "oracle",
                         "sample": f"{sample} scenarios of {args.config} per step (splits "
                                   f"[k*{sample}, (k+1)*{sample}))"},
        "e2e": {"value": v, "unit": "scenario_evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


LEARNERS = {"linreg": 0, "ibk": 1, "m5": 2}


def run_sweep(args, cfg, count):
    """--sweep T: the Tier-3 rule sweep (sr_sweep, NEXT-3) over the config's
    scenarios, T thresholds in [0.8, 1.4] x list lengths {1, 2, 3, 6}; one
    step = fits + the sweep kernel.  Single GPU."""
    import torch
    from paper_1910_07776_b200 import Context
    from paper_1910_07776_b200.speedrec import default_params
    torch.cuda.set_device(0)
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    thr = np.linspace(0.8, 1.4, args.sweep)
    cnt = np.array([1, 2, 3, 6])
    prm = default_params(learner=LEARNERS[args.learner])
    for _ in range(args.warmup):
        ctx.sweep(thr, cnt, 0, count, params=prm)
    ctx.set_timing(True)
    ctx.reset_kernel_stats()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rec, hit = ctx.sweep(thr, cnt, 0, count, params=prm)
    dt = (time.perf_counter() - t0) / args.steps
    stats = ctx.kernel_stats()
    ctx.close()
    i = int(np.argmin(abs(thr - 1.05)))
    print(json.dumps({
        "metric": "Tier-3 rule sweep: scenario evals/sec (fits + rule grid)", "value": count / dt,
        "unit": "scenario_evals/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt, "higher_is_better": True, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.description}", "scenarios": count,
                   "thresholds": int(args.sweep), "list_lengths": cnt.tolist()},
        "kernels": {k: {"launches": v[0], "ms": v[1]} for k, v in stats.items()},
        "precision_at_theta_%.3f" % thr[i]: {str(int(k)): float(hit[i, j] / max(rec[i, j], 1))
                                            for j, k in enumerate(cnt)},
    }), flush=True)


def knn_flops(n: np.ndarray, t: np.ndarray, d: int) -> float:
    """IBk (NEXT-1): per fit n*t*d distance terms, each a subtract and an FMA
    (3 flop); the scaling divisions and the k-best inserts are not counted."""
    n = n.astype(np.float64)
    t = t.astype(np.float64)
    return float(3.0 * np.where((n > 0) & (t > 0), n * t * d, 0.0).sum())


def m5_flops(n: np.ndarray, t: np.ndarray, d: int) -> float:
    """M5P (NEXT-2) yardstick: the root split search alone -- d features x
    (n - 1) candidate thresholds x two passes over the n rows (an add, and a
    subtract + multiply + add: 4 flop per row); the deeper nodes, the node
    models and the prediction are not counted."""
    n = n.astype(np.float64)
    t = t.astype(np.float64)
    return float(np.where((n > 1) & (t > 0), 4.0 * d * (n - 1) * n, 0.0).sum())


OTHER_CONFIGS = [("C1", "C1", ["--cpu-sample", "64"]), ("C2", "C2", ["--cpu-sample", "240"]),
                 ("C2-ibk", "C2", ["--learner", "ibk", "--cpu-sample", "240"]),
                 ("C2-m5", "C2", ["--learner", "m5", "--cpu-sample", "24"]),
                 ("C4", "C4", ["--splits", "592", "--cpu-sample", "32"]),
                 ("C5", "C5", ["--masks-k", "20", "--cpu-sample", "2048"]),
                 ("C4-ibk", "C4", ["--splits", "16", "--learner", "ibk"]),
                 ("C3-m5", "C3", ["--splits", "65536", "--learner", "m5", "--cpu-sample", "32"])]


def run_other_configs(args):
    """Secondary lines: the other four configs, each in its own process
    (same GPU, after the headline measurement), summarised into the headline
    JSON line under "other_configs"."""
    res = {}
    for name, cname, extra in OTHER_CONFIGS:
        cmd = [sys.executable, os.path.abspath(__file__), "--config", cname, "--steps", "5", "--warmup", "3",
               "--no-e2e", "--no-extra", "--learner", args.learner] + extra
        try:
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=600).stdout.strip().splitlines()
            d = json.loads(out[-1])
            r = d["roofline"]
            res[name] = {"value": d["value"], "unit": d["unit"], "ms_per_step": d["ms_per_step"],
                         "workload": d["config"]["workload"], "scenarios_per_step": d["config"]["splits_per_gpu"],
                         "scaling": d["scaling"],
                         "roofline": {k: r.get(k) for k in ("bound", "kernel", "achieved", "peak", "unit", "frac",
                                                            "traffic", "traffic_note", "kernel_share_of_step",
                                                            "effective", "frac_yardstick_p_eq_S")},
                         "cpu_baseline": d.get("cpu_baseline"), "accuracy": d.get("accuracy"),
                         "guard_cases": d.get("guard_cases"),
                         "top_masks_head": d.get("top_masks_head")}
        except Exception as e:   # reported, never fatal for the headline line
            res[name] = {"error": f"{type(e).__name__}: {e}"[:200]}
    return res


METRIC = "train/test scenario evals/sec at 1/2/4/8 B200 (roofline frac) vs CPU oracle"


def workload_config(cfg, args, per_gpu):
    ds = cfg.dataset
    return {"workload": f"{cfg.name}: {cfg.description}", "splits_per_gpu": per_gpu, "learner": args.learner,
            "programs": ds.n_programs, "variants": ds.n_slots, "counters": ds.n_counters,
            "optimizations": ds.n_opt_ids, "parallelism": f"scenario-sharded x{args.gpus}",
            "l2": "flushed between timed steps (256 MiB write); dataset 64 KiB is L2/smem resident by design"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--splits", type=int, default=None, help="scenarios per GPU (default: config size)")
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--masks-k", type=int, default=10,
                    help="C5: all 2^k subsets of counters [0, k) (the full config is k = 20)")
    ap.add_argument("--learner", default="linreg", choices=list(LEARNERS),
                    help="linreg = ridge LS (the paper's model); ibk = the NEXT-1 k-NN learner; "
                         "m5 = the NEXT-2 M5P model tree")
    ap.add_argument("--ref-sample", type=int, default=None,
                    help="scenarios per reference-arm step (default 4000; 32 for the Python M5P oracle)")
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="scenarios of the cpu_baseline sample (default 4000; 32 for the Python M5P oracle)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end leg (tuning runs)")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the secondary per-config lines (C1, C2, C4, C5) of the default run")
    ap.add_argument("--dump-tables", default=None,
                    help="rank 0 writes the gathered score tables (npz) here (tests/test_gpu_dist.py)")
    ap.add_argument("--sweep", type=int, default=0,
                    help="NEXT-3: time sr_sweep with this many thresholds x 4 list lengths instead of sr_evaluate")
    args = ap.parse_args()
    small = args.learner == "m5"            # the exact-rational Python oracle is ~1e4x slower
    if args.ref_sample is None:
        args.ref_sample = 32 if small else 4000
    if args.cpu_sample is None:
        args.cpu_sample = 32 if small else 4000

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import gen
    per_gpu = args.splits or {"C3": 1_000_000, "C1": 64, "C2": 240}.get(args.config, 100_000)
    cfg = gen.make_config(args.config, n_splits=per_gpu * world if args.config in ("C3", "C4") else None,
                          n_masks_k=args.masks_k if args.config == "C5" else None)
    if args.config not in ("C3", "C4"):
        per_gpu = cfg.scenarios.n_scenarios // world

    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    if args.sweep:
        return run_sweep(args, cfg, per_gpu)

    import torch
    from paper_1910_07776_b200 import dist as D
    local = local % max(torch.cuda.device_count(), 1)   # (ranks > GPUs only for gloo smoke runs)
    torch.cuda.set_device(local)
    dist = None
    backend = os.environ.get("SPEEDREC_DIST_BACKEND", "nccl")
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    xdev = "cpu" if backend != "nccl" else torch.device("cuda", local)   # device of exchanged tensors
    from paper_1910_07776_b200 import Context
    from paper_1910_07776_b200.speedrec import OPT_SCORE_DTYPE, SCN_SCORE_DTYPE
    stream = torch.cuda.Stream(device=local)      # one explicit stream for the library and the events
    torch.cuda.set_stream(stream)
    ctx = Context(local, stream=stream.cuda_stream)
    ds = cfg.dataset
    ctx.load(ds)
    ctx.define_scenarios(cfg.scenarios)
    O = ds.n_opt_ids
    dev = torch.device("cuda", local)
    c5 = args.config == "C5"
    if c5:
        # C5: popcount-stratified round-robin of the 2^k masks,
        # per-mask sums over the 128 LOO folds + top-64 in the kernels
        masks = D.stratified_masks(args.masks_k, rank, world)
        sc = cfg.scenarios
        sc.all_subsets_k = 0
        sc.feature_masks = np.stack([masks.astype(np.uint64), np.zeros(len(masks), np.uint64)], 1)
        sc.n_masks = len(masks)
        ctx.define_scenarios(sc)
        folds = sc.n_splits
        first, count = 0, len(masks) * folds
        out = dict(masks=torch.empty(len(masks) * 16, dtype=torch.uint8, device=dev),
                   top=torch.empty(64, dtype=torch.int64, device=dev),
                   totals=torch.zeros(4, dtype=torch.int64, device=dev))
    else:
        first, count = D.weak_range(per_gpu, rank)           # scenario shard of this rank
        out = dict(opt=torch.empty(count * O * OPT_SCORE_DTYPE.itemsize, dtype=torch.uint8, device=dev),
                   scn=torch.empty(count * SCN_SCORE_DTYPE.itemsize, dtype=torch.uint8, device=dev),
                   totals=torch.zeros(4, dtype=torch.int64, device=dev))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    from paper_1910_07776_b200.speedrec import default_params
    prm = default_params(learner=LEARNERS[args.learner], top_k=64)

    # score-table gather: fixed-size rows, rank order = scenario order
    if c5:
        all_masks = [D.stratified_masks(args.masks_k, r, world) for r in range(world)]
        mpad = torch.zeros(max(len(m) for m in all_masks) * 16, dtype=torch.uint8, device=dev)

    def gather_tables():
        if c5:
            mpad[:out["masks"].numel()].copy_(out["masks"])
            return {"masks": D.gather_rows(mpad.to(xdev), dist)}
        return {"opt": D.gather_rows(out["opt"].to(xdev), dist), "scn": D.gather_rows(out["scn"].to(xdev), dist)}

    for _ in range(args.warmup):
        ctx.evaluate(first, count, params=prm, out=out)
    torch.cuda.synchronize()

    # ---------------- timed region: K steps, device events, L2 flushed between steps
    ctx.set_timing(True)
    ctx.reset_kernel_stats()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    gevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    tables = None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            ctx.evaluate(first, count, params=prm, out=out)
            gevs[k][0].record(stream)
            if world > 1:
                tables = gather_tables()
            gevs[k][1].record(stream)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    if tables is None:
        tables = gather_tables()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    gather_ms = D.max_over_ranks(float(np.mean([a.elapsed_time(b) for a, b in gevs])), dist, device=xdev)
    stats = ctx.kernel_stats()
    ctx.set_timing(False)
    launches = sum(v[0] for v in stats.values())
    my_ms = float(np.mean(step_ms))
    ms = D.max_over_ranks(my_ms, dist, device=xdev)           # max over ranks (device-timed)
    tot = D.reduce_totals(out["totals"].to(xdev), dist)       # pooled A7 totals (exact)
    # whole-job throughput: every scenario all ranks evaluated (C5: all 2^k masks x folds)
    value = ((1 << args.masks_k) * folds if c5 else world * count) / (ms / 1e3)

    # ---------------- roofline of the dominant kernel (FP64 ALU/DMMA bound)
    big = ds.n_groups > 64          # CTA-per-fit path (C4): prediction runs in k_rank_big
    flops_pd = None
    flops_all = None
    name_dom = ("k_ibk_dist" if args.learner == "ibk" else "k_fit_big") if big else "k_fit_warp"
    if c5:
        # n, t per (fold, opt) do not depend on the mask: take them from one
        # untimed per-scenario pass over the folds of this rank's first mask,
        # then d = popcount(mask) per mask
        r1 = ctx.evaluate(0, folds, params=prm)
        n_tr, n_te = r1["opt"]["n_train"].ravel(), r1["opt"]["n_test"].ravel()
        pcs = np.array([bin(int(m)).count("1") for m in masks])
        if stats.get("k_mask_sfit", (0, 0.0))[0] > 0 or stats.get("k_mask_fit", (0, 0.0))[0] > 0:
            # feature-mask paths: per fit on the precomputed Gram;
            # the prefix-shared path (k_mask_sfit) does less
            # arithmetic than this yardstick, so its fraction is an effective one
            name_dom = "k_mask_sfit" if stats.get("k_mask_sfit", (0, 0.0))[0] > 0 else "k_mask_fit"
            n_fit = float(np.sum((n_tr > 0) & (n_te > 0)))
            # SURVEY 8(d)'s yardstick: p = |S| + 1 (mask features + intercept)
            ff = lambda d: n_fit * 2.0 * ((d + 1) ** 3 / 6 + (d + 1) ** 2 + (d + 1))
            ff_pd = lambda d: n_fit * 2.0 * (d ** 3 / 6 + d ** 2 + d)   # round-1's conservative p = |S|
        elif args.learner == "ibk":
            ff = lambda d: knn_flops(n_tr, n_te, d)
        elif args.learner == "m5":
            ff = lambda d: m5_flops(n_tr, n_te, d)
        else:
            ff = lambda d: fit_flops(n_tr, n_te, d, refine=2)
        flops_launch = sum(float(np.sum(pcs == d)) * ff(int(d)) for d in np.unique(pcs))
        if name_dom in ("k_mask_sfit", "k_mask_fit"):
            flops_pd = sum(float(np.sum(pcs == d)) * ff_pd(int(d)) for d in np.unique(pcs))
    else:
        opt = out["opt"].cpu().numpy().view(OPT_SCORE_DTYPE).reshape(count, O)
        n_tr, n_te = opt["n_train"].ravel(), opt["n_test"].ravel()
        if args.learner == "ibk":
            flops_launch = knn_flops(n_tr, n_te, ds.n_counters)
        elif args.learner == "m5":
            # executed split-search FP64 operations of the step's grown trees
            # (sr_last_work, the last timed evaluate); root-only yardstick as fallback
            work = ctx.last_work()
            flops_launch = float(work) if work > 0 else m5_flops(n_tr, n_te, ds.n_counters)
        elif big:
            flops_launch = fit_flops_big(n_tr, n_te, ds.n_counters)
        else:
            split = stats.get("k_pred_rank", (0, 0.0))[0] > 0     # split LS path: prediction in k_pred_rank
            flops_launch = fit_flops(n_tr, n_te, ds.n_counters, refine=2, predict=not split)
            flops_all = fit_flops(n_tr, n_te, ds.n_counters, refine=2)
    n_dom, ms_dom = stats.get(name_dom, (0, 0.0))
    avg_dom = ms_dom / max(n_dom, 1)                 # average launch duration (CUDA events, live)
    launches_per_step = max(n_dom // max(args.steps, 1), 1)
    flops_step = flops_launch                        # algorithmic flops of one step (all chunks)
    flops_launch = flops_step / launches_per_step    # chunks are equal-sized slices of the batch
    # DRAM traffic of one launch of the dominant kernel from the committed ncu
    # capture (profiles/traffic.json), when this run has the captured launch shape
    traffic, traffic_note = None, None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        ent = tj.get(name_dom)
        if ent and ent["workload"] == args.config and ent.get("learner", "linreg") == args.learner:
            per_unit = (ent["read"] + ent["write"]) / ent["units"]
            units = ent["units"] if name_dom == "k_mask_sfit" else count / launches_per_step
            traffic = per_unit * units
            traffic_note = f"{per_unit:.0f} B per {ent['per']} x {units:.0f} units per launch; {ent['source']}"
    except (OSError, ValueError, KeyError):
        pass
    clk_sum = clk.summary()
    sm_max = clk_sum.get("sm_max_mhz") or 1965.0
    props = torch.cuda.get_device_properties(dev)
    peak = props.multi_processor_count * FP64_FMA_PER_CLK_PER_SM * 2 * sm_max * 1e6 / 1e12
    # = flops per launch / average launch time; also right for unequal launches
    achieved = flops_step / (ms_dom / max(args.steps, 1) / 1e3) / 1e12 if ms_dom > 0 else 0.0
    share = ms_dom / max(sum(v[1] for v in stats.values()), 1e-9)
    # whole step: every algorithmic flop of the path over the step time (the
    # split LS path's prediction runs in k_pred_rank, outside the fit kernel)
    step_achieved = (flops_all if flops_all is not None else flops_step) / (ms / 1e3) / 1e12            # per GPU

    # ---------------- end to end: host buffers through the C-ABI, copies inside
    e2e = None
    if not args.no_e2e:
        hc = torch.from_numpy(ds.counters).pin_memory()
        hy = torch.from_numpy(ds.cycles).pin_memory()
        hr = torch.from_numpy(ds.runtime_ms).pin_memory()
        hb = torch.from_numpy(ds.opt_bit).pin_memory()
        htot = torch.zeros(4, dtype=torch.int64).pin_memory()
        from paper_1910_07776_b200.speedrec import sr_outputs, lib
        import ctypes as ct
        if c5:
            hmask = torch.empty(len(masks) * 16, dtype=torch.uint8).pin_memory()
            htop = torch.empty(64, dtype=torch.int64).pin_memory()
            hout = sr_outputs(None, None, None, None, htot.data_ptr(), hmask.data_ptr(), htop.data_ptr(), 0)
            d2h = hmask.numel() + htop.numel() * 8 + 32
        else:
            hopt = torch.empty(count * O * OPT_SCORE_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
            hscn = torch.empty(count * SCN_SCORE_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
            hout = sr_outputs(hopt.data_ptr(), hscn.data_ptr(), None, None, htot.data_ptr(), None, None, 0)
            d2h = hopt.numel() + hscn.numel() + 32
        e2e_ms = []
        for k in range(max(2, min(args.steps, 5)) + 1):
            flush.fill_(float(k))
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.load_dataset(ds.n_programs, ds.n_inputs, ds.n_runs, ds.n_counters, ds.n_opt_ids,
                             hc.numpy(), hy.numpy(), hr.numpy(), hb.numpy())
            ctx.define_scenarios(cfg.scenarios)
            ctx._check(lib().sr_evaluate(ctx._h, ct.byref(prm), first, count, ct.byref(hout)))
            b.record(stream)
            torch.cuda.synchronize()
            if k > 0:
                e2e_ms.append(a.elapsed_time(b))
        te = D.max_over_ranks(float(np.mean(e2e_ms)), dist, device=xdev)
        e2e = {"value": world * count / (te / 1e3), "unit": "scenario_evals/s",
               "h2d_bytes_per_step": int(hc.numel() * 8 + hy.numel() * 8 + hr.numel() * 8 + hb.numel()),
               "d2h_bytes_per_step": int(d2h)}

    # ---------------- CPU oracle baseline (rank 0, N=1 only, bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        L = LEARNERS[args.learner]
        if big and L == 1:
            v = v1 = ibk_fit_rate(cfg, threads)
            cores, st = 1, {}
            sample = "1 of the 6 fits of split 0 (optimization O0) on one core, scenarios/s = 1/(6 t)"
        else:
            st = {}
            v = oracle_rate(cfg, 0, args.cpu_sample, threads, L, stats=st)
            cores = oracle_cores(threads, L)
            n1 = max(1, args.cpu_sample // threads)       # single-core rate on ~1/threads of the sample
            v1 = oracle_rate(cfg, 0, n1, 1, L) if cores > 1 else v
            sample = f"first {args.cpu_sample} scenarios of {args.config} (same splits the GPU evaluates)"
        cpu = {"value": v, "unit": "scenario_evals/s", "cores": cores, "kind": "oracle", "sample": sample,
               "nproc": threads, "single_core_value": v1,
               "precision": "quad; long double for p > 65 overdetermined fits (SURVEY 8(c))" if L == 0 else
               ("exact IEEE (bit-exact definition)" if L == 1 else "FP64 + exact rationals (Python)"),
               "kappa": st or None}

    # rank 0: the gathered tables in global scenario (C5: mask) order
    gathered, pooled, guard_cases, per_exp = None, None, None, None
    if rank == 0:
        if c5:
            gathered = {"masks": D.scatter_mask_rows(tables["masks"].cpu().numpy(), all_masks, 1 << args.masks_k)}
        else:
            gathered = {k: v.cpu().numpy() for k, v in tables.items()}
            pooled = D.pooled_ratio(gathered["opt"])
            from paper_1910_07776_b200.speedrec import OPT_SCORE_DTYPE as _OD, SCN_SCORE_DTYPE as _SD
            g_opt = gathered["opt"].view(_OD).reshape(-1, O)
            guard_cases = int(gathered["scn"].view(_SD)["n_guard"].astype(np.int64).sum())
            per_exp = per_experiment_accuracy(cfg, g_opt)
    top_global = None
    if c5:   # C5 A7: local top-64 (library) -> global mask ids -> exact merge over ranks
        from paper_1910_07776_b200.speedrec import MASK_SCORE_DTYPE
        rows = out["masks"].cpu().numpy().view(MASK_SCORE_DTYPE)
        tl = out["top"].cpu().numpy()
        corr = [int(rows["n_correct"][i]) if i >= 0 else 0 for i in tl]
        top_global = D.merge_top_masks(D.local_top_to_global(tl, masks).tolist(), corr, 64, dist, device=xdev)
    if rank == 0:
        tt = tot.cpu().numpy()
        line = {
            "metric": METRIC, "value": value, "unit": "scenario_evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if c5 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, args, count),
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic, "traffic_note": traffic_note,
                         "kernel": name_dom, "kernel_ms": avg_dom, "kernel_share_of_step": share,
                         "flops_per_launch": flops_launch, "launches_per_step": launches_per_step,
                         "peak_note": f"FP64 (DFMA/DMMA shared pipe): {props.multi_processor_count} SMs x "
                                      f"{FP64_FMA_PER_CLK_PER_SM} FMA/clk x 2 x {sm_max:.0f} MHz",
                         "effective": name_dom == "k_mask_sfit",
                         "step_achieved": step_achieved, "step_frac": step_achieved / peak if peak else None,
                         "frac_yardstick_p_eq_S": (flops_pd / (ms_dom / max(args.steps, 1) / 1e3) / 1e12 / peak
                                                   if flops_pd and ms_dom > 0 else None),
                         "flops_note": ("SURVEY 8(d) C5 yardstick p^3/6+p^2+p per fit on the precomputed "
                                        "Gram with p = |S|+1; the prefix-shared path (DESIGN 5.8) executes fewer flops, "
                                        "so frac is an effective fraction" if name_dom == "k_mask_sfit"
                                        else "M5P: the FP64 operations the grown trees' split searches "
                                        "executed (sr_last_work: first-pass adds + second-pass sub/mul/add per "
                                        "candidate, DESIGN 5.11)" if args.learner == "m5"
                                        else "algorithmic flops of the fits, prediction (t d) counted in "
                                        "k_pred_rank's share when the split LS path runs (DESIGN 5.12, 6); "
                                        "step_* = all algorithmic flops over the whole step")},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "gather": {"collective": "all_gather_into_tensor" if world > 1 else "none (1 GPU)",
                       "backend": backend if world > 1 else None, "ms_per_step": gather_ms,
                       "bytes_per_rank": int(sum(v.numel() for v in tables.values()) // world) if world > 1 else 0,
                       "in_step": True},
            "pooled_ratio": pooled, "guard_cases": guard_cases,
            "paper_context": PAPER_TABLE3,
            "clocks": clk_sum,
            "accuracy": {"pooled_sign_accuracy_pct": 100.0 * tt[0] / max(tt[1], 1), "cases": int(tt[1]),
                         "recommendations": int(tt[2]), "rec_hits": int(tt[3]),
                         "per_experiment_pct": per_exp, "learner": args.learner, "data": "synthetic"},
            "kernels": {k: {"launches": v[0], "ms": v[1]} for k, v in stats.items()},
        }
        if c5:
            line["config"].update(masks_k=args.masks_k, masks_per_gpu=int(len(masks)), folds=int(folds),
                                  partition="popcount-stratified round-robin (SURVEY 8(e))")
            line["top_masks_head"] = [int(m) for m in top_global[:8]]
        if args.dump_tables:
            extra = {"top": np.asarray(top_global)} if c5 else {}
            np.savez(args.dump_tables, totals=tot.cpu().numpy(), **gathered, **extra)
        if world == 1 and args.config == "C3" and not args.no_extra:
            ctx.synchronize()
            line["other_configs"] = run_other_configs(args)
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
