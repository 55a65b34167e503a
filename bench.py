#!/usr/bin/env python
"""Benchmark of the EI cost+gradient hot path (one `ei_cost_grad` = one step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Workload: BASELINE.json configs[3] (C4: a stack of 64 slices of 512x512, 720 angles over 180 deg,
768 detector pixels, M=7, per-angle mask drift) by default -- the largest configuration that
fits one GPU (991 MB of measured curves, 65.4 G ray-sample updates per evaluation); --config
C1..C5 selects another (C2 is the small latency-bound slice, C1 the oracle-sized case).  Inputs are synthetic
(paper_2202_08627_b200.synth), resident in HBM before the timed region; L2 is flushed
(256 MiB write, untimed) before every timed step.  Each step is timed with CUDA events on
the launching stream; per-kernel times come from events the library records around its own
launches during the same timed steps (ei_plan_set_timing).  N>1 (torchrun): one process per
GPU, each rank evaluates its own seeded slice set (slices are independent problems,
PAPER.md:203): no collective on the data path, weak scaling, max-over-ranks timing.

`--impl reference` times the fp64 CPU oracle (oracle/, the correctness reference) on the host
cores, on bounded samples of the same workload.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2202_08627_b200 import dist as edist  # noqa: E402
from paper_2202_08627_b200 import synth  # noqa: E402

METRIC = "cost+gradient evals/sec"
UNIT = "evals/s"


def load_traffic(cfg_name, kernel):
    """roofline.traffic: DRAM bytes (read + write) per launch of `kernel` from the committed
    `ncu --set full` capture of this config (profiles/traffic.json, tools/ncu_traffic.py)."""
    try:
        e = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))[cfg_name]
        return e["kernels"][kernel]["dram_bytes_per_launch"], e["source"]
    except Exception:
        return None, None


def load_traffic_field(cfg_name, kernel, field):
    try:
        e = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))[cfg_name]
        return e["kernels"][kernel].get(field)
    except Exception:
        return None


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


ONCHIP_PEAKS = os.path.join("profiles", "r02", "peaks.json")


def onchip_peak(sm_mhz):
    """K1/K3 roofline peak: the shared-memory (LDS.128) bandwidth MEASURED on a B200 of this pool
    by tools/microbench.cu (tools/measure_peaks.py -> profiles/r02/peaks.json, with the SM clock
    seen during that measurement), scaled to this run's median SM clock.  Falls back to the
    guide's unit count (128 B/clk/SM x 148 SMs x clock) only if the file is missing."""
    try:
        d = json.load(open(os.path.join(ROOT, ONCHIP_PEAKS)))
        mhz0 = d.get("sm_mhz") or sm_mhz          # SM clock inside the microbenchmark kernel
        peak = d["smem_lds128_gbs"] * sm_mhz / mhz0
        return peak, ("measured: LDS.128 %.0f GB/s at %.0f MHz (%s), x %.0f/%.0f MHz this run"
                      % (d["smem_lds128_gbs"], mhz0, ONCHIP_PEAKS, sm_mhz, mhz0))
    except Exception:
        return (128.0 * 148 * sm_mhz * 1e6 / 1e9,
                "derived (no measured file): 128 B/clk/SM x 148 SMs x %.0f MHz" % sm_mhz)


# ---------------------------------------------------------------------------------------
# algorithmic counts
# ---------------------------------------------------------------------------------------
def ray_sample_updates(cfg) -> int:
    """Exact number of (ray, dominant line) Joseph samples with >= 1 tap inside the grid,
    per slice per direction (SURVEY.md §8(d) definition), in fp64."""
    N, ND = cfg.N, cfg.n_det
    ctr, dctr = (N - 1) / 2.0, (ND - 1) / 2.0
    y = np.arange(N) - ctr
    k = np.arange(ND) - dctr
    total = 0
    for th in cfg.angles:
        c, s = np.cos(th), np.sin(th)
        cd, so = (c, s) if abs(c) >= abs(s) else (s, c)
        xs = (k[:, None] * cfg.det_pitch / cd) / cfg.pixel - (so / cd) * y[None, :] + ctr
        total += int(np.count_nonzero((xs > -1.0) & (xs < N)))
    return total


def kernel_bytes(cfg, rsu, mirror_pairs=0):
    """Algorithmic bytes per launch (all S slices): K1/K3 gather 2 taps x 3 fp32 maps per
    ray-sample update (24 B, on-chip); K2 streams P (12 B) + s_exp (4M B) in and G (12 B) out
    per (s, theta, t), flat (12 B) per (s, t).  With mirror pairs (360-degree scans, theta and
    theta + pi projected / back-projected once) K1 and K3 execute only the primaries' samples:
    the executed share is (N_theta - pairs) / N_theta (the two angles of a pair have the same
    sample count)."""
    S, NA, ND, M = cfg.S, cfg.n_angles, cfg.n_det, cfg.M
    share = (NA - mirror_pairs) / NA
    return {"K1_project": 24.0 * rsu * S * share,
            "K3_backproject": 24.0 * rsu * S * share,
            "K2_curve": float(S * NA * ND * (12 + 4 * M + 12) + S * ND * 12)}


def kernel_bytes_h(cfg, rsu, mirror_pairs=0):
    """The same for the single-map model (NEXT-3): K1/K3 gather 2 taps x 1 fp32 map (8 B) per
    ray-sample update; K2 streams P_h (4 B) + s_exp (4M B) in and the G_h pair (8 B) out per
    (s, theta, t), flat (12 B) per (s, t)."""
    S, NA, ND, M = cfg.S, cfg.n_angles, cfg.n_det, cfg.M
    share = (NA - mirror_pairs) / NA
    return {"K1_project": 8.0 * rsu * S * share,
            "K3_backproject": 8.0 * rsu * S * share,
            "K2_curve": float(S * NA * ND * (4 + 4 * M + 8) + S * ND * 12)}


def kernel_table(kb, kern_ms, n_rec, ms_step, sm_mhz, hbm_peak, cfg_name=None):
    """Per-kernel time, share of the step and roofline fraction (K1/K3 against the shared-memory
    data-pipe peak, K2 against HBM), and the dominant kernel.  Beside the algorithmic fraction, the
    DRAM bytes the committed ncu capture of this config measured per launch (profiles/traffic.json)
    over the same CUDA-event time: `dram_frac` is the kernel's HBM utilisation on its actual bytes
    (K2 writes K3's 36-B triple layout where SURVEY's algorithmic count has 12 B of gradient)."""
    per_kernel_ms = {k: v / max(n_rec, 1) for k, v in kern_ms.items()}
    l1_peak, _ = onchip_peak(sm_mhz)                                  # GB/s, DESIGN.md §6
    kernels = {}
    for k in ("K1_project", "K2_curve", "K3_backproject"):
        bound = "hbm" if k == "K2_curve" else "l1"
        peak = hbm_peak if bound == "hbm" else l1_peak
        ach = kb[k] / (per_kernel_ms[k] * 1e-3) / 1e9 if per_kernel_ms[k] > 0 else 0.0
        kernels[k] = {"ms": round(per_kernel_ms[k], 5), "share": round(per_kernel_ms[k] / ms_step, 4),
                      "bound": bound, "achieved": round(ach, 1), "peak": round(peak, 1), "unit": "GB/s",
                      "frac": round(ach / peak, 4), "bytes_per_launch": kb[k]}
        dram, _ = load_traffic(cfg_name, k) if cfg_name else (None, None)
        if dram and per_kernel_ms[k] > 0:
            dgbs = dram / (per_kernel_ms[k] * 1e-3) / 1e9
            kernels[k].update({"dram_bytes_per_launch": dram, "dram_gbs": round(dgbs, 1),
                               "dram_frac": round(dgbs / hbm_peak, 4)})
        lts = load_traffic_field(cfg_name, k, "lts_bytes_per_launch") if cfg_name else None
        if bound == "l1" and lts and per_kernel_ms[k] > 0:
            # the shared-memory data path also absorbs the TMA fills of the staging ring: their
            # bytes arrive through L2 (lts__t_bytes of the committed capture, which also counts
            # the kernel's output writes, ~1-2 %), so (gathers + fills) / time is the data path's
            # use.  K1 only: it executes its algorithmic 24 B per sample, while K3's pixel pairs
            # share entries between lanes, so bytes do not count its wavefronts (the ncu
            # summaries derive wavefronts per SM-cycle for both)
            kernels[k]["l2_bytes_per_launch"] = lts
            if k == "K1_project":
                kernels[k]["smem_frac_incl_fills"] = round(
                    (kb[k] + lts) / (per_kernel_ms[k] * 1e-3) / 1e9 / peak, 4)
    kernels["K0_pack"] = {"ms": round(per_kernel_ms["K0_pack"], 5),
                          "share": round(per_kernel_ms["K0_pack"] / ms_step, 4)}
    dom = max(("K1_project", "K2_curve", "K3_backproject"), key=lambda k: per_kernel_ms[k])
    return kernels, dom


# ---------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100",
                                          "-i", str(index)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append((time.time(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        win = [p for (t, p) in self.samples if t0 - 0.15 <= t <= t1 + 0.15]
        if not win and self.samples:   # timed region shorter than the sampling period
            mid = 0.5 * (t0 + t1)
            win = [min(self.samples, key=lambda s: abs(s[0] - mid))[1]]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(p[1]) for p in win if num(p[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in win for i in range(4) if p[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": num(win[0][2]), "reasons": reasons, "samples": len(win),
                "power_w_max": max((num(p[3]) or 0.0) for p in win)}


# ---------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------
def make_gpu_case(cfg, ei, torch, noise=True):
    """Synthetic inputs per the recipe (synth); the two model-dependent steps (R16 scaling,
    R20 noise-free curves) use the product path itself."""
    one = ei.Plan(1, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
    sino = torch.zeros(1, 1, cfg.n_angles, cfg.n_det, device="cuda")

    def proj(img):
        ei.ei_project(one, torch.from_numpy(np.ascontiguousarray(img, np.float32)).cuda().view(1, 1, cfg.N, cfg.N),
                      1, sino)
        return sino[0, 0]

    def max_proj(img):
        return float(proj(img).max())

    def max_shift(delta):
        P = proj(delta).double()
        d = torch.empty_like(P)
        d[:, 1:-1] = (P[:, 2:] - P[:, :-2]) / (2 * cfg.det_pitch)
        d[:, 0] = (P[:, 1] - P[:, 0]) / cfg.det_pitch
        d[:, -1] = (P[:, -1] - P[:, -2]) / cfg.det_pitch
        return float((cfg.z * d).abs().max())

    def model(case):
        plan = ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z,
                       cfg.angles)
        out = torch.zeros(cfg.S, cfg.n_angles, cfg.M, cfg.n_det, device="cuda")
        dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        ei.ei_forward(plan, dv(case.mu), dv(case.delta), dv(case.sigma), dv(case.flat), dv(case.mask),
                      None if case.drift is None else dv(case.drift), out)
        torch.cuda.synchronize()
        plan.destroy()
        return out.cpu().numpy()

    case = synth.make_case(cfg, max_shift, max_proj, model, noise=noise)
    one.destroy()
    return case


def step_percentiles(ev):
    """p10 / p50 / p90 of this rank's per-step device times (ms), CUDA events around each step."""
    t = np.sort(np.array([a.elapsed_time(b) for a, b in ev]))
    q = lambda f: float(t[min(len(t) - 1, int(round(f * (len(t) - 1))))])
    return {"p10": round(q(0.1), 5), "p50": round(q(0.5), 5), "p90": round(q(0.9), 5)}


def run_gpu(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2202_08627_b200 import ei

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = edist.rank_config(cfg, rank)            # weak scaling: each rank its own seeded stack
    t_gen = time.time()
    case = make_gpu_case(cfg, ei, torch)
    t_gen = time.time() - t_gen
    maps = synth.perturbed(case.maps(), cfg.seed + 7)          # mid-optimisation iterate (R21)
    lam = args.lam
    plan = ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    mu, delta, sigma = (dv(m) for m in maps)
    flat, mask = dv(case.flat), dv(case.mask)
    drift = None if case.drift is None else dv(case.drift)
    s_exp = dv(case.s_exp)
    ws = ei.Workspace(plan, dev)
    stream = torch.cuda.current_stream()

    def step():
        ei.ei_cost_grad(plan, mu, delta, sigma, flat, mask, drift, s_exp, lam, ws.cost, ws.g[0], ws.g[1],
                        ws.g[2], ws.status, stream)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MiB > 126 MB L2
    for _ in range(max(args.warmup, 3)):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    # keep the GPU at load clocks for the sampler while it starts (untimed)
    sampler = ClockSampler(local_rank) if rank == 0 else None
    t_end = time.time() + 0.5
    while time.time() < t_end:
        step()
        torch.cuda.synchronize()
    ws.status.zero_()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    s0 = ei.ei_plan_stats(plan)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    torch.cuda.nvtx.range_push("timed")                           # ncu --nvtx-include "timed/"
    for i in range(K):
        flush.fill_(1.0)                                          # untimed L2 flush
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    t1 = time.time()
    if world > 1:
        dist.barrier()
    ms = edist.max_over_ranks(sum(a.elapsed_time(b) for a, b in ev))   # slowest rank = the step
    s1 = ei.ei_plan_stats(plan)
    # per-kernel split: the same K steps again with the library's per-kernel CUDA events (events
    # between launches serialise the kernels, i.e. switch off the programmatic-dependent-launch
    # overlap, so this pass is kept out of the step time above)
    ei.ei_plan_set_timing(plan, K)
    for i in range(K):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    kern_ms, n_rec = ei.ei_plan_read_timing(plan)
    ei.ei_plan_set_timing(plan, 0)
    launches = s1[5] - s0[5]
    plan_info = ei.ei_plan_info(plan)
    status = ws.status.cpu().numpy().tolist()
    cost0 = float(ws.cost[0].item())
    # the clock sampler (an nvidia-smi query every few ms) stops before the end-to-end leg: its
    # driver queries and CPU time land on the synchronous host-buffer calls timed below
    if sampler:
        sampler.stop()

    # ---- end-to-end through the host-buffer C-ABI entry point (pinned host memory) ----
    def pinned(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        return t.numpy()
    h_in = [pinned(m) for m in maps] + [pinned(case.flat), pinned(case.mask)]
    h_drift = None if case.drift is None else pinned(case.drift)
    h_sexp = pinned(case.s_exp)
    S, N = cfg.S, cfg.N
    h_cost = pinned(np.zeros(S))
    h_g = [pinned(np.zeros((S, N, N), np.float32)) for _ in range(3)]
    h_st = pinned(np.zeros(4, np.int32))

    def e2e_step():
        ei.ei_cost_grad_host(plan, *h_in, h_drift, h_sexp, lam, h_cost, *h_g, h_st, stream)

    for _ in range(2):
        e2e_step()
    Ke = max(1, min(K, 50))
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(Ke)]
    if world > 1:
        dist.barrier()
    for i in range(Ke):
        flush.fill_(1.0)
        ee[i][0].record(stream)
        e2e_step()
        ee[i][1].record(stream)
    torch.cuda.synchronize()
    # median over the steps (each step is one synchronous host call: CPU scheduling noise on the
    # box shows up as outliers); the mean is reported beside it
    e2e_all = sorted(a.elapsed_time(b) for a, b in ee)
    e2e_ms = edist.max_over_ranks(e2e_all[len(e2e_all) // 2])
    e2e_mean = edist.max_over_ranks(sum(e2e_all) / Ke)
    h2d = 4 * (3 * S * N * N + S * 3 * cfg.n_det + cfg.M + (cfg.n_angles if case.drift is not None else 0)
               + S * cfg.n_angles * cfg.M * cfg.n_det)
    d2h = 8 * S + 4 * 3 * S * N * N + 16
    if rank != 0:
        return None

    clocks = sampler.summary(t0, t1)
    peaks = load_peaks()
    ms_step = ms / K
    step_stats = step_percentiles(ev)
    rsu = ray_sample_updates(cfg)
    kb = kernel_bytes(cfg, rsu, plan_info.get("mirror_pairs", 0))
    sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    kernels, dom = kernel_table(kb, kern_ms, n_rec, ms_step, sm_mhz, peaks.get("hbm_gbs", 6650.0), cfg.name)
    d = kernels[dom]
    roofline = {"kernel": dom, "bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"],
                "unit": "GB/s", "frac": d["frac"], "traffic": load_traffic(cfg.name, dom)[0],
                "traffic_unit": "dram bytes per launch", "traffic_source": load_traffic(cfg.name, dom)[1],
                "peak_source": onchip_peak(sm_mhz)[1] if d["bound"] == "l1" else
                               "measured hbm_gbs (MEASURED_PEAKS.json)"}
    value = world * 1000.0 / ms_step
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "ms_per_step_pct": step_stats,
        "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(cfg, lam),
        "l2": "flushed before every timed step (256 MiB write, untimed)",
        "parallelism": "slice-parallel replicas" if world > 1 else "1 GPU",
        # SURVEY §8(d) counts every angle's samples ("effective"); with mirror pairs (360-degree
        # scans) K1/K3 execute only the primaries' samples ("executed")
        "ray_sample_updates_per_s": round(world * 6 * rsu * cfg.S / (ms_step * 1e-3), 1),
        "ray_sample_updates_per_s_kind": "effective (every angle counted)" if plan_info.get("mirror_pairs", 0)
                                         else "executed (= effective: no mirror pairs)",
        "ray_sample_updates_per_s_executed": round(world * 6 * rsu * cfg.S * (cfg.n_angles - plan_info.get(
            "mirror_pairs", 0)) / cfg.n_angles / (ms_step * 1e-3), 1),
        "slice_evals_per_s": round(world * cfg.S * 1000.0 / ms_step, 3),
        "ray_sample_updates_per_eval": 6 * rsu * cfg.S,
        "roofline": roofline, "kernels": kernels,
        "e2e": {"value": round(world * 1000.0 / e2e_ms, 3), "unit": UNIT, "ms_per_step": round(e2e_ms, 4),
                "ms_mean": round(e2e_mean, 4), "statistic": "median of %d steps" % Ke,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "ei_cost_grad_host (pinned host buffers)"},
        "gpu_launches": int(launches), "launches_per_step": launches / K,
        "clocks": clocks, "status": status, "plan": plan_info, "cost_slice0": cost0, "input_gen_s": round(t_gen, 2),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, case, maps, lam, budget_s=args.cpu_budget)
    return line


def run_gpu_angles(args, cfg, rank, world, local_rank):
    """Strong scaling of ONE stack over its angles: every rank holds the same
    maps, evaluates its angles (mirror pairs kept together, dist.angle_shard) and one NCCL
    all-reduce of the gradient and cost completes the evaluation; the step includes it."""
    import torch
    import torch.distributed as dist
    from paper_2202_08627_b200 import ei

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    case = make_gpu_case(cfg, ei, torch)                  # same seed on every rank: same data
    maps = synth.perturbed(case.maps(), cfg.seed + 7)
    lam = args.lam
    sh = edist.AngleShardEval(ei, cfg, rank, world, dev)
    se, dr = sh.local_inputs(case.s_exp, case.drift)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    dm = [dv(m) for m in maps]
    flat, mask = dv(case.flat), dv(case.mask)
    stream = torch.cuda.current_stream()

    def step():
        sh.cost_grad(dm, flat, mask, dr, se, lam, stream)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for _ in range(max(args.warmup, 3)):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank) if rank == 0 else None
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    s0 = ei.ei_plan_stats(sh.plan)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    for i in range(K):
        flush.fill_(1.0)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    t1 = time.time()
    dist.barrier()
    ms = edist.max_over_ranks(sum(a.elapsed_time(b) for a, b in ev))
    s1 = ei.ei_plan_stats(sh.plan)
    if sampler:
        sampler.stop()
    if rank != 0:
        return None
    ms_step = ms / K
    step_stats = step_percentiles(ev)
    rsu = ray_sample_updates(cfg)
    return {
        "metric": METRIC, "value": round(1000.0 / ms_step, 3), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "ms_per_step_pct": step_stats,
        "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(cfg, lam),
        "parallelism": "angle-sharded x%d, NCCL all-reduce of gradient + cost per evaluation" % world,
        "l2": "flushed before every timed step (256 MiB write, untimed)",
        "ray_sample_updates_per_s": round(6 * rsu * cfg.S / (ms_step * 1e-3), 1),
        "angles_rank0": int(len(sh.idx)), "gpu_launches": int(s1[5] - s0[5]),
        "clocks": sampler.summary(t0, t1), "plan": ei.ei_plan_info(sh.plan),
        "e2e": None,
    }


def bench_config(cfg, lam):
    """The workload identity, the same dict on the GPU arm and the reference arm (both evaluate
    the x_pert point of the same seeded case); how a run was executed (parallelism, L2 policy)
    sits in top-level keys."""
    return {"workload": "%s: %s" % (cfg.name, describe(cfg)), "slices_per_gpu": cfg.S,
            "lambda": lam, "eval_point": "x_pert (R21)"}


def describe(cfg):
    return ("%dx %dx%d grid, %d angles over [0,%g) deg, %d detector px, M=%d" %
            (cfg.S, cfg.N, cfg.N, cfg.n_angles, cfg.span_deg, cfg.n_det, cfg.M))


# ---------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------------------
def cpu_baseline(cfg, case, maps, lam, budget_s=15.0, min_units=1):
    """Time the fp64 oracle (as it stands) on bounded samples: whole evaluations of one slice
    each; returns evals/s of the full workload (S slices per eval)."""
    from oracle import ora
    t0 = time.time()
    n = 0
    while n < min_units or time.time() - t0 < budget_s:
        s = n % cfg.S
        ora.cost_grad(cfg.angles, *maps, case.flat, case.mask, case.drift, case.s_exp, lam,
                      dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z, slices=[s])
        n += 1
        if time.time() - t0 > budget_s:
            break
    dt = time.time() - t0
    slices_per_s = n / dt
    return {"value": round(slices_per_s / cfg.S, 6), "unit": UNIT, "cores": ora.num_threads(),
            "kind": "oracle",
            "sample": "%d single-slice fp64 cost+gradient evaluations of %s (%.1f s); value = "
                      "slices/s / %d slices per eval" % (n, cfg.name, dt, cfg.S)}


def run_reference(args, cfg, rank):
    if rank != 0:
        return None
    from oracle import ora
    ora.build()

    def max_shift(delta):
        P = ora.project(delta, cfg.angles, cfg.n_det, cfg.pixel, cfg.det_pitch)
        return float(max(np.abs(cfg.z * ora.diff_t(r, cfg.det_pitch)).max() for r in P))

    def max_proj(img):
        return float(ora.project(img, cfg.angles, cfg.n_det, cfg.pixel, cfg.det_pitch).max())

    # the oracle times on the same workload shape; s_exp only needs the right shape and value
    # range for timing, so slices beyond the first reuse slice 0's curves
    one = dataclasses.replace(cfg, S=1)
    c1 = synth.make_case(one, max_shift, max_proj,
                         lambda c: ora.forward(cfg.angles, c.mu, c.delta, c.sigma, c.flat, c.mask, c.drift,
                                               dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)[0])
    maps = synth.perturbed(c1.maps(), cfg.seed + 7)
    times = []
    for i in range(args.warmup + args.steps):
        t = time.time()
        ora.cost_grad(cfg.angles, *maps, c1.flat, c1.mask, c1.drift, c1.s_exp, args.lam,
                      dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
        if i >= args.warmup:
            times.append(time.time() - t)
    per_slice = sum(times) / len(times)
    value = 1.0 / (per_slice * cfg.S)
    sample = ("%d timed single-slice fp64 oracle cost+gradient evaluations of %s (one slice = 1/%d "
              "eval)" % (len(times), cfg.name, cfg.S))
    return {"metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(per_slice * 1e3 * cfg.S, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": bench_config(cfg, args.lam), "parallelism": "1 process, oracle threads on host cores",
            "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": ora.num_threads(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ---------------------------------------------------------------------------------------
# the paper's single-map model on the paper's scan geometry (NEXT-3, config P1): a context line
# ---------------------------------------------------------------------------------------
PAPER_CONTEXT = {
    "paper_best_cell_s": 14.5, "paper_best_cell_iterations": 36,
    "paper_s_per_iteration": round(14.5 / 36, 3),
    "paper_hardware": "standard workstation, Intel i5 at 2.10 GHz, single thread (PAPER.md:186, :203)",
    "paper_workload": "220 x 220 slice, 400 projections over 360 deg, one mask position, Numba Radon, "
                      "m_r = 0, 20 flat scans (Table 2, PAPER.md:166-186)",
    "note": "context only: the paper reports time per L-BFGS iteration (>= 1 cost+gradient "
            "evaluation), not evaluations per second",
}


def run_gpu_h(args, cfg):
    import torch
    from paper_2202_08627_b200 import ei
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    t_gen = time.time()
    ang = cfg.angles

    def max_shift(img):   # product path: max |D R[img]| (unit z) from ei_project (no parity claim)
        plan1 = ei.Plan(1, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, 1.0, ang)
        sino = torch.zeros(1, 1, cfg.n_angles, cfg.n_det, device=dev)
        ei.ei_project(plan1, torch.from_numpy(np.ascontiguousarray(img[None, None])).to(dev), 1, sino)
        P = sino[0, 0].double()
        d = torch.cat([P[:, 1:2] - P[:, 0:1], 0.5 * (P[:, 2:] - P[:, :-2]), P[:, -1:] - P[:, -2:-1]], 1)
        return float(d.abs().max() / cfg.det_pitch)

    def model(case):
        c = case.cfg
        plan = ei.Plan(c.S, c.N, c.n_angles, c.n_det, c.M, c.pixel, c.det_pitch, c.z, ang)
        out = torch.zeros(c.S, c.n_angles, c.M, c.n_det, device=dev)
        dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        ei.ei_forward_h(plan, dv(case.h), case.gamma, dv(case.flat), dv(case.mask),
                        None if case.drift is None else dv(case.drift), out)
        return out.cpu().numpy()

    case = synth.make_h_case(cfg, synth.H_GAMMA, max_shift, model)
    cfg = case.cfg
    t_gen = time.time() - t_gen
    h = synth.perturbed((case.h,), cfg.seed + 7)[0]
    lam = synth.H_LAMBDA
    plan = ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, ang)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    hd, flat, mask, s_exp = dv(h), dv(case.flat), dv(case.mask), dv(case.s_exp)
    drift = None if case.drift is None else dv(case.drift)
    cost = torch.zeros(cfg.S, dtype=torch.float64, device=dev)
    g = torch.zeros(cfg.S, cfg.N, cfg.N, device=dev)
    st = torch.zeros(4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        ei.ei_cost_grad_h(plan, hd, case.gamma, flat, mask, drift, s_exp, lam, cost, g, None, st, stream)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for _ in range(max(args.warmup, 3)):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    t_end = time.time() + 0.5
    while time.time() < t_end:
        step()
        torch.cuda.synchronize()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    s0 = ei.ei_plan_stats(plan)
    torch.cuda.synchronize()
    t0 = time.time()
    for i in range(K):
        flush.fill_(1.0)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    t1 = time.time()
    ms_step = sum(a.elapsed_time(b) for a, b in ev) / K
    step_stats = step_percentiles(ev)
    s1 = ei.ei_plan_stats(plan)
    ei.ei_plan_set_timing(plan, K)
    for i in range(K):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    kern_ms, n_rec = ei.ei_plan_read_timing(plan)
    ei.ei_plan_set_timing(plan, 0)
    sampler.stop()
    clocks = sampler.summary(t0, t1)
    rsu = ray_sample_updates(cfg)
    peaks = load_peaks()
    sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    kb = kernel_bytes_h(cfg, rsu, ei.ei_plan_info(plan).get("mirror_pairs", 0))
    kernels, dom = kernel_table(kb, kern_ms, n_rec, ms_step, sm_mhz, peaks.get("hbm_gbs", 6650.0), cfg.name)
    d = kernels[dom]
    traffic, tsrc = load_traffic(cfg.name, dom)
    roofline = {"kernel": dom, "bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"],
                "unit": "GB/s", "frac": d["frac"], "traffic": traffic,
                "traffic_unit": "dram bytes per launch", "traffic_source": tsrc,
                "peak_source": onchip_peak(sm_mhz)[1] if d["bound"] == "l1" else
                               "measured hbm_gbs (MEASURED_PEAKS.json)"}
    line = {
        "metric": "cost+gradient evals/sec (single-map model, eq. 4)", "value": round(1000.0 / ms_step, 3),
        "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "ms_per_step_pct": step_stats,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "%s: %s (paper scan geometry, PAPER.md:89-93), gamma=%g" %
                   (cfg.name, describe(cfg), case.gamma), "lambda": lam, "eval_point": "x_pert (R21)",
                   "mask_position": float(case.mask[0]),
                   "l2": "flushed before every timed step (256 MiB write, untimed)", "parallelism": "1 GPU"},
        "ray_sample_updates_per_s": round(2 * rsu * cfg.S / (ms_step * 1e-3), 1),
        "roofline": roofline, "kernels": kernels,
        "gpu_launches": int(s1[5] - s0[5]), "clocks": clocks, "status": st.cpu().numpy().tolist(),
        "paper_context": PAPER_CONTEXT, "input_gen_s": round(t_gen, 2),
    }
    if not args.no_cpu_baseline:
        from oracle import ora
        t = time.time()
        n = 0
        while n < 1 or time.time() - t < args.cpu_budget:
            ora.cost_grad_h(cfg.angles, h, case.gamma, case.flat, case.mask, case.drift, case.s_exp, lam,
                            dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
            n += 1
        dt = time.time() - t
        line["cpu_baseline"] = {"value": round(n / dt, 4), "unit": UNIT, "cores": ora.num_threads(),
                                "kind": "oracle",
                                "sample": "%d fp64 oracle single-map cost+gradient evaluations of %s "
                                          "(%.1f s)" % (n, cfg.name, dt)}
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=sorted(synth.CONFIGS) + sorted(synth.H_CONFIGS),
                    help="C1-C5: three-map model (BASELINE.json configs); P1: the paper's single-map "
                         "model on its own scan geometry (context line)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lam", type=float, default=1e-2)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="slices", choices=["slices", "angles"],
                    help="N > 1: 'slices' = every rank its own stack (weak scaling, default); "
                         "'angles' = one stack split over angles with an all-reduce (strong)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3                                           # timing rule: W >= 3
    rank, world, local_rank = edist.env_rank()
    if args.config in synth.H_CONFIGS:
        if args.impl == "reference" or world > 1:
            raise SystemExit("P1 (single-map context line) runs on one GPU with --impl ours only")
        print(json.dumps(run_gpu_h(args, synth.H_CONFIGS[args.config])), flush=True)
        return
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        line = run_reference(args, cfg, rank)
    else:
        if world > 1:
            import torch
            torch.cuda.set_device(local_rank)
            edist.init("nccl", torch.device("cuda", local_rank))
        if args.shard == "angles" and world > 1:
            line = run_gpu_angles(args, cfg, rank, world, local_rank)
        else:
            line = run_gpu(args, cfg, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
