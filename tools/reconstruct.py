"""Time-to-solution of the full iterative reconstruction (NEXT-1): host L-BFGS (strong Wolfe) over
the C ABI, from x0 = 0 (BASELINE.json configs: "the start estimate is all-zero maps").

    python tools/reconstruct.py [--config C1] [--noise 0|1] [--iters 5000] [--lam 0]
                                [--stop rel_tol|discrepancy] [--drift-slices S] [--every 10]

  * three-map model (C1, C2, ...): `lbfgs.ei_objective` over ei_cost_grad;
  * --stop discrepancy: stop at cost <= sum of the measured counts (Poisson data; Morozov);
  * --drift-slices S: joint estimation of the maps and the mask drift m_o(theta) of the first S
    slices of the config (C4: drift random walk) as one problem (`lbfgs.ei_objective_drift`);
  * P1: the paper's single-map model on its own scan geometry (context for Table 2).
Inputs are generated with the product path (bench.make_gpu_case; no parity claim rests on them).
Prints one JSON line: iterations, evaluations, wall time, final cost, stop reason, the RMS error of
each map as a fraction of its dynamic range (2-pixel border excluded) and its
relative L2 error, the drift error (RMS up to a constant) and the error trajectory."""
import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2202_08627_b200 import ei, lbfgs, synth  # noqa: E402


def rms_of_range(x, t, b=2):
    d = (np.asarray(x, np.float64) - t)[..., b:-b, b:-b]
    return float(np.sqrt((d ** 2).mean()) / (t.max() - t.min()))


def drift_rms(est, truth):
    d = np.asarray(est, np.float64) - truth
    d = d - d.mean()
    t = truth - truth.mean()
    return float(np.sqrt((d ** 2).mean()) / np.sqrt((t ** 2).mean()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--noise", type=int, default=1)
    ap.add_argument("--iters", type=int, default=5000)
    ap.add_argument("--lam", type=float, default=0.0)
    ap.add_argument("--stop", default="rel_tol", choices=["rel_tol", "discrepancy"])
    ap.add_argument("--rel-tol", type=float, default=1e-9)
    ap.add_argument("--drift-slices", type=int, default=0)
    ap.add_argument("--every", type=int, default=10)
    args = ap.parse_args()
    if args.config in synth.H_CONFIGS:
        return main_h(args)
    cfg = synth.CONFIGS[args.config]
    if args.drift_slices:
        cfg = dataclasses.replace(cfg, S=args.drift_slices)
    case = bench.make_gpu_case(cfg, ei, torch, noise=bool(args.noise))
    dev = torch.device("cuda")
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    plan = ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
    truth = [m.astype(np.float64) for m in case.maps()]
    traj = []
    target = None
    if args.stop == "discrepancy":
        target = case.s_exp.astype(np.float64).reshape(cfg.S, -1).sum(1)
    if args.drift_slices:
        # one stacked tensor (maps + zero-padded drift block): the optimizer's one-kernel vector path
        fg, x0, split = lbfgs.ei_objective_drift_stacked(plan, d(case.flat), d(case.mask), d(case.s_exp), args.lam)
        if target is not None:
            target = target.sum()

        def errs(x):
            parts = split(x)
            e = {q: rms_of_range(parts[i].cpu().numpy(), truth[i]) for i, q in enumerate(("mu", "delta", "sigma"))}
            e["drift"] = drift_rms(parts[3].cpu().numpy(), case.drift.astype(np.float64))
            return e
    else:
        fg = lbfgs.ei_objective(plan, d(case.flat), d(case.mask), None if case.drift is None else d(case.drift),
                                d(case.s_exp), args.lam)
        x0 = torch.zeros(3, cfg.S, cfg.N, cfg.N, device=dev)

        def errs(x):
            xx = x.cpu().numpy()
            return {q: rms_of_range(xx[i], truth[i]) for i, q in enumerate(("mu", "delta", "sigma"))}

    def cb(it, f, x):
        if it % args.every == 0:
            traj.append({"iter": it, "cost": float(f.sum()), **errs(x)})
    fg(x0)
    torch.cuda.synchronize()
    t0 = time.time()
    res = lbfgs.minimize(fg, x0, max_iter=args.iters, rel_tol=args.rel_tol, target=target, callback=cb)
    torch.cuda.synchronize()
    wall = time.time() - t0      # includes the trajectory's error evaluations (every --every its)
    e = errs(res.x)
    rel = None
    if not args.drift_slices:
        xx = res.x.cpu().numpy()
        rel = {q: float(np.linalg.norm(xx[i] - truth[i]) / np.linalg.norm(truth[i]))
               for i, q in enumerate(("mu", "delta", "sigma"))}
    print(json.dumps({"config": cfg.name, "slices": cfg.S, "noise": bool(args.noise), "lambda": args.lam,
                      "stop": args.stop, "joint_drift": bool(args.drift_slices),
                      "iterations": res.n_iter, "evals": res.n_evals, "seconds": round(wall, 3),
                      "ms_per_iteration": round(1e3 * wall / max(res.n_iter, 1), 3),
                      "cost0": float(res.history[0].sum()), "cost": float(res.cost.sum()),
                      "target": None if target is None else float(np.sum(target)),
                      "converged": bool(res.converged.all()), "reason": res.reason,
                      "rms_of_range_2px_border": e, "rel_l2": rel, "trajectory": traj,
                      "optimizer": "L-BFGS, history 10, strong Wolfe (c1 1e-4, c2 0.9)"}))


def main_h(args):
    """The paper's single-map model on its own scan geometry (P1, gamma = 5,
    start h = 0): the time-to-solution comparable in kind to the paper's Table 2 (36 L-BFGS
    iterations in 14.5 s on one i5 core for the best cell)."""
    cfg = synth.H_CONFIGS[args.config]
    dev = torch.device("cuda")
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ang = cfg.angles

    def max_shift(img):
        plan1 = ei.Plan(1, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, 1.0, ang)
        sino = torch.zeros(1, 1, cfg.n_angles, cfg.n_det, device=dev)
        ei.ei_project(plan1, d(img[None, None]), 1, sino)
        P = sino[0, 0].double()
        dd = torch.cat([P[:, 1:2] - P[:, 0:1], 0.5 * (P[:, 2:] - P[:, :-2]), P[:, -1:] - P[:, -2:-1]], 1)
        return float(dd.abs().max() / cfg.det_pitch)

    def model(case):
        c = case.cfg
        plan = ei.Plan(c.S, c.N, c.n_angles, c.n_det, c.M, c.pixel, c.det_pitch, c.z, ang)
        out = torch.zeros(c.S, c.n_angles, c.M, c.n_det, device=dev)
        ei.ei_forward_h(plan, d(case.h), case.gamma, d(case.flat), d(case.mask),
                        None if case.drift is None else d(case.drift), out)
        return out.cpu().numpy()

    case = synth.make_h_case(cfg, synth.H_GAMMA, max_shift, model, noise=bool(args.noise))
    cfg = case.cfg
    plan = ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, ang)
    fg = lbfgs.ei_objective_h(plan, case.gamma, d(case.flat), d(case.mask),
                              None if case.drift is None else d(case.drift), d(case.s_exp), args.lam)
    x0 = torch.zeros(1, cfg.S, cfg.N, cfg.N, device=dev)
    target = case.s_exp.astype(np.float64).sum() if args.stop == "discrepancy" else None
    fg(x0)
    torch.cuda.synchronize()
    t0 = time.time()
    res = lbfgs.minimize(fg, x0, max_iter=args.iters, rel_tol=args.rel_tol, target=target)
    torch.cuda.synchronize()
    wall = time.time() - t0
    got = res.x.cpu().numpy()[0]
    h = case.h.astype(np.float64)
    print(json.dumps({"config": cfg.name, "model": "single-map h (eq. 4)", "noise": bool(args.noise),
                      "gamma": case.gamma, "lambda": args.lam, "stop": args.stop, "iterations": res.n_iter,
                      "evals": res.n_evals, "seconds": round(wall, 4),
                      "ms_per_iteration": round(1e3 * wall / max(res.n_iter, 1), 3),
                      "cost0": float(res.history[0][0]), "cost": float(res.cost[0]),
                      "converged": bool(res.converged.all()), "reason": res.reason,
                      "rms_of_range_2px_border": rms_of_range(got, h),
                      "rel_err_h": float(np.linalg.norm(got - h) / np.linalg.norm(h)),
                      "paper_context": "best Table 2 cell: 36 iterations, 14.5 s, i5 2.1 GHz single thread "
                                       "(PAPER.md:175-186)"}))


if __name__ == "__main__":
    main()
