"""Time-to-solution of the full iterative reconstruction (NEXT-1): host L-BFGS over ei_cost_grad.

    python tools/reconstruct.py [--config C1] [--noise 0|1] [--iters 300] [--lam 1e-2]

Inputs are generated with the product path (bench.make_gpu_case); prints one JSON line with the
iterations, evaluations, wall time, final cost and the relative L2 error of each recovered map."""
import argparse
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--noise", type=int, default=1)
    ap.add_argument("--iters", type=int, default=300)
    ap.add_argument("--lam", type=float, default=1e-2)
    args = ap.parse_args()
    if args.config in synth.H_CONFIGS:
        return main_h(args)
    cfg = synth.CONFIGS[args.config]
    case = bench.make_gpu_case(cfg, ei, torch, noise=bool(args.noise))
    dev = torch.device("cuda")
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    plan = ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
    fg = lbfgs.ei_objective(plan, d(case.flat), d(case.mask), None if case.drift is None else d(case.drift),
                            d(case.s_exp), args.lam)
    x0 = torch.zeros(3, cfg.S, cfg.N, cfg.N, device=dev)
    torch.cuda.synchronize()
    t0 = time.time()
    res = lbfgs.minimize(fg, x0, max_iter=args.iters, rel_tol=1e-10)
    torch.cuda.synchronize()
    wall = time.time() - t0
    truth = np.stack(case.maps())
    got = res.x.cpu().numpy()
    err = {q: float(np.linalg.norm(got[i] - truth[i]) / np.linalg.norm(truth[i]))
           for i, q in enumerate(("mu", "delta", "sigma"))}
    print(json.dumps({"config": cfg.name, "noise": bool(args.noise), "lambda": args.lam,
                      "iterations": res.n_iter, "evals": res.n_evals, "seconds": round(wall, 3),
                      "ms_per_eval": round(1e3 * wall / res.n_evals, 4),
                      "cost0": float(res.history[0][0]), "cost": float(res.cost[0]),
                      "converged": bool(res.converged.all()), "rel_err": err}))


def main_h(args):
    """The paper's single-map model on its own scan geometry (P1, gamma = 5,
    lambda = 1e-2, start h = 0): the time-to-solution comparable in kind to the paper's Table 2
    (36 L-BFGS iterations in 14.5 s on one i5 core for the best cell)."""
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
    fg(x0)
    torch.cuda.synchronize()
    t0 = time.time()
    res = lbfgs.minimize(fg, x0, max_iter=args.iters, rel_tol=1e-10)
    torch.cuda.synchronize()
    wall = time.time() - t0
    got = res.x.cpu().numpy()[0]
    err = float(np.linalg.norm(got - case.h) / np.linalg.norm(case.h))
    print(json.dumps({"config": cfg.name, "model": "single-map h (eq. 4)", "noise": bool(args.noise),
                      "gamma": case.gamma, "lambda": args.lam, "iterations": res.n_iter,
                      "evals": res.n_evals, "seconds": round(wall, 4),
                      "ms_per_eval": round(1e3 * wall / res.n_evals, 4),
                      "cost0": float(res.history[0][0]), "cost": float(res.cost[0]),
                      "converged": bool(res.converged.all()), "rel_err_h": err,
                      "paper_context": "best Table 2 cell: 36 iterations, 14.5 s, i5 2.1 GHz single thread "
                                       "(PAPER.md:175-186)"}))


if __name__ == "__main__":
    main()
