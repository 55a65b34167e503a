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


if __name__ == "__main__":
    main()
