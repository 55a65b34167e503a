"""Where the host L-BFGS loop's time goes (NEXT-1; not the hot path): C1 noise-free, N iterations
under torch.profiler; prints ms per iteration with and without the profiler and the top ops.
    python tools/dbg/prof_lbfgs.py [iters]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2202_08627_b200 import ei, lbfgs, synth  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
cfg = synth.CONFIGS["C1"]
case = bench.make_gpu_case(cfg, ei, torch, noise=False)
dev = torch.device("cuda")
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
plan = ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
fg = lbfgs.ei_objective(plan, d(case.flat), d(case.mask), None if case.drift is None else d(case.drift),
                        d(case.s_exp), 0.0)
x0 = torch.zeros(3, cfg.S, cfg.N, cfg.N, device=dev)
fg(x0)
torch.cuda.synchronize()
t0 = time.time()
res = lbfgs.minimize(fg, x0, max_iter=iters, rel_tol=0.0)
torch.cuda.synchronize()
t = time.time() - t0
print("plain: %d iterations, %d evals, %.3f ms/iteration, %.3f ms/eval" % (res.n_iter, res.n_evals, 1e3 * t / res.n_iter,
                                                                       1e3 * t / res.n_evals))
ncalls = {"n": 0, "t": 0.0}
fg0 = fg


def fg_timed(x):
    torch.cuda.synchronize()
    a = time.time()
    r = fg0(x)
    torch.cuda.synchronize()
    ncalls["n"] += 1
    ncalls["t"] += time.time() - a
    return r


t0 = time.time()
res = lbfgs.minimize(fg_timed, x0, max_iter=iters, rel_tol=0.0)
torch.cuda.synchronize()
t = time.time() - t0
print("evaluation share: %.3f ms per eval (synchronised), %.1f %% of the loop" % (1e3 * ncalls["t"] / ncalls["n"],
                                                                                100 * ncalls["t"] / t))
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    lbfgs.minimize(fg, x0, max_iter=min(iters, 30), rel_tol=0.0)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=25))
