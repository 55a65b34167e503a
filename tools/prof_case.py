"""Profiling driver: run ei_cost_grad on a config (optionally fewer slices) a few times.
    python tools/prof_case.py C4 [S] [iters]
Inputs are drawn by synth (unscaled maps, uniform s_exp): kernel timing depends on geometry,
not on the values.  Used under ncu; not a benchmark."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_08627_b200 import ei, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = synth.CONFIGS[name]
S = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.S
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
sl, _ = synth.draw_slice(cfg, 0)
dev = torch.device("cuda")
maps = [torch.from_numpy(np.ascontiguousarray(np.broadcast_to(m.astype(np.float32) * sc, (S, cfg.N, cfg.N)))).to(dev)
        for m, sc in ((sl.mu, 0.01), (sl.delta, 1e-3), (sl.sigma, 1e-5))]
flat = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(sl.flat, (S, 3, cfg.n_det)))).to(dev)
mask = torch.from_numpy(cfg.mask).to(dev)
s_exp = torch.rand(S, cfg.n_angles, cfg.M, cfg.n_det, device=dev) * 1e4
plan = ei.Plan(S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
ws = ei.Workspace(plan)
for _ in range(iters):
    ei.cost_grad(plan, maps, flat, mask, None, s_exp, 1e-2, ws)
torch.cuda.synchronize()
print(name, S, ei.ei_plan_info(plan), ws.cost[:2].tolist())
