"""Small end-to-end exercise of every libei entry point for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize_case.py [R1|R3|C1]
Inputs from synth (no oracle: sanitizer runs check memory/race/sync behaviour, not values)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_08627_b200 import ei, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "R1"
cfg = synth.CONFIGS[name] if name in synth.CONFIGS else synth.small_config(
    name, **({} if name == "R1" else dict(S=2, N=48, n_angles=40, span_deg=360.0, n_det=70, M=3, K=5,
                                          drift_sd=0.002, w_jit=0.1, texture=0.05, seed=95)))
dev = torch.device("cuda")
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
S, N, NA, ND, M = cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M
sl, _ = synth.draw_slice(cfg, 0)
maps = [d(np.broadcast_to(m.astype(np.float32) * sc, (S, N, N))) for m, sc in ((sl.mu, 0.01), (sl.delta, 1e-3), (sl.sigma, 1e-5))]
flat = d(np.broadcast_to(sl.flat, (S, 3, ND)))
mask = d(cfg.mask)
drift = d(np.linspace(-0.01, 0.01, NA).astype(np.float32))
s_exp = torch.rand(S, NA, M, ND, device=dev) * 1e4
plan = ei.Plan(S, N, NA, ND, M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
ws = ei.Workspace(plan)
ei.cost_grad(plan, maps, flat, mask, drift, s_exp, 1e-2, ws)
ei.cost_grad(plan, maps, flat, mask, drift, s_exp, 1e-2, ws, want_drift=True)
smod = torch.zeros(S, NA, M, ND, device=dev)
ei.ei_forward(plan, *maps, flat, mask, drift, smod)
sino = torch.zeros(S, 3, NA, ND, device=dev)
ei.ei_project(plan, torch.stack(maps, 1).contiguous(), 3, sino)
back = torch.zeros(S, 3, N, N, device=dev)
ei.ei_backproject(plan, sino, 3, back)
one = torch.zeros(S, 1, NA, ND, device=dev)
ei.ei_project(plan, maps[0][:, None].contiguous(), 1, one)
b1 = torch.zeros(S, 1, N, N, device=dev)
ei.ei_backproject(plan, one, 1, b1)
cost = torch.zeros(S, dtype=torch.float64, device=dev)
g = torch.zeros(S, N, N, device=dev)
gd = torch.zeros(S, NA, device=dev)
st = torch.zeros(4, dtype=torch.int32, device=dev)
ei.ei_cost_grad_h(plan, maps[0], 5.0, flat, mask, drift, s_exp, 1e-2, cost, g, gd, st)
ei.ei_forward_h(plan, maps[0], 5.0, flat, mask, drift, smod)
fs = d(synth.sampled_flat(np.ascontiguousarray(np.broadcast_to(sl.flat, (S, 3, ND))), 33, noise=False))
ei.ei_cost_grad_hs(plan, maps[0], 5.0, fs, mask, drift, s_exp, 1e-2, cost, g, gd, st)
ei.ei_forward_hs(plan, maps[0], 5.0, fs, mask, drift, smod)
h_in = [m.cpu().numpy() for m in maps]
hc = np.zeros(S)
hg = [np.zeros((S, N, N), np.float32) for _ in range(3)]
hs = np.zeros(4, np.int32)
for _ in range(2):
    ei.ei_cost_grad_host(plan, *h_in, flat.cpu().numpy(), cfg.mask, drift.cpu().numpy(), s_exp.cpu().numpy(),
                         1e-2, hc, *hg, hs)
torch.cuda.synchronize()
print("ok", name, ei.ei_plan_info(plan))
