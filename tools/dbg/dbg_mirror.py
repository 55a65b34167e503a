import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2202_08627_b200 import ei, synth
from oracle import ora
import _cases
case = _cases.cached_case("R3"); cfg = case.cfg
plan = ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
print(ei.ei_plan_info(plan))
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
rel = lambda a, b: float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))
x = synth.uniform((cfg.S, 1, cfg.N, cfg.N), 21)
Rx = torch.zeros(cfg.S, 1, cfg.n_angles, cfg.n_det, device="cuda")
ei.ei_project(plan, dev(x), 1, Rx)
ref = ora.project(x[0, 0].astype(np.float64), cfg.angles, cfg.n_det)
print("proj1 rel", rel(Rx.cpu().numpy()[0, 0], ref))
d = np.abs(Rx.cpu().numpy()[0, 0] - ref).max(axis=1); print("worst rows", np.argsort(d)[-5:], d[np.argsort(d)[-5:]])
y = synth.uniform((cfg.S, 1, cfg.n_angles, cfg.n_det), 22)
Rty = torch.zeros(cfg.S, 1, cfg.N, cfg.N, device="cuda")
ei.ei_backproject(plan, dev(y), 1, Rty)
refb = ora.backproject(y[0, 0].astype(np.float64), cfg.angles, cfg.N)
print("bp1 rel", rel(Rty.cpu().numpy()[0, 0], refb))
g = Rx.cpu().numpy()[0, 0]
for r in (10, 30):
    print("row", r, "angle", np.rad2deg(cfg.angles[r]))
    print(" gpu", np.round(g[r, :12], 3), np.round(g[r, -12:], 3))
    print(" ref", np.round(ref[r, :12], 3), np.round(ref[r, -12:], 3))
S3 = torch.zeros(cfg.S, 3, cfg.n_angles, cfg.n_det, device="cuda")
x3 = np.concatenate([x, x, x], axis=1)
ei.ei_project(plan, dev(x3), 3, S3)
print("proj3 vs proj1 row10 maxdiff", np.abs(S3.cpu().numpy()[0, 0, 10] - g[10]).max(), "proj3 rel", rel(S3.cpu().numpy()[0, 0], ref))
