"""Diagnose the GPU-vs-SciPy final-cost gap of tests/test_gpu_lbfgs.py::test_lbfgs_matches_scipy_on_oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import _cases  # noqa: E402
from paper_2202_08627_b200 import ei, lbfgs  # noqa: E402
import scipy.optimize as so  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

case = _cases.cached_case("C1")
cfg = case.cfg
lam = 1e10
N = cfg.N
ofg = _cases.oracle_objective(case, lam)


def f_np(v):
    c, g = ofg(torch.from_numpy(v.reshape(3, 1, N, N)))
    return float(c[0]), g.numpy().ravel()


with threadpool_limits(limits=1, user_api="blas"):
    ref = so.minimize(f_np, np.zeros(3 * N * N), jac=True, method="L-BFGS-B",
                      options=dict(maxiter=3000, ftol=1e-13, gtol=1e-12, maxcor=10))
print("scipy", ref.fun, ref.nit)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
plan = ei.Plan(1, N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
fg = lbfgs.ei_objective(plan, d(case.flat), d(case.mask), None, d(case.s_exp), lam)
hist = []
res = lbfgs.minimize(fg, torch.zeros(3, 1, N, N, device="cuda"), max_iter=3000, rel_tol=1e-12,
                     callback=lambda it, f, x: hist.append(float(f[0])))
print("gpu", float(res.cost[0]), res.reason, res.n_iter, res.n_evals, "tail", hist[-5:])
xs = torch.from_numpy(ref.x.reshape(3, 1, N, N).astype(np.float32)).cuda()
cg, gg = fg(xs)
print("gpu cost at scipy x*", float(cg[0]), "grad norm", float(gg.double().norm()))
xg = res.x.double().cpu()
co, go = ofg(xg)
print("oracle cost at gpu x", float(co[0]), "oracle grad norm there", float(go.norm()))
cg2, gg2 = fg(res.x)
print("gpu grad norm at gpu x", float(gg2.double().norm()), "gpu-oracle grad rel diff",
      float((gg2.double().cpu() - go).norm() / go.norm()))
