"""K3 per-CTA timeline (debug build only, like tools/dbg/k1_trace.py):
    EI_NVCC_DEFS=-DEI_TRACE python -c "from paper_2202_08627_b200 import build; build.build(force=True)"
    python tools/dbg/k3_trace.py C2 [iters]
Prints, for the last ei_cost_grad call, each K3 CTA's start, first-staged-chunk and end times."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08627_b200 import ei, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = synth.CONFIGS[name]
S = cfg.S if name != "C4" else 8
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
info = ei.ei_plan_info(plan)
nt = (cfg.N + 31) // 32
KS = info["k3_angle_split"]
n = nt * nt * S * KS
buf = (ctypes.c_ulonglong * (4 * n))()
fn = ei._lib.ei_debug_k3_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert fn(ctypes.addressof(buf), n) == 0
tr = np.frombuffer(buf, dtype=np.uint64).reshape(n, 4).astype(np.int64)
# n is an upper bound (split grids give only some tiles KS parts): keep the records written
tr = tr[tr[:, 2] > 0]
n = len(tr)
t0 = tr[:, 0].min()
st, da, en = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
sm, nch = tr[:, 3] & 0xffffffff, tr[:, 3] >> 32
print(name, info)
print("CTAs %d span %.2f us; start: min %.2f max %.2f; first data: min %.2f mean %.2f max %.2f; end: min %.2f mean %.2f"
      % (n, en.max(), st.min(), st.max(), da.min(), da.mean(), da.max(), en.min(), en.mean()))
print("work (end - first data): mean %.2f max %.2f min %.2f" % ((en - da).mean(), (en - da).max(), (en - da).min()))
for c in np.unique(nch):
    m = nch == c
    print("chunks %d: n %d  work mean %.2f  end mean %.2f max %.2f" % (c, m.sum(), (en - da)[m].mean(), en[m].mean(), en[m].max()))
cnt = np.bincount(sm)
print("CTAs per SM:", np.bincount(cnt))
late = np.argsort(-en)[:10]
for i in late:
    print("  cta %4d sm %3d start %.2f data %.2f end %.2f nch %d (SM has %d CTAs)" % (i, sm[i], st[i], da[i], en[i], nch[i], cnt[sm[i]]))
