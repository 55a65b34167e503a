"""K1 per-CTA timeline (debug build only): which CTAs define the kernel's duration.

    EI_NVCC_DEFS=-DEI_TRACE python -c "from paper_2202_08627_b200 import build; build.build(force=True)"
    python tools/dbg/k1_trace.py C2 [iters]

Runs ei_cost_grad on a config, reads the {start, end, SM, rows} record every K1 CTA of the last
call wrote (%globaltimer), and prints the span, the per-CTA duration spread, per-SM busy time and
the durations by ray tile / row split.  Not a benchmark (the trace adds a barrier per CTA).
"""
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
ngr = info["k1_groups"]
RS = info["k1_row_split"]
cap = 65536
buf = (ctypes.c_ulonglong * (4 * cap))()
fn = ei._lib.ei_debug_k1_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert fn(ctypes.addressof(buf), cap) == 0
tr = np.frombuffer(buf, dtype=np.uint64).reshape(cap, 4).astype(np.int64)
n = ngr * S * RS * ((cfg.n_det + 31) // 32)          # 32-ray tiles: the most CTAs a plan can have
tr = tr[:n]
t_last = tr[:, 1].max()
tr = tr[(tr[:, 1] > t_last - 10**9) & (tr[:, 0] > 0)]  # records of the last call only
n = len(tr)
ntile = n // (ngr * S * RS)
print("ray tile: %d rays (%d tiles)" % ((cfg.n_det + ntile - 1) // ntile, ntile))
t0 = tr[:, 0].min()
st, en, sm = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, tr[:, 2]
rows, un = tr[:, 3] & 0xffffffff, tr[:, 3] >> 32
dur = en - st
print(name, info)
print("CTAs %d  span %.2f us  start spread %.2f us  dur mean %.2f max %.2f min %.2f" %
      (n, en.max(), st.max(), dur.mean(), dur.max(), dur.min()))
busy = np.zeros(sm.max() + 1)
for i in range(n):
    busy[sm[i]] += dur[i]
print("per-SM CTA-time: mean %.2f max %.2f (2 CTAs/SM co-resident)" % (busy.mean(), busy.max()))
print("last end per SM: mean %.2f  min %.2f  max %.2f" %
      tuple(f(np.array([en[sm == q].max() for q in np.unique(sm)])) for f in (np.mean, np.min, np.max)))
tile = un % ntile
grp = (un // ntile) % ngr
rs = un // (ntile * ngr) // S
for t in range(ntile):
    m = tile == t
    print("tile %2d: dur mean %.2f max %.2f  rows mean %.1f" % (t, dur[m].mean(), dur[m].max(), rows[m].mean()))
for r in range(RS):
    m = rs == r
    print("rs %d: dur mean %.2f max %.2f" % (r, dur[m].mean(), dur[m].max()))
order = np.argsort(-dur)[:12]
print("slowest CTAs (block tile grp rs sm start dur rows):")
for i in order:
    print("  %5d %3d %3d %2d %4d %7.2f %7.2f %4d" % (i, tile[i], grp[i], rs[i], sm[i], st[i], dur[i], rows[i]))
# completion time of each angle group (all its units, every tile and row split): when a
# dataflow successor (K2 rows, K3 angle chunks) could start on that group's angles
gend = np.array([en[grp == g].max() for g in range(ngr)])
print("group completion (us): min %.2f  p25 %.2f  median %.2f  p75 %.2f  max %.2f" %
      tuple(np.percentile(gend, q) for q in (0, 25, 50, 75, 100)))
print("  sorted:", " ".join("%.1f" % v for v in np.sort(gend)))
np.save("gpurun_out/k1_trace_%s.npy" % name, tr)
