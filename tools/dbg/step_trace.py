"""Timeline of one evaluation (debug build only): earliest CTA start / latest CTA end of every
kernel of ei_cost_grad, with programmatic dependent launch active as in bench.py.
    EI_NVCC_DEFS=-DEI_TRACE python -c "from paper_2202_08627_b200 import build; build.build(force=True)"
    python tools/dbg/step_trace.py C2 [reps]
Times are %globaltimer (ns) relative to K0's first CTA; the per-CTA trace records add a barrier
per CTA, so this shows the shape of the step, not bench numbers."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08627_b200 import ei, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = synth.CONFIGS[name] if name in synth.CONFIGS else synth.H_CONFIGS[name]
hmodel = name in synth.H_CONFIGS
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
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
spans = {k: getattr(ei._lib, "ei_debug_span_" + k) for k in ("pack", "proj", "curve", "bp")}
for f in spans.values():
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
rows = []
for r in range(reps + 2):
    flush.fill_(1.0)
    torch.cuda.synchronize()
    for f in spans.values():
        assert f(None, 1) == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if hmodel:   # the paper's single-map model (NEXT-3)
        ei.ei_cost_grad_h(plan, maps[0], synth.H_GAMMA, flat, mask, None, s_exp, 1e-2, ws.cost, ws.g[0], None,
                          ws.status)
    else:
        ei.cost_grad(plan, maps, flat, mask, None, s_exp, 1e-2, ws)
    e1.record()
    torch.cuda.synchronize()
    got = {}
    for k, f in spans.items():
        buf = (ctypes.c_ulonglong * 8)()
        assert f(ctypes.addressof(buf), 0) == 0
        got[k] = np.frombuffer(buf, dtype=np.uint64).astype(np.float64).reshape(4, 2)
    if r >= 2:
        rows.append((e0.elapsed_time(e1) * 1e3, got))
t_ev = np.median([x[0] for x in rows])
print(name, ei.ei_plan_info(plan), "event-timed step %.1f us (median of %d)" % (t_ev, len(rows)))
names = [("K0 pack", "pack", 0), ("K1 project", "proj", 0), ("K2 curve", "curve", 0),
         ("K3 backproject", "bp", 0), ("ks_reduce", "bp", 1)]   # a mirror fold runs between K2 and K3
acc = {n: [] for n, _, _ in names}
for _, got in rows:
    t0 = got["pack"][0, 0]
    for n, k, i in names:
        a, b = got[k][i]
        if b > 0:
            acc[n].append(((a - t0) / 1e3, (b - t0) / 1e3))
for n, _, _ in names:
    if acc[n]:
        v = np.median(np.array(acc[n]), axis=0)
        print("  %-15s start %7.2f us  end %7.2f us  span %6.2f us" % (n, v[0], v[1], v[1] - v[0]))
