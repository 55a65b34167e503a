"""Where the end-to-end (host buffers) time of one evaluation goes, on the GPU box:
    python tools/dbg/e2e_probe.py [C2]
pinned H2D / D2H copy bandwidth at the call's sizes (one and two copy streams), the device-only
step, and the ei_cost_grad_host call timed by events and by the host clock."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08627_b200 import ei, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = synth.CONFIGS[name]
S, N = cfg.S, cfg.N
dev = torch.device("cuda")
n_in = 3 * S * N * N + S * 3 * cfg.n_det + cfg.M
n_sexp = S * cfg.n_angles * cfg.M * cfg.n_det
n_out = 3 * S * N * N


def time_ms(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for n, label in ((n_sexp, "s_exp"), (n_in + n_sexp, "all inputs")):
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device=dev)
    ms = time_ms(lambda: d.copy_(h, non_blocking=True))
    print("H2D %-10s %8.3f MB  %.4f ms  %.1f GB/s" % (label, 4 * n / 1e6, ms, 4 * n / ms / 1e6))
h = torch.empty(n_out, dtype=torch.float32).pin_memory()
d = torch.empty(n_out, dtype=torch.float32, device=dev)
ms = time_ms(lambda: h.copy_(d, non_blocking=True))
print("D2H grads      %8.3f MB  %.4f ms  %.1f GB/s" % (4 * n_out / 1e6, ms, 4 * n_out / ms / 1e6))
# two streams, half each
n = n_sexp
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def two():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d[: n // 2].copy_(h[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2):
        d[n // 2:].copy_(h[n // 2:], non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


ms = time_ms(two)
print("H2D s_exp on 2 streams  %.4f ms  %.1f GB/s" % (ms, 4 * n / ms / 1e6))

case_maps = [np.random.rand(S, N, N).astype(np.float32) * 1e-3 for _ in range(3)]
sl, _ = synth.draw_slice(cfg, 0)
flat = np.ascontiguousarray(np.broadcast_to(sl.flat, (S, 3, cfg.n_det))).astype(np.float32)
mask = cfg.mask.astype(np.float32)
s_exp = (np.random.rand(S, cfg.n_angles, cfg.M, cfg.n_det) * 1e4).astype(np.float32)


def pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()


plan = ei.Plan(S, N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)
h_in = [pinned(m) for m in case_maps] + [pinned(flat), pinned(mask)]
h_sexp = pinned(s_exp)
h_cost = pinned(np.zeros(S))
h_g = [pinned(np.zeros((S, N, N), np.float32)) for _ in range(3)]
h_st = pinned(np.zeros(4, np.int32))
stream = torch.cuda.current_stream()


def e2e():
    ei.ei_cost_grad_host(plan, *h_in, None, h_sexp, 1e-2, h_cost, *h_g, h_st, stream)


ms = time_ms(e2e)
t = []
for _ in range(50):
    t0 = time.perf_counter()
    e2e()
    t.append((time.perf_counter() - t0) * 1e3)
print("ei_cost_grad_host: events %.4f ms, host clock median %.4f ms (min %.4f)" % (ms, np.median(t), min(t)))
ws = ei.Workspace(plan)
maps_d = [torch.from_numpy(m).to(dev) for m in case_maps]
fl_d, mk_d, se_d = (torch.from_numpy(x).to(dev) for x in (flat, mask, s_exp))
ms = time_ms(lambda: ei.cost_grad(plan, maps_d, fl_d, mk_d, None, se_d, 1e-2, ws))
print("device-only ei_cost_grad %.4f ms" % ms)
