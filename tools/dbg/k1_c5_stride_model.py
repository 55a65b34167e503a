"""Per-angle choice among strided ray partitions of a 64-ray K1 tile for C5 ray-fast quarter warps
(rays base + k rq, k = 1, 2, 4, 8): LDS.128 wavefronts relative to k = 1 (DESIGN.md §9 item 3).
CPU only: python tools/dbg/k1_c5_stride_model.py"""
import numpy as np, math
N, ND, NA = 2048, 3072, 240
ang = np.arange(NA) * math.pi / NA
ctr, dctr = 0.5*(N-1), 0.5*(ND-1)
rows = list(range(0, N, 97))
def ent(th, k, i):
    cs, sn = math.cos(th), math.sin(th)
    rd = abs(cs) >= abs(sn)
    cd, so = (cs, sn) if rd else (sn, cs)
    xs = (k - dctr) / cd - (so / cd) * (i - ctr) + ctr
    return np.floor(xs).astype(np.int64) + 1
def rays(kstride, Q):
    rq = np.arange(8)
    if kstride == 1: return 8*Q + rq
    if kstride == 2: return (Q//2)*16 + Q%2 + 2*rq
    if kstride == 4: return (Q//4)*32 + Q%4 + 4*rq
    if kstride == 8: return Q + 8*rq
def wf128(e):
    u = np.unique(e); return max(1, np.bincount(u % 8, minlength=8).max())
def wf64(e):  # half warp: 16 lanes, 16 bank pairs
    u = np.unique(e); return max(1, np.bincount(u % 16, minlength=16).max())
tot = {1:0, 2:0, 4:0, 8:0, 'best':0}; tot64 = {1:0,'best':0}; n=0
for a in range(0, NA, 2):
    th = ang[a]
    per = {}
    for ks in (1,2,4,8):
        w = 0
        for kt in range(0, ND-64, 512):
            for i in rows:
                for Q in range(8):
                    w += wf128(ent(th, kt + rays(ks, Q), i))
        per[ks] = w
    b = min(per, key=per.get)
    for ks in (1,2,4,8): tot[ks] += per[ks]
    tot['best'] += per[b]
print({k: round(v/tot[1],3) for k,v in tot.items()})
