"""Bank-conflict model of K1 ray-fast quarter warps on C5 (DESIGN.md §9 item 3): wavefronts per
sample of the A-plane LDS.128 (quarter warp, entry mod 8) and B-plane LDS.64 (half warp, entry mod
16) when a quarter warp takes 8, 7 or 6 adjacent rays of one angle.  CPU only: python tools/dbg/k1_c5_quarter_model.py"""
import numpy as np, math
N, ND, NA = 2048, 3072, 240
ang = np.arange(NA) * math.pi / NA
ctr, dctr = 0.5*(N-1), 0.5*(ND-1)
rows = [0, N//4, N//2, 3*N//4, N-1] + list(range(100, N, 173))
def ent(th, k, i):
    cs, sn = math.cos(th), math.sin(th)
    rd = abs(cs) >= abs(sn)
    cd, so = (cs, sn) if rd else (sn, cs)
    xs = (k - dctr) / cd - (so / cd) * (i - ctr) + ctr
    return np.floor(xs).astype(np.int64) + 1
def cost(e, lanes, banks):
    tot = 0
    for q0 in range(0, len(e), lanes):
        q = e[q0:q0+lanes]; q = q[q >= -10**9]
        if len(q) == 0: continue
        u = np.unique(q)
        tot += max(1, np.bincount(u % banks, minlength=banks).max())
    return tot
def run(rpq, label, stride=1):
    # quarter = rpq rays of one angle; pad to 8 lanes with invalid (-inf) entries
    wfA = wfB = samples = 0
    for a in range(0, NA, 3):
        th = ang[a]
        for kt in range(0, ND - 64, 256):
            for w in range(8):
                for i in rows:
                    # warp = 4 quarters, angles th + j*dth (j=0..3)
                    eA = []
                    for aq in range(4):
                        t2 = ang[min(a + aq, NA-1)]
                        ks = kt + w * rpq + np.arange(rpq)
                        e = ent(t2, ks, i)
                        lane = np.full(8, -2**62); lane[:rpq] = e
                        eA.append(lane)
                    eA = np.concatenate(eA)
                    wfA += cost(eA, 8, 8); wfB += cost(eA, 16, 16); samples += 4 * rpq
    print("%s: LDS128 %.3f LDS64 %.3f wavefronts/sample (x32: %.2f)" % (label, wfA/samples, wfB/samples, 32*(wfA+wfB)/samples))
run(8, "8 rays/quarter")
run(7, "7 rays/quarter")
run(6, "6 rays/quarter")
