"""Pinned host buffers vs DMA bandwidth on the GPU box (a KVM guest: copy speed depends on how
the buffer's pages are backed):
    python tools/dbg/hostmem_probe.py
H2D / D2H bandwidth of C2's s_exp size (3.9 MB) and C4's (991 MB) from buffers made by
torch.pin_memory (cudaHostAlloc), by cudaHostRegister of 4-KB-page anonymous memory, and by
cudaHostRegister of 2-MB-aligned memory advised MADV_HUGEPAGE (transparent huge pages)."""
import ctypes
import mmap
import os

import numpy as np
import torch

print("THP enabled:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
print("THP defrag:", open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if cudart is None:
    cudart = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
cudart.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
MADV_HUGEPAGE = 14
HUGE = 2 << 20


def anon(nbytes, huge):
    size = (nbytes + HUGE - 1) // HUGE * HUGE
    raw = libc.mmap(None, size + HUGE, mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
    base = (raw + HUGE - 1) // HUGE * HUGE
    if huge:
        assert libc.madvise(base, size, MADV_HUGEPAGE) == 0
    arr = np.ctypeslib.as_array((ctypes.c_float * (size // 4)).from_address(base))
    arr[:] = 1.0   # first touch
    rc = cudart.cudaHostRegister(base, size, 0)
    assert rc == 0, rc
    return torch.from_numpy(arr[: nbytes // 4])


def bw(h, d, h2d, reps):
    for _ in range(2):
        (d.copy_(h, non_blocking=True) if h2d else h.copy_(d, non_blocking=True))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        (d.copy_(h, non_blocking=True) if h2d else h.copy_(d, non_blocking=True))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return h.numel() * 4 / float(np.median(ts)) / 1e6


for n, reps in ((360 * 7 * 384, 30), (64 * 720 * 7 * 768, 3)):
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for label, make in (("pin_memory", lambda: torch.ones(n).pin_memory()),
                        ("register 4K", lambda: anon(4 * n, False)),
                        ("register THP", lambda: anon(4 * n, True))):
        res = []
        for _ in range(3):
            h = make()
            res.append((bw(h, d, True, reps), bw(h, d, False, reps)))
        print("%9.1f MB %-13s" % (4 * n / 1e6, label), "  ".join("H2D %5.1f D2H %5.1f" % r for r in res))
    del d
