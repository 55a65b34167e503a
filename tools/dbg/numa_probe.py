"""Host-buffer placement vs copy bandwidth on the GPU box:
    python tools/dbg/numa_probe.py
prints the GPU's NUMA node / local CPUs (sysfs), this process's CPU affinity, and the pinned H2D /
D2H bandwidth of buffers allocated (first-touched) while the process is bound to the GPU-local
CPUs, to the other CPUs, and unbound."""
import os
import subprocess

import numpy as np
import torch


def cpulist(s):
    out = set()
    for part in s.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        else:
            out.add(int(part))
    return out


bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", "0"],
                     capture_output=True, text=True).stdout.strip().lower()
dom, rest = bus.split(":", 1)
sysdir = "/sys/bus/pci/devices/%s:%s" % (dom[-4:], rest)
node = open(os.path.join(sysdir, "numa_node")).read().strip() if os.path.exists(sysdir) else "?"
local = cpulist(open(os.path.join(sysdir, "local_cpulist")).read()) if os.path.exists(sysdir) else set()
aff0 = os.sched_getaffinity(0)
print("gpu", bus, "numa_node", node, "local cpus", len(local), "affinity", len(aff0),
      "affinity & local", len(aff0 & local))
nodes = sorted(d for d in os.listdir("/sys/devices/system/node") if d.startswith("node"))
for d in nodes:
    print(" ", d, "cpus", open("/sys/devices/system/node/%s/cpulist" % d).read().strip())

dev = torch.device("cuda")
n = 360 * 7 * 384   # C2's s_exp
d = torch.empty(n, dtype=torch.float32, device=dev)


def bw(h, h2d=True, reps=30):
    for _ in range(3):
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
    return 4 * n / float(np.median(ts)) / 1e6


def trial(label, cpus):
    if cpus:
        os.sched_setaffinity(0, cpus)
    bufs = []
    for k in range(3):
        h = torch.empty(n, dtype=torch.float32).pin_memory()
        h.fill_(1.0)
        bufs.append(h)
    res = [(bw(h), bw(h, False)) for h in bufs]
    os.sched_setaffinity(0, aff0)
    print("%-14s" % label, "  ".join("H2D %5.1f D2H %5.1f GB/s" % r for r in res))


trial("unbound", None)
if local & aff0:
    trial("gpu-local", local & aff0)
other = aff0 - local
if other:
    trial("other cpus", other)
trial("unbound again", None)
