"""H2D bandwidth from pinned memory with 1, 2 or 4 concurrent copy streams (1 GiB total)."""
import torch

n = 1 << 28   # floats = 1 GiB
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for k in (1, 2, 4, 1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    part = n // k
    for i, s in enumerate(streams):
        s.wait_event(a)
        with torch.cuda.stream(s):
            d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
    for s in streams:
        b.wait_stream(s) if hasattr(b, "wait_stream") else None
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b)
    print("streams %d: %.1f GB/s" % (k, 4 * n / ms / 1e6))
