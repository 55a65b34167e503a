"""Per-kernel share of the step from an ncu launch list (`--metrics gpu__time_duration.sum --csv`).
    python tools/launch_share.py gpurun_out/x/launches.csv
Only libei kernels are counted (torch's L2-flush fill kernels are listed separately).  ncu
serialises launches and runs them cold, so absolute times are not bench numbers; the SHARE of
each kernel in the step is what must agree with bench.py's CUDA-event split."""
import csv
import sys
from collections import OrderedDict

OURS = ("pack_pairs_kernel", "check_small_kernel", "backproject3_kernel", "backproject1_kernel",
        "backproject_kernel", "project_kernel", "curve_kernel",
        "pack_sino_kernel", "ks_reduce_kernel", "fold_kernel")   # backproject before project: substring match


def main(path):
    lines = [l for l in open(path) if l.startswith('"')]          # skip ncu's ==PROF== lines
    rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
    per = OrderedDict()
    other = OrderedDict()
    for r in rows:
        name = r["Kernel Name"]
        short = next((k for k in OURS if k in name), None)
        v = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)   # -> us
        d = per if short else other
        key = (short + next((t for t in ("<3>", "<1>", "<0>") if t in name), "")) if short else name[:50]
        d.setdefault(key, []).append(v)
    tot = sum(sum(v) for v in per.values())
    print("libei launches: %d   (other kernels: %d)" % (sum(len(v) for v in per.values()),
                                                       sum(len(v) for v in other.values())))
    print("%-28s %6s %12s %12s %8s" % ("kernel", "count", "mean_us", "total_us", "share"))
    for k, v in per.items():
        print("%-28s %6d %12.2f %12.1f %8.3f" % (k, len(v), sum(v) / len(v), sum(v), sum(v) / tot))
    for k, v in other.items():
        print("  (not ours) %-40s %4d x %.2f us" % (k, len(v), sum(v) / len(v)))


if __name__ == "__main__":
    main(sys.argv[1])
