"""Regenerate DESIGN.md §9's status table from committed bench lines:
    python tools/status_table.py v12 [r02]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "v12"
rnd = sys.argv[2] if len(sys.argv) > 2 else "r02"


def line(c):
    return json.loads(open(os.path.join(ROOT, "profiles", rnd, "bench_%s_%s.json" % (c, tag))).read().splitlines()[-1])


rows = []
for c in ["C1", "C2", "C3", "C4", "C5"]:
    d = line(c)
    k = d["kernels"]
    rows.append("| %s | %.1f µs | %.1f | %.2f T | %.1f | %.2f / %.2f / %.2f | %.3g (%d) |" % (
        c, d["ms_per_step"] * 1000, d["value"], d["ray_sample_updates_per_s"] / 1e12, d["e2e"]["value"],
        k["K1_project"]["frac"], k["K2_curve"]["frac"], k["K3_backproject"]["frac"],
        d["cpu_baseline"]["value"], d["cpu_baseline"]["cores"]))
p1 = line("P1")
k = p1.get("kernels")   # the single-map line has no host-buffer (e2e) leg
fr = "%.2f / %.2f / %.2f" % tuple(k[n]["frac"] for n in ("K1_project", "K2_curve", "K3_backproject")) if k else "—"
rows.append("| P1 (single-map model, paper geometry) | %.1f µs | %.0f | %.2f T | — | %s | %.3g (%d) |" % (
    p1["ms_per_step"] * 1000, p1["value"], p1["ray_sample_updates_per_s"] / 1e12, fr, p1["cpu_baseline"]["value"],
    p1["cpu_baseline"]["cores"]))
print("\n".join(rows))
