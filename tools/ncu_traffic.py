"""Record per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the libei
kernels from one `ncu --set full` capture into profiles/traffic.json, keyed by bench config:
    python tools/ncu_traffic.py gpurun_out/x/full_c2.ncu-rep C2 "<ncu command>"
bench.py fills roofline.traffic from that file for its config and dominant kernel (null if
absent).  ncu's default cache control flushes caches before each replayed kernel, so this is
the cold-cache HBM traffic of one launch."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = (("backproject3_kernel", "K3_backproject"), ("backproject_kernel<3", "K3_backproject"),
         ("project_kernel<3", "K1_project"),
         ("curve_kernel<1>", "K2_curve"), ("pack_pairs_kernel<3>", "K0_pack"))   # K1/K3 have 2 template args
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, cfg, cmd):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    got = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        key = next((k for pat, k in NAMES if pat in name), None)   # backproject listed first
        if key is None or key in got:
            continue
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[h.index(m)]) * SCALE[units[h.index(m)]]
        def metric(m):
            return float(r[h.index(m)]) * SCALE[units[h.index(m)]] if m in h and r[h.index(m)] else None
        got[key] = {"dram_bytes_per_launch": b,
                    "lts_bytes_per_launch": metric("lts__t_bytes.sum"),
                    "l1tex_bytes_per_launch": metric("l1tex__t_bytes.sum"),
                    "duration_us_cold": float(r[h.index("gpu__time_duration.sum")]) *
                    (1e-3 if units[h.index("gpu__time_duration.sum")] == "ns" else
                     1e3 if units[h.index("gpu__time_duration.sum")] == "ms" else 1.0)}
    path = os.path.join(ROOT, "profiles", "traffic.json")
    db = json.load(open(path)) if os.path.exists(path) else {}
    db[cfg] = {"source": os.path.relpath(rep, ROOT), "command": cmd, "kernels": got}
    json.dump(db, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(db[cfg], indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
