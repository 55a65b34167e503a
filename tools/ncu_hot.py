"""Hottest SASS instructions of a kernel in an ncu report (needs --import-source / --set full):
    python tools/ncu_hot.py rep.ncu-rep [top] [--ops]
Prints the instructions with the most warp-level executions (and their stall samples), or with
--ops an opcode histogram weighted by executions."""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
ie, ss, src = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
data = [(int(r[ie] or 0), int(r[ss] or 0), r[src].strip(), r[0]) for r in rows[1:] if len(r) > ie]
tot = sum(d[0] for d in data)
print("total warp instructions", tot)
if "--ops" in sys.argv:
    ops = {}
    for n, s, t, a in data:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", t)
        if m:
            k = m.group(2)
            ops[k] = ops.get(k, 0) + n
    for k, v in sorted(ops.items(), key=lambda x: -x[1])[:top]:
        print("%10d %6.3f %s" % (v, v / tot, k))
else:
    for i, (n, s, t, a) in enumerate(data):
        pass
    for n, s, t, a in sorted(data, key=lambda x: -x[0])[:top]:
        print("%10d %6d  %s  %s" % (n, s, a[-5:], t))
