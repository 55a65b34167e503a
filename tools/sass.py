"""Print the SASS of one kernel from an object/.so:  python tools/sass.py <file> <name-substring> [--hist]"""
import re
import subprocess
import sys

path, pat = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", txt)
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    if pat in name:
        lines = [l for l in f.split("\n") if re.match(r"\s*/\*[0-9a-f]{4}\*/", l)]
        if "--hist" in sys.argv:
            ops = {}
            for l in lines:
                m = re.match(r"\s*/\*[0-9a-f]{4}\*/\s*(@!?U?P\w+\s+)?([A-Z0-9_.]+)", l)
                if m:
                    ops[m.group(2)] = ops.get(m.group(2), 0) + 1
            for k, v in sorted(ops.items(), key=lambda x: -x[1]):
                print("%5d %s" % (v, k))
        else:
            print(name)
            print("\n".join(lines))
        break
