"""Stall reasons per SASS opcode from an ncu source page (python tools/ncu_ops.py rep.ncu-rep [ops...])."""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
h, data = rows[0], rows[1:]
ix = {k: i for i, k in enumerate(h)}
S = ix["Warp Stall Sampling (All Samples)"]
st = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
per = collections.defaultdict(collections.Counter)
tot = 0
for r in data:
    src = r[ix["Source"]].strip()
    if not src:
        continue
    t = src.split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    n = int(r[S] or 0)
    tot += n
    per[op]["_samples"] += n
    for k in st:
        per[op][k] += int(r[ix[k]] or 0)
ops = sys.argv[2:] or [k for k, _ in sorted(per.items(), key=lambda x: -x[1]["_samples"])[:8]]
for op in ops:
    c = per[op]
    n = c["_samples"]
    top = ", ".join(f"{k[6:]} {v / max(n, 1) * 100:.0f}%" for k, v in c.most_common(7) if k != "_samples")
    print(f"{op:10s} {n / tot * 100:5.1f}% of samples: {top}")
