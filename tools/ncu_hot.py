"""Summarise an ncu report's source page: hottest SASS lines by warp-stall samples,
and shared-memory bank-conflict lines. Usage: python tools/ncu_hot.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
data = rows[1:]
S = ix["Warp Stall Sampling (All Samples)"]
tot = sum(int(r[S] or 0) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -int(r[S] or 0))[:n]:
    print(f"{int(r[S]) / tot * 100:5.1f}%  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:90]}")
if "L1 Conflicts Shared N-Way" in ix:
    C = ix["L1 Wavefronts Shared Excessive"]
    bad = sorted(data, key=lambda r: -int(r[C] or 0))[:8]
    print("-- shared excessive wavefronts")
    for r in bad:
        if int(r[C] or 0):
            print(r[C], r[ix['Address']][-5:], r[ix['Source']].strip()[:90])

# ---- optional region breakdown: python tools/ncu_hot.py rep N start_hex end_hex (address suffixes)
if len(sys.argv) > 4:
    a0, a1 = int(sys.argv[3], 16), int(sys.argv[4], 16)
    st_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    agg = {k: 0 for k in st_cols}
    n_ins = 0
    samp = 0
    for r in data:
        ad = int(r[ix["Address"]], 16) & 0xFFFFF
        if a0 <= ad <= a1:
            n_ins += 1
            samp += int(r[S] or 0)
            for k in st_cols:
                agg[k] += int(r[ix[k]] or 0)
    print(f"-- region {sys.argv[3]}..{sys.argv[4]}: {n_ins} instrs, {samp} samples ({samp / tot * 100:.1f}%)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
        print(f"   {k:24} {v:7d} {v / max(samp, 1) * 100:5.1f}%")
