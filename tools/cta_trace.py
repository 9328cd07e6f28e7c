"""Summarise an OOMB_CTA_TRACE dump: per-phase CTA durations and per-SM idle gaps.
Usage: python tools/cta_trace.py trace.bin [slot names comma-separated]"""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
n, slots = np.frombuffer(raw[:16], np.int64)
a = np.frombuffer(raw[16:], np.uint64).reshape(n, slots).astype(np.int64)
names = sys.argv[2].split(",") if len(sys.argv) > 2 else [f"s{i}" for i in range(slots)]
ok = a[:, 1] > 0
a = a[ok]
t0 = a[:, 1].min()
sm = a[:, 0]
print(f"ctas {len(a)} (of {n}), kernel span {(a[:, 1:7].max() - t0) / 1e3:.1f} us, SMs {len(np.unique(sm))}")
marks = [i for i in range(1, slots) if names[i] and not names[i].startswith("#")]
for i, j in zip(marks[:-1], marks[1:]):
    d = (a[:, j] - a[:, i]) / 1e3
    d = d[(a[:, j] > 0) & (a[:, i] > 0)]
    if len(d):
        print(f"  {names[i]:>10} -> {names[j]:<10} mean {d.mean():7.2f} us  p50 {np.median(d):7.2f}  p90 {np.percentile(d, 90):7.2f}  sum/SM {d.sum() / 148 / 1e3:7.3f} ms")
last = max(marks)
tot = (a[:, last] - a[:, 1]) / 1e3
print(f"  CTA lifetime mean {tot.mean():.2f} us, sum/SM {tot.sum() / 148 / 1e3:.3f} ms")
# gaps between consecutive CTAs on the same SM (launch overhead + co-residency effects)
gaps = []
for s in np.unique(sm):
    r = a[sm == s]
    r = r[np.argsort(r[:, 1])]
    gaps += list((r[1:, 1] - r[:-1, last]) / 1e3)
gaps = np.array(gaps)
print(f"  SM gap between CTAs: mean {gaps.mean():.2f} us p50 {np.median(gaps):.2f} (negative = overlap)")
if slots > 7:
    items = a[:, 7]
    ml = (a[:, marks[-2]] - a[:, marks[2]]) / 1e3 if len(marks) > 3 else None
    for lo, hi in [(0, 8), (8, 16), (16, 32), (32, 64), (64, 10**9)]:
        m = (items >= lo) & (items < hi)
        if m.any():
            print(f"  items [{lo},{hi}): ctas {m.sum():5d}  lifetime {tot[m].mean():7.2f} us  per-item {(tot[m] / items[m]).mean():.3f} us")
