"""Summarise an OOMB_KV_TRACE dump of attn_bwd_dkdv_kernel (per-CTA wait / phase cycle counters).
Usage: python tools/kv_trace.py dump.bin [sm_mhz]"""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
mhz = float(sys.argv[2]) if len(sys.argv) > 2 else 1500.0
n, slots = np.frombuffer(raw[:16], np.int64)
a = np.frombuffer(raw[16:], np.uint64).reshape(n, slots).astype(np.int64)
a = a[a[:, 1] > 0]
span = (a[:, 2].max() - a[:, 1].min()) / 1e3
print(f"ctas {len(a)}  kernel span {span:.1f} us  units {a[:, 3].sum()}  items {a[:, 4].sum()}  "
      f"items/unit {a[:, 4].sum() / max(a[:, 3].sum(), 1):.2f}")
names = {5: "sm: wait unit desc", 6: "sm: wait S(item0)", 7: "sm: wait S(other)", 8: "sm: wait dP",
         9: "sm: wait acc_done", 10: "sm: epilogue", 11: "sm: P phase", 12: "sm: dS phase", 21: "sm: total",
         13: "mma: wait Q/dO", 14: "mma: wait P", 15: "mma: wait dS", 16: "mma: wait acc_free", 17: "mma: wait K/V",
         18: "prod: wait Q/dO slot", 19: "prod: wait K/V slot", 20: "prod: wait desc slot"}
tot = a[:, 21].mean()
for k in sorted(names):
    v = a[:, k].mean()
    print(f"  {names[k]:24s} {v / mhz:9.2f} us/CTA  {v / tot * 100:6.1f} %  per item {a[:, k].sum() / max(a[:, 4].sum(), 1):8.0f} clk")
