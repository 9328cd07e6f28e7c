import sys
import numpy as np
raw = open(sys.argv[1], "rb").read()
n, slots = np.frombuffer(raw[:16], np.int64)
a = np.frombuffer(raw[16:], np.uint64).reshape(n, slots).astype(np.int64)
a = a[(a[:, 1] > 0) & (a[:, 6] > 0)]
print("ctas", len(a))
for x, y, name in [(1, 2, "S seen -> LDTM x4 done"), (2, 3, "mask + max + m_new"), (3, 4, "rescale? + 128 exp + pack + STTM"),
                   (4, 5, "rowsum + wait::st + arrive"), (5, 6, "arrive -> S(j+2) seen"), (1, 6, "2-block period (WG0)")]:
    v = a[:, y] - a[:, x]
    print(f"  {name:40s} mean {v.mean():7.0f} ns  p50 {np.median(v):7.0f}")
