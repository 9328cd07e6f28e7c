import sys
import numpy as np
raw = open(sys.argv[1], "rb").read()
n, slots = np.frombuffer(raw[:16], np.int64)
a = np.frombuffer(raw[16:], np.uint64).reshape(n, slots).astype(np.int64)
a = a[(a[:, 8] > 0) & (a[:, 17] > 0) & (a[:, 16] > 0)]
print("ctas with item 8/9:", len(a))
def d(x, y, name):
    v = (a[:, y] - a[:, x])
    print(f"  {name:44s} mean {v.mean():8.0f} ns  p50 {np.median(v):8.0f}")
d(8, 9, "sm: S(8) seen -> P(8) stored")
d(9, 10, "sm: P stored -> dP(8) seen")
d(10, 11, "sm: dP seen -> dS(8) stored")
d(11, 17, "sm: dS stored -> S(9) seen")
d(8, 17, "sm: item period")
d(12, 13, "mma: wait P(8) + issue dV(8)")
d(13, 14, "mma: issue S(9) (+qdo wait)")
d(14, 15, "mma: wait dS(8) + issue dK(8)")
d(15, 16, "mma: issue dP(9)")
d(9, 13, "P(8) stored -> dV(8) issued")
d(11, 15, "dS(8) stored -> dK(8) issued")
