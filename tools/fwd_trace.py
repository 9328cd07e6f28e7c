import sys
import numpy as np
raw = open(sys.argv[1], "rb").read()
n, slots = np.frombuffer(raw[:16], np.int64)
a = np.frombuffer(raw[16:], np.uint64).reshape(n, slots).astype(np.int64)
a = a[(a[:, 1] > 0) & (a[:, 5] > 0) & (a[:, 12] > 0)]
print("ctas:", len(a))
def d(x, y, name):
    v = (a[:, y] - a[:, x])
    print(f"  {name:44s} mean {v.mean():8.0f} ns  p50 {np.median(v):8.0f}")
d(1, 2, "sm: S(8) seen -> row max done")
d(2, 3, "sm: max exchange barrier")
d(3, 4, "sm: exp/pack/store -> P(8) arrive")
d(4, 5, "sm: P(8) arrive -> S(9) seen")
d(1, 5, "sm: block period")
d(10, 11, "mma: issue S(9) (+K wait)")
d(11, 12, "mma: wait P(8)+V, issue PV(8)")
d(4, 12, "P(8) arrive -> PV(8) issued")
d(10, 13, "mma: PV(7) issued -> K(9) ready")
d(13, 11, "mma: issue 8 S(9) MMAs")
d(11, 14, "mma: S(9) issued -> P(8) seen")
d(14, 15, "mma: P(8) seen -> V(8) ready")
d(15, 12, "mma: issue 8 PV(8) MMAs")
d(4, 14, "P(8) arrive -> MMA sees it")
b = a[a[:, 6] > 0]
print("observer ctas", len(b))
a = b
d(11, 6, "S(9) issued -> s_full(9) completes (observer)")
d(6, 5, "s_full(9) completes -> softmax sees it")
d(4, 6, "P(8) arrive -> s_full(9) completes")
d(4, 7, "P(8) arrive -> before s_full(9) wait")
d(7, 5, "s_full(9) wait")
