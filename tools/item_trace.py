import sys
import numpy as np
raw = open(sys.argv[1], "rb").read()
n, slots = np.frombuffer(raw[:16], np.int64)
a = np.frombuffer(raw[16:], np.uint64).reshape(n, slots).astype(np.int64)
a = a[(a[:, 8] > 0) & (a[:, 12] > 0) & (a[:, 10] > 0)]
print("ctas with item 8/9:", len(a))
def d(x, y, name):
    v = (a[:, y] - a[:, x])
    print(f"  {name:40s} mean {v.mean():8.0f} ns  p50 {np.median(v):8.0f}")
d(8, 9, "softmax h0 item8 (sdp seen -> arrive)")
d(9, 10, "h0 arrive -> MMA issued dvdk0(8)")
d(10, 11, "MMA issue sdp0(9)")
d(11, 12, "issued -> h0 sees sdp0(9)")
d(8, 12, "h0 item period")
d(13, 14, "softmax h1 item8")
d(13, 15, "h1 item period")
d(8, 13, "h0 start -> h1 start")
if slots > 17:
    d(10, 16, "MMA: dvdk0 issued -> qdo_full(9) passed")
    d(16, 17, "MMA: S^T_0(9) 8 MMAs issued")
    d(17, 11, "MMA: dP^T_0(9) 8 MMAs issued + commit")
