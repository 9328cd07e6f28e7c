import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2602_02108_b200.tiered_memory import TierConfig
from paper_2602_02108_b200.trainer import ChunkTrainer, flatten, unflatten, param_shapes
from tests.golden.make_model_golden import model_cfg
z = np.load("tests/golden/model_step.npz")
mode = sys.argv[1] if len(sys.argv) > 1 else "dense"
cfg = model_cfg(mode)
mt = len(z["tokens"]) + cfg.chunk_size
plain = ChunkTrainer(cfg, max_tokens=mt, dtype="fp32")
_, g0 = plain.train_step(unflatten(z["params"], cfg, plain.dev), z["tokens"])
f0 = flatten(g0, cfg).cpu().numpy()
for cap in (1000, 40, 30, 24, 20):
    tr = ChunkTrainer(cfg, max_tokens=mt, dtype="fp32", tier=TierConfig(device_capacity_pages=cap, bandwidth_bytes_per_s=16e9))
    _, g1 = tr.train_step(unflatten(z["params"], cfg, tr.dev), z["tokens"])
    f1 = flatten(g1, cfg).cpu().numpy()
    ev = np.array([(e.kind, e.layer, e.page, e.chunk, e.phase, e.bytes) for e in tr.last_log], np.int64)
    bad = []
    o = 0
    for name, layer, shape in param_shapes(cfg):
        n = int(np.prod(shape))
        d = np.abs(f1[o:o+n] - f0[o:o+n]).max()
        if d > 0: bad.append((name, layer, float(d)))
        o += n
    print("cap", cap, "evicts", int((ev[:,0]==2).sum()), "fetch_done", int((ev[:,0]==1).sum()), "diff params", bad[:6])
    if cap == 20:
        want = z[f"{mode}_offload_events"]
        same = ev.shape == want.shape and np.array_equal(ev, want)
        print("events equal to reference:", same, ev.shape, want.shape)
        if not same:
            n = min(len(ev), len(want))
            i = next((i for i in range(n) if not np.array_equal(ev[i], want[i])), n)
            print("first diff at", i, ev[max(0,i-3):i+3].tolist(), want[max(0,i-3):i+3].tolist())
    if cap == 20:
        for name, L in (("ours", ev), ("ref", want)):
            idx = [(i, L[i].tolist()) for i in range(len(L)) if L[i][1] == 1 and L[i][2] == 0]
            print(name, "layer1 page0 events:", idx[-12:])
    if cap == 20:
        K = {0: "issue", 1: "done", 2: "evict", 3: "cbeg", 4: "cend", 5: "acc"}
        for i in range(500, 575):
            a = ev[i].tolist() if i < len(ev) else None
            b = want[i].tolist() if i < len(want) else None
            if a and b and a[0] in (3, 4) and b[0] in (3, 4) and a == b:
                continue
            print(i, "ours", K.get(a[0]) if a else None, a[1:] if a else None, "| ref", K.get(b[0]) if b else None, b[1:] if b else None)
