"""Pure host cost of each per-chunk API call (queue drained before each call)."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import bench
cfg = dict(bench.CONFIGS["c3"]); cfg["T"] = 1 << 18
r = bench.Run(cfg, 0, torch.device("cuda:0"))
r.step(); torch.cuda.synchronize()
C = cfg["C"]
tm = {}
def t(name, f):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); f(); dt = time.perf_counter() - t0
    tm.setdefault(name, []).append(dt)
for rep in range(2):
    r.cache.reset()
    for i in range(r.S):
        q, k, v = r.q[i % r.RQ], r.k_all[i * C:(i + 1) * C], r.v_all[i * C:(i + 1) * C]
        t("select", lambda: r._select(i, q))
        t("append", lambda: r.cache.append_chunk(0, k, v))
        t("fwd", lambda: r.A.attn_forward(r.mc, q, r.cache, 0, r.sels[i], k, v, out=r.o_all[i], lse=r.lse_all[i]))
    for i in reversed(range(r.S)):
        q, k, v = r.q[i % r.RQ], r.k_all[i * C:(i + 1) * C], r.v_all[i * C:(i + 1) * C]
        g = r.grads
        saved = r.A.AttnSaved(r.o_all[i], r.lse_all[i], r.sels[i])
        t("bwd", lambda: r.A.attn_backward(r.mc, r.do[i % r.RQ], q, r.cache, 0, k, v, saved, grads=g))
        t("acc", lambda: r.cache.accumulate_grad_pages(0, r.own[i], g.dk_cur, g.dv_cur))
for k, v in tm.items():
    v = v[len(v) // 2:]
    print(f"{k:8s} host us per call: mean {1e6 * sum(v) / len(v):8.1f}  max {1e6 * max(v):8.1f}")
