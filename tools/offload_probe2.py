"""Where the exposed time of the offload protocol goes: per-phase wall time and host time per
protocol call (AttentionChunkLoop + TieredEngine at c3), capped vs all-resident."""
import collections, json, os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import torch
from paper_2602_02108_b200 import ModelConfig, PagedCache
from paper_2602_02108_b200 import attention as A
from paper_2602_02108_b200.chunk_loop import AttentionChunkLoop
from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine

T = int(os.environ.get("T", 1 << 20)); C, P, Hq, Hkv, hd = 4096, 128, 28, 4, 128
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(7)
S = T // C
k_all = torch.randn(T, Hkv, hd, device=dev, generator=g).bfloat16()
v_all = torch.randn(T, Hkv, hd, device=dev, generator=g).bfloat16()
qs = [torch.randn(C, Hq, hd, device=dev, generator=g).bfloat16() for _ in range(8)]
dos = [torch.randn(C, Hq, hd, device=dev, generator=g).bfloat16() for _ in range(8)]
o_all = torch.empty(S, C, Hq, hd, device=dev, dtype=torch.bfloat16)
lse_all = torch.empty(S, C, Hq, device=dev)
grads = A.AttnGrads(torch.empty(C, Hq, hd, device=dev), torch.empty(C, Hkv, hd, device=dev), torch.empty(C, Hkv, hd, device=dev))
mc = ModelConfig(n_layers=1, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=hd, chunk_size=C, page_size=P,
                 retrieval_budget=8192, attention_mode=["topk"])
n_pages = T // P
acc = collections.defaultdict(float)


def wrap(obj, name):
    f = getattr(obj, name)
    def w(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        acc[name] += time.perf_counter() - t
        return r
    setattr(obj, name, w)


for n in ("attn_forward", "attn_backward", "select_pages_topk"):
    wrap(A, n)
# host time per C entry point
from paper_2602_02108_b200 import _lib
_orig_call = _lib.call
def _timed_call(name, *a):
    t = time.perf_counter()
    try:
        return _orig_call(name, *a)
    finally:
        acc["C:" + name] += time.perf_counter() - t
_lib.call = _timed_call
import paper_2602_02108_b200.attention as _att, paper_2602_02108_b200.paged_kv as _pk, paper_2602_02108_b200.tiered_memory as _tm, paper_2602_02108_b200.chunk_loop as _cl
for m in (_att, _pk, _tm, _cl):
    m.call = _timed_call


def one_step(frac, pipelined=True):
    acc.clear()
    cap = int(frac * n_pages)
    use_eng = frac < 1.0
    slots = min(n_pages, cap + 4096 + 64) if use_eng else -1
    cache = PagedCache(mc, dtype="bf16", max_tokens=T, device_capacity_pages=slots)
    eng = None
    if use_eng:
        eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap, bandwidth_bytes_per_s=55e9))
        eng.set_prefetch_headroom_pages(C // P)
        for n in ("fetch_async", "wait", "record_access", "end_layer_use", "on_pages_appended", "on_grads_scattered"):
            wrap(eng, n)
    for n in ("append_chunk", "accumulate_grad_pages"):
        wrap(cache, n)
    loop = AttentionChunkLoop(cache, engine=eng)
    wrap(loop, "union")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(S):
        nq = qs[(i + 1) % 8] if pipelined and i + 1 < S else None
        loop.forward_chunk(i, qs[i % 8], k_all[i * C:(i + 1) * C], v_all[i * C:(i + 1) * C], next_q=nq,
                           out=o_all[i], lse=lse_all[i])
    t_enq_f = time.perf_counter() - t0
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    loop.begin_backward()
    for i in reversed(range(S)):
        loop.backward_chunk(i, dos[i % 8], qs[i % 8], k_all[i * C:(i + 1) * C], v_all[i * C:(i + 1) * C], grads=grads)
    t_enq_b = time.perf_counter() - t1
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r = {"cap_frac": frac, "pipelined": pipelined, "fwd_s": round(t1 - t0, 4), "fwd_host_enqueue_s": round(t_enq_f, 4),
         "bwd_s": round(t2 - t1, 4), "bwd_host_enqueue_s": round(t_enq_b, 4),
         "host_s": {k: round(v, 4) for k, v in sorted(acc.items(), key=lambda x: -x[1])}}
    if eng is not None:
        r.update(h2d_fwd=eng.h2d_bytes(0), h2d_bwd=eng.h2d_bytes(1), d2h=eng.d2h_bytes())
        eng.release_all_reservations()
        eng.close()
    del loop, eng, cache
    torch.cuda.empty_cache()
    return r


one_step(1.0)
for frac, pipe in ((1.0, True), (0.75, True), (0.75, True), (1.0, True), (0.75, True)):
    r = one_step(frac, pipe)
    print(json.dumps({k: r[k] for k in ("cap_frac", "fwd_s", "bwd_s", "fwd_host_enqueue_s", "bwd_host_enqueue_s")}),
          json.dumps({k: v for k, v in r["host_s"].items() if v > 0.02}), flush=True)
if os.environ.get("PROFILE"):
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    one_step(0.75, True)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
