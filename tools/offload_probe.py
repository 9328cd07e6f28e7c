"""c3 through the reference's residency protocol (AttentionChunkLoop + TieredEngine) at a given
device capacity: wall time per 1M-token layer step vs the all-resident loop, and the traffic."""
import os, sys, time, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2602_02108_b200 import ModelConfig, PagedCache
from paper_2602_02108_b200.chunk_loop import AttentionChunkLoop
from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine

T = int(os.environ.get("T", 1 << 20)); C, P, Hq, Hkv, hd = 4096, 128, 28, 4, 128
caps = [float(x) for x in os.environ.get("CAPS", "1.0,0.75,0.5").split(",")]
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(7)
S = T // C
k_all = torch.randn(T, Hkv, hd, device=dev, generator=g).bfloat16()
v_all = torch.randn(T, Hkv, hd, device=dev, generator=g).bfloat16()
qs = [torch.randn(C, Hq, hd, device=dev, generator=g).bfloat16() for _ in range(8)]
dos = [torch.randn(C, Hq, hd, device=dev, generator=g).bfloat16() for _ in range(8)]
mc = ModelConfig(n_layers=1, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=hd, chunk_size=C, page_size=P,
                 retrieval_budget=8192, attention_mode=["topk"])
n_pages = T // P
res = []
def one_step(frac):
    cap = int(frac * n_pages)
    use_eng = frac < 1.0
    slots = min(n_pages, cap + 4096 + 64) if use_eng else -1
    cache = PagedCache(mc, dtype="bf16", max_tokens=T, device_capacity_pages=slots)
    eng = None
    if use_eng:
        eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap, bandwidth_bytes_per_s=55e9))
        eng.set_prefetch_headroom_pages(C // P)
    loop = AttentionChunkLoop(cache, engine=eng)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(S):
        loop.forward_chunk(i, qs[i % 8], k_all[i * C:(i + 1) * C], v_all[i * C:(i + 1) * C])
    loop.begin_backward()
    for i in reversed(range(S)):
        loop.backward_chunk(i, dos[i % 8], qs[i % 8], k_all[i * C:(i + 1) * C], v_all[i * C:(i + 1) * C])
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    r = {"cap_frac": frac, "cap_pages": cap, "wall_s": wall}
    if eng is not None:
        r.update(h2d_fwd=eng.h2d_bytes(0), h2d_bwd=eng.h2d_bytes(1), d2h=eng.d2h_bytes())
        eng.release_all_reservations()
        eng.close()
    del loop, eng, cache
    torch.cuda.empty_cache()
    return r
one_step(1.0)  # warm-up: lazy loading, tensor maps, pool growth
for frac in caps:
    print(json.dumps(one_step(frac)), flush=True)
raise SystemExit(0)
for frac in caps:
    cap = int(frac * n_pages)
    use_eng = frac < 1.0
    slots = min(n_pages, cap + 4096 + 64) if use_eng else -1
    cache = PagedCache(mc, dtype="bf16", max_tokens=T, device_capacity_pages=slots)
    eng = None
    if use_eng:
        eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap, bandwidth_bytes_per_s=55e9))
        eng.set_prefetch_headroom_pages(C // P)
    loop = AttentionChunkLoop(cache, engine=eng)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(S):
        loop.forward_chunk(i, qs[i % 8], k_all[i * C:(i + 1) * C], v_all[i * C:(i + 1) * C])
    loop.begin_backward()
    for i in reversed(range(S)):
        loop.backward_chunk(i, dos[i % 8], qs[i % 8], k_all[i * C:(i + 1) * C], v_all[i * C:(i + 1) * C])
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    r = {"cap_frac": frac, "cap_pages": cap, "wall_s": wall}
    if eng is not None:
        r.update(h2d_fwd=eng.h2d_bytes(0), h2d_bwd=eng.h2d_bytes(1), d2h=eng.d2h_bytes())
        eng.release_all_reservations()
        eng.close()
    res.append(r)
    print(json.dumps(r), flush=True)
    del loop, eng, cache
    torch.cuda.empty_cache()
