"""Offload transparency at BASELINE's full c3 size: the 1M-token layer step that bench.py's
`offload` key times (AttentionChunkLoop + TieredEngine with the device pool capped at 75 % of
the layer's pages, bench.offload_measure) gives BITWISE the same selections, outputs, LSEs,
per-chunk gradients and gradient pool as the all-resident step (test_tiered_memory.cpp:429-454,
"offload on/off bitwise identical", at the benchmark's size).

Per-chunk tensors are compared through an exact integer digest of their bits (a weighted sum of
the raw words in int64), so a 1M-token run does not have to keep every gradient twice."""
import pytest
import torch

pytestmark = pytest.mark.gpu

T, C, P, HQ, HKV, HD, K_SEL, RQ = 1 << 20, 4096, 128, 28, 4, 128, 64, 4
S = T // C


def digest(t: torch.Tensor) -> int:
    w = t.contiguous().view(-1).view(torch.int16 if t.element_size() == 2 else torch.int32).to(torch.int64)
    idx = torch.arange(w.numel(), device=w.device, dtype=torch.int64)
    return int(((w + 40503) * (idx * 2654435761 % 1000003 + 1)).sum())


@pytest.fixture(scope="module")
def data():
    g = torch.Generator(device="cuda").manual_seed(11)
    rnd = lambda *s: torch.randn(*s, device="cuda", generator=g).bfloat16()
    return dict(K=rnd(T, HKV, HD), V=rnd(T, HKV, HD), q=[rnd(C, HQ, HD) for _ in range(RQ)],
                do=[rnd(C, HQ, HD) for _ in range(RQ)])


def layer_step(d, cap_frac):
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200.chunk_loop import AttentionChunkLoop
    from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine
    cfg = ModelConfig(n_layers=1, n_q_heads=HQ, n_kv_heads=HKV, head_dim=HD, chunk_size=C, page_size=P,
                      retrieval_budget=K_SEL * P, attention_mode=["topk"])
    n_pages = T // P
    use = cap_frac < 1.0
    cap = int(cap_frac * n_pages)
    # the same pool and engine settings as bench.offload_measure
    cache = PagedCache(cfg, dtype="bf16", max_tokens=T,
                       device_capacity_pages=min(n_pages, cap + 4096 + 64) if use else -1)
    eng = None
    if use:
        eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap, bandwidth_bytes_per_s=55e9))
        eng.set_prefetch_headroom_pages(C // P)
    loop = AttentionChunkLoop(cache, engine=eng)
    K, V, q, do = d["K"], d["V"], d["q"], d["do"]
    out = torch.empty(C, HQ, HD, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(C, HQ, dtype=torch.float32, device="cuda")
    fwd, bwd = [], []
    for i in range(S):
        nq = q[(i + 1) % RQ] if i + 1 < S else None
        loop.forward_chunk(i, q[i % RQ], K[i * C:(i + 1) * C], V[i * C:(i + 1) * C], next_q=nq, out=out, lse=lse)
        fwd.append((digest(out), digest(lse)))
    loop.begin_backward()
    for i in reversed(range(S)):
        gr = loop.backward_chunk(i, do[i % RQ], q[i % RQ], K[i * C:(i + 1) * C], V[i * C:(i + 1) * C])
        bwd.append((digest(gr.dq), digest(gr.dk_cur), digest(gr.dv_cur)))
    torch.cuda.synchronize()
    cache.check_device_errors()
    stats = None
    if eng is not None:
        eng.release_all_reservations()
        stats = (eng.h2d_bytes(0) + eng.h2d_bytes(1), eng.d2h_bytes())
        eng.close()  # every page is readable again
    sels = [s.lists() for s in loop.sels]
    pool = []
    for p0 in range(0, n_pages, 512):
        gp = cache.gather_grad_pages(0, list(range(p0, min(n_pages, p0 + 512))))
        pool.append((digest(gp.k), digest(gp.v)))
    del loop, eng, cache
    torch.cuda.empty_cache()
    return fwd, bwd, sels, pool, stats


def test_offload_bitwise_identical_at_1m(data):
    a_fwd, a_bwd, a_sel, a_pool, _ = layer_step(data, 1.0)
    b_fwd, b_bwd, b_sel, b_pool, stats = layer_step(data, 0.75)
    assert stats[0] > 0 and stats[1] > 0, "the 75 % cap must force fetches and write-backs"
    assert a_sel == b_sel
    assert a_fwd == b_fwd
    assert a_bwd == b_bwd
    assert a_pool == b_pool
