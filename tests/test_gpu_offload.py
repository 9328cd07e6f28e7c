"""Real offload on the device: a multi-chunk attention layer run with a capacity-
limited TieredEngine (pages written back to pinned host memory and fetched back
on side streams) must give BITWISE the same outputs and gradient pages as the
all-resident run (test_tiered_memory.cpp:429-454, "offload on/off bitwise
identical"), and its CUDA-event ScheduleLog must pass validate_schedule with no
residency violations."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def make(mode, capacity=None, n_layers=2):
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200.chunk_loop import AttentionChunkLoop
    from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine
    cfg = ModelConfig(n_layers=n_layers, n_q_heads=28, n_kv_heads=4, head_dim=128, chunk_size=512, page_size=128,
                      retrieval_budget=3 * 128, local_window=3, attention_mode=[mode])
    slots = -1 if capacity is None else capacity + 24  # physical slots: capacity + in-flight staging
    cache = PagedCache(cfg, dtype="bf16", max_tokens=8 * 512, device_capacity_pages=slots)
    eng = None
    if capacity is not None:
        eng = TieredEngine(cache, TierConfig(device_capacity_pages=capacity, bandwidth_bytes_per_s=25e9))
        eng.set_prefetch_headroom_pages(cfg.pages_per_chunk())
    return cache, [AttentionChunkLoop(cache, layer=l, engine=eng) for l in range(n_layers)], eng


def run(mode, capacity, n_chunks=6, seed=3, n_layers=2, pipelined=None):
    """Two attention layers interleaved per chunk, as the trainer runs them (chunk_trainer.hpp:131-186):
    while one layer attends, the other layer's pages are the eviction candidates. pipelined (default:
    with an engine): every chunk's selection is issued one chunk ahead on a side stream."""
    pipelined = capacity is not None if pipelined is None else pipelined
    cache, loops, eng = make(mode, capacity, n_layers)
    g = torch.Generator(device="cuda").manual_seed(seed)
    C = cache.cfg.chunk_size
    rnd = lambda h: [[torch.randn(C, h, 128, device="cuda", generator=g).bfloat16() for _ in range(n_chunks)]
                     for _ in range(n_layers)]
    qs, ks, vs, dos = rnd(28), rnd(4), rnd(4), rnd(28)
    outs, grads = [], []
    for i in range(n_chunks):
        for l, loop in enumerate(loops):
            nq = qs[l][i + 1] if pipelined and i + 1 < n_chunks else None
            s = loop.forward_chunk(i, qs[l][i], ks[l][i], vs[l][i], next_q=nq)
            outs.append((s.out.clone(), s.lse.clone()))
    loops[0].begin_backward()
    for i in reversed(range(n_chunks)):
        for l in reversed(range(n_layers)):
            gr = loops[l].backward_chunk(i, dos[l][i], qs[l][i], ks[l][i], vs[l][i])
            grads.append((gr.dq.clone(), gr.dk_cur.clone(), gr.dv_cur.clone()))
    torch.cuda.synchronize()
    cache.check_device_errors()  # no kernel read a slot that was not resident
    log = None
    if eng is not None:
        eng.release_all_reservations()
        log = eng.log()
        stats = (eng.h2d_bytes(0), eng.h2d_bytes(1), eng.d2h_bytes())
        # the engine leaves; the pool (capacity + 24 slots) cannot take every page back, and the
        # outputs were read above: drop what stays on the host (close() would raise ResidencyError)
        eng.close(discard=True)
    else:
        stats = None
    sels = [s.lists() for loop in loops for s in loop.sels]
    return outs, grads, sels, log, stats, cache


def _explain(log, rep):
    """First violations with the events of the same page around them (diagnostics)."""
    lines = rep.violations[:5]
    for msg in rep.violations[:3]:
        if "page=" not in msg:
            continue
        page = int(msg.split("page=")[1].split()[0])
        evs = [(i, e.kind, e.chunk, e.phase, e.bytes, round(e.t * 1e6, 2)) for i, e in enumerate(log.events)
               if e.page == page]
        lines.append(f"page {page}: {evs[:40]}")
    return "\n".join(lines)


@pytest.mark.parametrize("mode", ["topk", "dense", "local"])
def test_offload_bitwise_identical(mode):
    from paper_2602_02108_b200.tiered_memory import validate_schedule
    a_out, a_gr, a_sel, _, _, a_cache = run(mode, None)
    cap = 12 if mode != "dense" else 24  # dense: one layer's whole past (20 pages) + its chunk (4)
    b_out, b_gr, b_sel, log, stats, b_cache = run(mode, cap)
    assert a_sel == b_sel
    for (o1, l1), (o2, l2) in zip(a_out, b_out):
        assert torch.equal(o1, o2) and torch.equal(l1, l2)
    for x, y in zip(a_gr, b_gr):
        for u, w in zip(x, y):
            assert torch.equal(u, w)
    assert stats[2] > 0 and stats[0] + stats[1] > 0, "the capacity must force write-backs and fetches"
    rep = validate_schedule(log)
    assert rep.violations == [], _explain(log, rep)
    assert any(e.kind == "evict" and e.bytes > 0 for e in log.events)


def test_offload_pages_round_trip_exactly():
    """Every page evicted to the host and fetched back carries identical K/V bytes."""
    from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    cfg = ModelConfig(n_layers=1, n_q_heads=28, n_kv_heads=4, head_dim=128, chunk_size=512, page_size=128,
                      retrieval_budget=256)
    cache = PagedCache(cfg, dtype="bf16", max_tokens=16 * 128, device_capacity_pages=16)
    k = torch.randn(16 * 128, 4, 128, device="cuda").bfloat16()
    v = torch.randn(16 * 128, 4, 128, device="cuda").bfloat16()
    eng = TieredEngine(cache, TierConfig(device_capacity_pages=8, bandwidth_bytes_per_s=25e9))
    for c in range(4):  # appended pages are reserved until the layer is done with them (tiered_memory.hpp:131-145)
        r = cache.append_chunk(0, k[c * 512:(c + 1) * 512], v[c * 512:(c + 1) * 512])
        eng.on_pages_appended(0, r)
        eng.end_layer_use(0, list(range(4 * c, 4 * c + 4)))  # capacity 8 -> older pages written back
    tiers = [cache.tier(0, p) for p in range(16)]
    assert sum(tiers) == 8
    evicted = [p for p in range(16) if tiers[p]]
    eng.wait(eng.fetch_async(0, evicted[:4]))        # 4 come back (4 more go out)
    eng.record_access(0, evicted[:4])
    got = cache.gather_pages(0, evicted[:4])
    for j, p in enumerate(evicted[:4]):
        assert torch.equal(got.k[j * 128:(j + 1) * 128], k[p * 128:(p + 1) * 128])
        assert torch.equal(got.v[j * 128:(j + 1) * 128], v[p * 128:(p + 1) * 128])
    eng.close()


def test_restore_all_needs_free_slots_and_keeps_data():
    """oomb_tier_restore_all: all-or-nothing ConfigError when the pool lacks free device slots for
    the host-tier pages; with room, every page comes back resident with its K/V and gradients
    bitwise (what engine close() relies on)."""
    from paper_2602_02108_b200 import ConfigError, ModelConfig, PagedCache
    from paper_2602_02108_b200.chunk_loop import AttentionChunkLoop
    from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine
    cfg = ModelConfig(n_layers=1, n_q_heads=28, n_kv_heads=4, head_dim=128, chunk_size=512, page_size=128,
                      retrieval_budget=3 * 128, local_window=3, attention_mode=["topk"])
    g = torch.Generator(device="cuda").manual_seed(5)
    n = 10  # 40 pages: with 36 device slots and capacity 20 the host holds more pages than there are free slots
    rnd = lambda h: [torch.randn(512, h, 128, device="cuda", generator=g).bfloat16() for _ in range(n)]
    qs, ks, vs, dos = rnd(28), rnd(4), rnd(4), rnd(28)
    pools = []
    for slots, cap in ((-1, None), (20 + 16, 20), (-1, 20)):
        cache = PagedCache(cfg, dtype="bf16", max_tokens=n * 512, device_capacity_pages=slots)
        eng = None
        if cap is not None:
            eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap, bandwidth_bytes_per_s=25e9))
            eng.set_prefetch_headroom_pages(cfg.pages_per_chunk())
        loop = AttentionChunkLoop(cache, engine=eng)
        for i in range(n):
            loop.forward_chunk(i, qs[i], ks[i], vs[i])
        loop.begin_backward()
        for i in reversed(range(n)):
            loop.backward_chunk(i, dos[i], qs[i], ks[i], vs[i])
        torch.cuda.synchronize()
        if eng is not None:
            eng.release_all_reservations()
            host = [p for p in range(cache.n_pages(0)) if cache.tier(0, p) != 0]
            assert host, "the capacity must leave pages on the host"
            if slots > 0:
                with pytest.raises(ConfigError):
                    eng.restore_all()
                assert [p for p in range(cache.n_pages(0)) if cache.tier(0, p) != 0] == host  # nothing moved
                from paper_2602_02108_b200.errors import ResidencyError
                with pytest.raises(ResidencyError):  # detaching without room loses those pages, loudly
                    eng.close()
                assert all(cache.tier(0, p) == 3 for p in host)
                with pytest.raises(ResidencyError):
                    cache.gather_grad_pages(0, host[:1])
                continue
            eng.restore_all()
            assert all(cache.tier(0, p) == 0 for p in range(cache.n_pages(0)))
            eng.close()
        ids = list(range(cache.n_pages(0)))
        kv, gr = cache.gather_pages(0, ids), cache.gather_grad_pages(0, ids)
        pools.append((kv.k.clone(), kv.v.clone(), gr.k.clone(), gr.v.clone()))
    for a, b in zip(*pools):
        assert torch.equal(a, b)
