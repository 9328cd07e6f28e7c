"""Real offload engine edge cases: attaching to a pool that already holds pages,
the reference's own pattern (fill pages, tag them host, then build the engine), detaching without
room to restore, appending into an evicted tail page, and duplicate ids in one fetch. Data must
never be lost silently: every page comes back bit-identical, or the read raises ResidencyError."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _cache(slots=-1, pages=16):
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    cfg = ModelConfig(n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=128, chunk_size=128, page_size=128,
                      retrieval_budget=256, attention_mode=["topk"])
    return PagedCache(cfg, dtype="bf16", max_tokens=pages * 128, device_capacity_pages=slots)


def _kv(n_rows, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(n_rows, 2, 128, device="cuda", generator=g).bfloat16(),
            torch.randn(n_rows, 2, 128, device="cuda", generator=g).bfloat16())


def _engine(cache, capacity):
    from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine
    return TieredEngine(cache, TierConfig(device_capacity_pages=capacity, bandwidth_bytes_per_s=25e9))


def test_attach_to_filled_pool_writes_back_before_evicting():
    """Pages appended before the engine existed have no host copy: their first eviction must write
    them back (K/V and gradients), so fetching them again restores them bit for bit."""
    cache = _cache()
    k, v = _kv(6 * 128, 1)
    cache.append_chunk(0, k, v)
    dk = torch.randn(3 * 128, 2, 128, device="cuda")
    dv = torch.randn(3 * 128, 2, 128, device="cuda")
    cache.scatter_add_grads(0, [0, 1, 2], dk, dv)
    want = cache.gather_pages(0, range(6))
    want_g = cache.gather_grad_pages(0, range(6))
    eng = _engine(cache, 2)
    eng.end_layer_use(0, [])  # capacity enforcement: 4 of the 6 pages go to the host
    assert sum(cache.tier(0, p) for p in range(6)) == 4
    for p in range(6):
        h = eng.fetch_async(0, [p])
        eng.wait(h)
        got = cache.gather_pages(0, [p])
        got_g = cache.gather_grad_pages(0, [p])
        sl = slice(p * 128, (p + 1) * 128)
        assert torch.equal(got.k, want.k[sl]) and torch.equal(got.v, want.v[sl])
        assert torch.equal(got_g.k, want_g.k[sl]) and torch.equal(got_g.v, want_g.v[sl])
        eng.end_layer_use(0, [p])
    eng.close()
    torch.cuda.synchronize()
    cache.check_device_errors()


def test_reference_pattern_set_tier_then_engine():
    """test_tiered_memory.cpp's pattern: fill pages, set_tier(host), construct the engine, fetch.
    The engine moves the host-tagged pages' data to pinned memory and frees their slots at attach."""
    cache = _cache(slots=6)
    k, v = _kv(4 * 128, 2)
    cache.append_chunk(0, k, v)
    want = cache.gather_pages(0, range(4))
    cache.set_tier(0, 1, 1)
    cache.set_tier(0, 2, 1)
    eng = _engine(cache, 4)
    slots = cache.device_slots(0)
    assert slots[1, 0] < 0 and slots[2, 0] < 0  # no slot leaked to a host-tier page
    h = eng.fetch_async(0, [1, 2])
    eng.wait(h)
    got = cache.gather_pages(0, range(4))
    assert torch.equal(got.k, want.k) and torch.equal(got.v, want.v)
    # the pool's 6 slots: 4 resident pages + 2 free ones -> two more pages still fit
    k2, v2 = _kv(2 * 128, 3)
    eng.end_layer_use(0, [1, 2])
    cache.append_chunk(0, k2, v2)
    eng.close()


def test_detach_without_room_reports_and_marks_pages_lost():
    from paper_2602_02108_b200.errors import ResidencyError
    cache = _cache(slots=3)
    eng = _engine(cache, 1)
    for c in range(5):  # 5 pages through a 3-slot pool at capacity 1
        k, v = _kv(128, 10 + c)
        r = cache.append_chunk(0, k, v)
        eng.on_pages_appended(0, r)
        eng.end_layer_use(0, [c])
    host = [p for p in range(5) if cache.tier(0, p) == 1]
    assert len(host) == 4
    with pytest.raises(ResidencyError):
        eng.close()  # 4 host-tier pages, 2 free slots: they cannot all come back
    assert [cache.tier(0, p) for p in host] == [3] * 4
    with pytest.raises(ResidencyError):
        cache.gather_pages(0, [host[0]])
    with pytest.raises(ResidencyError):
        cache.gather_grad_pages(0, [host[0]])
    dk = torch.zeros(128, 2, 128, device="cuda")
    with pytest.raises(ResidencyError):
        cache.accumulate_grad_pages(0, [host[0]], dk, dk.clone())
    cache.reset()  # a reset clears the lost tags with everything else
    k, v = _kv(128, 20)
    cache.append_chunk(0, k, v)
    assert cache.tier(0, 0) == 0


def test_append_into_evicted_tail_page_raises():
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200.errors import ResidencyError
    cfg = ModelConfig(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=128, chunk_size=128, page_size=128,
                      retrieval_budget=256, attention_mode=["topk"])
    cache = PagedCache(cfg, dtype="bf16", max_tokens=4 * 128)
    eng = _engine(cache, 1)
    k, v = _kv(64, 4)  # half a page
    r = cache.append_chunk(0, k, v)
    eng.on_pages_appended(0, r)
    eng.end_layer_use(0, [0])
    r1 = cache.append_chunk(1, k, v)  # layer 1's page takes the one device page: layer 0's tail goes out
    eng.on_pages_appended(1, r1)
    eng.end_layer_use(1, [0])
    assert cache.tier(0, 0) == 1
    with pytest.raises(ResidencyError):
        cache.append_chunk(0, k, v)
    assert cache.filled(0) == 64  # the failed append left the page table untouched
    h = eng.fetch_async(0, [0])
    eng.wait(h)
    cache.append_chunk(0, k, v)  # resident again: the rows land in place
    got = cache.gather_pages(0, [0])
    assert torch.equal(got.k[:64], k) and torch.equal(got.k[64:], k)
    eng.close(discard=True)
    torch.cuda.synchronize()
    cache.check_device_errors()


def test_duplicate_ids_in_one_fetch_take_one_slot():
    cache = _cache(slots=3)
    k, v = _kv(2 * 128, 5)
    cache.append_chunk(0, k, v)
    want = cache.gather_pages(0, [0, 1])
    eng = _engine(cache, 1)
    eng.end_layer_use(0, [])
    for it in range(8):  # a leaked slot per duplicate fetch would exhaust the 3-slot pool
        p = it % 2
        h = eng.fetch_async(0, [p, p, p])
        eng.wait(h)
        got = cache.gather_pages(0, [p])
        assert torch.equal(got.k, want.k[p * 128:(p + 1) * 128])
        eng.end_layer_use(0, [p])
    slots = cache.device_slots(0)
    assert int((slots[:, 0] >= 0).sum()) == 1
    eng.close(discard=True)
