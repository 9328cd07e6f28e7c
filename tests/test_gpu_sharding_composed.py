"""Composed KV-group x page-range split on one GPU (BASELINE configs[3]: Qwen2.5-7B's
4 KV groups on 8 GPUs = 4 KV shards x 2 page ranges).

Eight simulated ranks each own a PagedCache built by ShardPlan.make_cache: one KV group's heads, and
K/V + gradient storage only for the pages of its range (id % 2); K_avg is kept for every page. Over
several chunks of a top-k layer, each rank scores its group (the partial votes of the ranks holding
the same page range are reduced in global group order), selects, attends its owned pages (range
rank 0 also the chunk's own keys), the (O, LSE) pairs of a range group are merged exactly, the
backward runs with the merged (O, LSE), the dM_i read-back adds the owned pages among the chunk's
own, and dQ / dk_cur / dv_cur are summed over the range group in rank order. The result must
match the unsplit layer: selections bitwise, out / lse / dq / dk_cur / dv_cur and every owner's
gradient pages within the bf16 tolerance of BASELINE north_star (2e-2), and each rank's device
pool must hold only its share of the pages."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / max(b.norm(), 1e-30))


def _run(world, mode, dtype, chunks=4, seed=5):
    from paper_2602_02108_b200 import ModelConfig
    from paper_2602_02108_b200 import attention as A
    from paper_2602_02108_b200.sharding import ShardPlan, fixed_order_sum, lse_merge
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    C, P, Hq, Hkv, hd = 512, 128, 28, 4, 128
    m = C // P
    cfg = ModelConfig(n_layers=1, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=hd, chunk_size=C, page_size=P,
                      retrieval_budget=3 * P, attention_mode=["topk"])
    g = torch.Generator(device="cuda").manual_seed(seed)
    T = chunks * C
    K = torch.randn(T, Hkv, hd, device="cuda", generator=g).to(tdt)
    V = torch.randn(T, Hkv, hd, device="cuda", generator=g).to(tdt)
    Q = [torch.randn(C, Hq, hd, device="cuda", generator=g).to(tdt) for _ in range(chunks)]
    DO = [torch.randn(C, Hq, hd, device="cuda", generator=g).to(tdt) for _ in range(chunks)]
    plans = [ShardPlan(r, world, Hkv, Hq, mode) for r in range(world)]
    caches = [p.make_cache(cfg, dtype=dtype, max_tokens=T) for p in plans]
    R = plans[0].range_world
    outs, lses, sels = [[None] * chunks for _ in range(world)], [[None] * chunks for _ in range(world)], \
        [[None] * chunks for _ in range(world)]
    full_lists = []
    for i in range(chunks):
        ks, ke = i * C, (i + 1) * C
        n_cand = i * m
        # selection: partial votes of each rank's groups, reduced over the ranks of a page range
        lists_by_rank = []
        if n_cand > 0:
            parts = []
            for p, c in zip(plans, caches):
                from paper_2602_02108_b200.sharding import score_pages_partial
                parts.append(score_pages_partial(c, 0, p.kv.shard_q(Q[i]), n_cand))
            for p in plans:
                vote = fixed_order_sum(torch.cat([parts[r] for r in p.kv_ranks()]).contiguous())
                lists_by_rank.append(A.select_topk_rows(caches[p.rank], vote, cfg.budget_pages()).lists())
            assert all(l == lists_by_rank[0] for l in lists_by_rank)
        else:
            lists_by_rank = [[[] for _ in range(m)] for _ in plans]
        full_lists.append(lists_by_rank[0])
        parts_o = [None] * world
        for p, c in zip(plans, caches):
            kl, vl = p.kv.shard_kv(K[ks:ke]), p.kv.shard_kv(V[ks:ke])
            c.append_chunk(0, kl, vl)
            sel = A.Selection.from_lists(c, lists_by_rank[p.rank])
            sub = sel.filter_owned() if R > 1 else sel
            sels[p.rank][i] = sub
            parts_o[p.rank] = A.attn_forward(c.cfg, p.kv.shard_q(Q[i]), c, 0, sub, kl, vl,
                                             past_only=p.range_idx != 0)
        for p in plans:
            rr = p.range_ranks()
            o, l = lse_merge(torch.stack([parts_o[r].out for r in rr]), torch.stack([parts_o[r].lse for r in rr]))
            outs[p.rank][i], lses[p.rank][i] = o, l
    grads = [[None] * chunks for _ in range(world)]
    for i in reversed(range(chunks)):
        ks, ke = i * C, (i + 1) * C
        own = list(range(i * m, (i + 1) * m))
        part_g = [None] * world
        for p, c in zip(plans, caches):
            kl, vl = p.kv.shard_kv(K[ks:ke]), p.kv.shard_kv(V[ks:ke])
            saved = A.AttnSaved(outs[p.rank][i], lses[p.rank][i], sels[p.rank][i])
            gr = A.attn_backward(c.cfg, p.kv.shard_q(DO[i]), p.kv.shard_q(Q[i]), c, 0, kl, vl, saved,
                                 past_only=p.range_idx != 0)
            c.accumulate_grad_pages(0, own, gr.dk_cur, gr.dv_cur)
            part_g[p.rank] = (gr.dq.clone(), gr.dk_cur.clone(), gr.dv_cur.clone())
        for p in plans:
            rr = p.range_ranks()
            red = []
            for j in range(3):
                st = torch.stack([part_g[r][j] for r in rr])
                red.append(fixed_order_sum(st.reshape(len(rr), 1, -1)).reshape(st.shape[1:]))
            grads[p.rank][i] = red
    torch.cuda.synchronize()
    for c in caches:
        c.check_device_errors()
    return plans, caches, outs, lses, grads, full_lists


@pytest.mark.parametrize("world,mode", [(8, "auto"), (2, "range"), (4, "2x2")])
def test_composed_split_matches_unsplit(world, mode):
    plans1, caches1, outs1, lses1, grads1, lists1 = _run(1, "auto", "bf16")
    plans, caches, outs, lses, grads, lists = _run(world, mode, "bf16")
    assert lists == lists1  # the selection does not depend on the split
    chunks = len(outs1[0])
    n_pages = caches1[0].n_pages(0)
    gp_full = caches1[0].gather_grad_pages(0, list(range(n_pages - 4)))
    for p, c in zip(plans, caches):
        a, b = p.kv.q_range
        ka, kb = p.kv.kv_range
        for i in range(chunks):
            assert _rel(outs[p.rank][i].float(), outs1[0][i][:, a:b].float()) < 2e-2
            assert _rel(lses[p.rank][i], lses1[0][i][:, a:b]) < 2e-2
            assert _rel(grads[p.rank][i][0], grads1[0][i][0][:, a:b]) < 2e-2
            assert _rel(grads[p.rank][i][1], grads1[0][i][1][:, ka:kb]) < 2e-2
            assert _rel(grads[p.rank][i][2], grads1[0][i][2][:, ka:kb]) < 2e-2
        # the gradient pages this rank owns equal the unsplit layer's; it stores no other page
        owned = [x for x in range(n_pages - 4) if c.owns(x)]
        gp = c.gather_grad_pages(0, owned)
        idx = torch.tensor(owned, device="cuda")
        P = c.cfg.page_size
        want_k = gp_full.k.view(-1, P, *gp_full.k.shape[1:])[idx].reshape(-1, *gp_full.k.shape[1:])[:, ka:kb]
        want_v = gp_full.v.view(-1, P, *gp_full.v.shape[1:])[idx].reshape(-1, *gp_full.v.shape[1:])[:, ka:kb]
        assert _rel(gp.k, want_k) < 2e-2 and _rel(gp.v, want_v) < 2e-2
        slots = c.device_slots(0)
        R = p.range_world
        assert all((slots[x, 0] >= 0) == c.owns(x) for x in range(n_pages))
        assert int((slots[:, 0] >= 0).sum()) == (n_pages + R - 1 - p.range_idx) // R
        if R > 1:
            from paper_2602_02108_b200.errors import ResidencyError
            remote = next(x for x in range(n_pages) if not c.owns(x))
            with pytest.raises(ResidencyError):
                c.gather_pages(0, [remote])


def test_owned_pool_is_one_over_r_of_the_pages():
    """Per-rank HBM: a page-range shard's K/V and gradient pools are sized to its share of the pages,
    and its K_avg (scoring metadata) still covers every page, bit-equal to the unsplit pool's."""
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    cfg = ModelConfig(n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=128, chunk_size=512, page_size=128,
                      retrieval_budget=256, attention_mode=["topk"])
    T = 8 * 512
    g = torch.Generator(device="cuda").manual_seed(1)
    k = torch.randn(T, 2, 128, device="cuda", generator=g).bfloat16()
    v = torch.randn(T, 2, 128, device="cuda", generator=g).bfloat16()
    full = PagedCache(cfg, dtype="bf16", max_tokens=T)
    full.append_chunk(0, k, v)
    free0 = torch.cuda.mem_get_info()[0]
    shards = [PagedCache(cfg, dtype="bf16", max_tokens=T, page_owner=(4, r)) for r in range(4)]
    used = (free0 - torch.cuda.mem_get_info()[0]) / 4
    for s in shards:
        s.append_chunk(0, k, v)
    n = T // 128
    page_bytes = 128 * 2 * 128 * (2 * 2 + 2 * 4)  # K, V bf16 + dK, dV fp32
    assert used < 0.3 * n * page_bytes + (64 << 20)
    for r, s in enumerate(shards):
        assert s.page_table(0).tolist() == full.page_table(0).tolist()  # reference arena ids unchanged
        assert torch.equal(s.page_mean_keys(0), full.page_mean_keys(0))
        assert [s.tier(0, x) for x in range(n)] == [0 if x % 4 == r else 2 for x in range(n)]
        got = s.gather_pages(0, [x for x in range(n) if x % 4 == r])
        want = full.gather_pages(0, [x for x in range(n) if x % 4 == r])
        assert torch.equal(got.k, want.k) and torch.equal(got.v, want.v)
