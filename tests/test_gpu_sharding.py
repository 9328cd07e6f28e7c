"""KV-group sharding on one GPU: two "ranks" (two caches holding half of the KV
groups each) reproduce the unsharded layer bitwise — the vote from the
per-group partials reduced in global group order, the top-k ids, and every
attention output / gradient of their heads."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_sharded_equals_unsharded_bitwise():
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200 import attention as A
    from paper_2602_02108_b200.sharding import KVGroupShard, fixed_order_sum, score_pages_partial
    cfg = ModelConfig(n_layers=1, n_q_heads=28, n_kv_heads=4, head_dim=128, chunk_size=512, page_size=128,
                      retrieval_budget=3 * 128, attention_mode=["topk"])
    g = torch.Generator(device="cuda").manual_seed(11)
    past = torch.randn(12 * 128, 4, 128, device="cuda", generator=g).bfloat16()
    pv = torch.randn(12 * 128, 4, 128, device="cuda", generator=g).bfloat16()
    q = torch.randn(512, 28, 128, device="cuda", generator=g).bfloat16()
    k = torch.randn(512, 4, 128, device="cuda", generator=g).bfloat16()
    v = torch.randn(512, 4, 128, device="cuda", generator=g).bfloat16()
    do = torch.randn(512, 28, 128, device="cuda", generator=g).bfloat16()

    full = PagedCache(cfg, dtype="bf16", max_tokens=8192)
    full.append_chunk(0, past, pv)
    sel_full = A.select_pages_topk(full, 0, q, 12)
    ref_vote = sel_full.vote.clone()

    shards = [KVGroupShard(r, 2, 4, 28) for r in range(2)]
    caches = []
    parts = []
    for sh in shards:
        c = PagedCache(sh.local_config(cfg), dtype="bf16", max_tokens=8192)
        c.append_chunk(0, sh.shard_kv(past), sh.shard_kv(pv))
        parts.append(score_pages_partial(c, 0, sh.shard_q(q), 12))
        caches.append(c)
    vote = fixed_order_sum(torch.cat(parts).contiguous())  # == all-gather in rank order + fixed-order sum
    torch.cuda.synchronize()
    assert torch.equal(vote, ref_vote)
    lists = A.select_topk_rows(caches[0], vote, cfg.budget_pages()).lists()
    assert lists == sel_full.lists()

    full.append_chunk(0, k, v)
    s_full = A.attn_forward(cfg, q, full, 0, lists, k, v)
    g_full = A.attn_backward(cfg, do, q, full, 0, k, v, s_full)
    gp_full = full.gather_grad_pages(0, list(range(12)))
    for sh, c in zip(shards, caches):
        lc = c.cfg
        c.append_chunk(0, sh.shard_kv(k), sh.shard_kv(v))
        s = A.attn_forward(lc, sh.shard_q(q), c, 0, lists, sh.shard_kv(k), sh.shard_kv(v))
        gr = A.attn_backward(lc, sh.shard_q(do), sh.shard_q(q), c, 0, sh.shard_kv(k), sh.shard_kv(v), s)
        gp = c.gather_grad_pages(0, list(range(12)))
        a, b = sh.q_range
        ka, kb = sh.kv_range
        assert torch.equal(s.out, s_full.out[:, a:b]) and torch.equal(s.lse, s_full.lse[:, a:b])
        assert torch.equal(gr.dq, g_full.dq[:, a:b])
        assert torch.equal(gr.dk_cur, g_full.dk_cur[:, ka:kb]) and torch.equal(gr.dv_cur, g_full.dv_cur[:, ka:kb])
        assert torch.equal(gp.k, gp_full.k[:, ka:kb]) and torch.equal(gp.v, gp_full.v[:, ka:kb])
