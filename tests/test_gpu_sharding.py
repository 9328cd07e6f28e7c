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


def _rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / max(b.norm(), 1e-30))


@pytest.mark.parametrize("dtype,world", [("bf16", 2), ("bf16", 3), ("fp32", 2)])
def test_page_range_split_matches_unsplit(dtype, world):
    """Page-range split simulated on one GPU: R shards attend the pages they own
    (id % R), shard 0 also the chunk's keys; the exact LSE merge of their partial outputs and the
    rank-ordered sum of their partial dQ reproduce the unsplit layer, and the gradient pages of
    every shard's own pages equal the unsplit ones (tolerances of BASELINE north_star)."""
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200 import attention as A
    from paper_2602_02108_b200.sharding import PageRangeShard, fixed_order_sum, lse_merge
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    tol = 2e-2 if dtype == "bf16" else 1e-5
    cfg = ModelConfig(n_layers=1, n_q_heads=28, n_kv_heads=4, head_dim=128, chunk_size=512, page_size=128,
                      retrieval_budget=5 * 128, attention_mode=["topk"])
    g = torch.Generator(device="cuda").manual_seed(21 + world)
    n_past = 14
    past = torch.randn(n_past * 128, 4, 128, device="cuda", generator=g).to(tdt)
    pv = torch.randn(n_past * 128, 4, 128, device="cuda", generator=g).to(tdt)
    q = torch.randn(512, 28, 128, device="cuda", generator=g).to(tdt)
    k = torch.randn(512, 4, 128, device="cuda", generator=g).to(tdt)
    v = torch.randn(512, 4, 128, device="cuda", generator=g).to(tdt)
    do = torch.randn(512, 28, 128, device="cuda", generator=g).to(tdt)
    lists = [[0, 3, 5, 8, 13], [1, 2, 9, 11, 12], [4, 6, 7, 10, 0], [13, 12, 5]]

    def layer():
        c = PagedCache(cfg, dtype=dtype, max_tokens=8192)
        c.append_chunk(0, past, pv)
        c.append_chunk(0, k, v)
        return c

    full = layer()
    s_full = A.attn_forward(cfg, q, full, 0, lists, k, v)
    g_full = A.attn_backward(cfg, do, q, full, 0, k, v, s_full)
    gp_full = full.gather_grad_pages(0, list(range(n_past)))

    cache = layer()  # one pool stands in for the shards' pools: their pages are disjoint
    shards = [PageRangeShard(r, world) for r in range(world)]
    parts = []
    subs = []
    for sh in shards:
        sub = A.Selection.from_lists(cache, sh.split_lists(lists))
        subs.append(sub)
        parts.append(A.attn_forward(cfg, q, cache, 0, sub, k, v, past_only=sh.past_only))
    out, lse = lse_merge(torch.stack([p.out for p in parts]), torch.stack([p.lse for p in parts]))
    assert _rel(out.float(), s_full.out.float()) < tol
    assert _rel(lse, s_full.lse) < tol
    dqs, dk0, dv0 = [], None, None
    for sh, sub in zip(shards, subs):
        saved = A.AttnSaved(out, lse, sub)
        gr = A.attn_backward(cfg, do, q, cache, 0, k, v, saved, past_only=sh.past_only)
        dqs.append(gr.dq.clone())
        if sh.rank == 0:
            dk0, dv0 = gr.dk_cur.clone(), gr.dv_cur.clone()
        else:
            assert torch.count_nonzero(gr.dk_cur) == 0 and torch.count_nonzero(gr.dv_cur) == 0
    dq = fixed_order_sum(torch.stack(dqs).reshape(world, 1, -1)).reshape(g_full.dq.shape)
    assert _rel(dq, g_full.dq) < tol
    assert _rel(dk0, g_full.dk_cur) < tol and _rel(dv0, g_full.dv_cur) < tol
    gp = cache.gather_grad_pages(0, list(range(n_past)))
    assert _rel(gp.k, gp_full.k) < tol and _rel(gp.v, gp_full.v) < tol


def test_lse_merge_single_part_is_identity_and_empty_parts_vanish():
    from paper_2602_02108_b200.sharding import lse_merge
    g = torch.Generator(device="cuda").manual_seed(3)
    o = torch.randn(1, 64, 4, 128, device="cuda", generator=g)
    l = torch.randn(1, 64, 4, device="cuda", generator=g)
    out, lse = lse_merge(o, l)
    assert torch.allclose(out, o[0], rtol=1e-6, atol=1e-6) and torch.allclose(lse, l[0], rtol=1e-6, atol=1e-6)
    # a shard that attended nothing contributes lse = -inf, out = 0
    o2 = torch.stack([o[0], torch.zeros_like(o[0])])
    l2 = torch.stack([l[0], torch.full_like(l[0], float("-inf"))])
    out2, lse2 = lse_merge(o2, l2)
    assert torch.allclose(out2, o[0], rtol=1e-6, atol=1e-6) and torch.allclose(lse2, l[0], rtol=1e-6, atol=1e-6)


def test_nccl_comm_world1_exchanges_are_exact():
    """liboomb_comm.so over a real NCCL communicator (world 1 — one GPU per rank, one GPU here):
    the vote all-gather equals the fixed-order reduction bitwise, and the LSE merge and dQ reduce
    of a single rank are the identity. The same calls run unchanged at world 2..8."""
    from paper_2602_02108_b200.sharding import OombComm, fixed_order_sum
    comm = OombComm(0, 1, torch.cuda.current_device(), OombComm.unique_id())
    g = torch.Generator(device="cuda").manual_seed(21)
    parts = torch.rand(4, 32, 1000, device="cuda", generator=g)
    assert torch.equal(comm.vote_allgather(parts), fixed_order_sum(parts))
    o = torch.randn(256, 28, 128, device="cuda", generator=g).bfloat16()
    lse = torch.randn(256, 28, device="cuda", generator=g)
    out, lse2 = comm.lse_merge_allgather(o, lse)
    assert torch.equal(out, o) and torch.equal(lse2, lse)
    dq = torch.randn(256, 28, 128, device="cuda", generator=g)
    assert torch.equal(comm.dq_reduce(dq), dq)
    comm.close()


def test_bench_kv_shard_mode_world1():
    """bench.py --shard kv (one sequence split by KV-head group, votes all-gathered over NCCL)
    runs end to end and reports strong scaling; world 1 here, the same code at world 2 / 4."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--shard", "kv", "--config", "c3",
                        "--tokens", str(16 * 4096), "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["scaling"] == "strong" and line["value"] > 0 and line["gpu_launches"] > 0
    assert "KV-head group" in line["config"]["parallelism"] and line["sharding"]["kv_world"] == 1
