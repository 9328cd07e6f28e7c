"""Host logic of the KV-group sharded path on CPU with world_size-2 gloo.

Each rank computes, with the CPU oracle (the checker), the partial votes of ITS
KV groups only; combine_votes all-gathers them in global group order and sums
in that fixed order. Both ranks must end with the bitwise-identical vote, equal
to the single-process reduction of the same per-group partials, and within
fp32 rounding of the reference's all-head vote; the top-k ids must agree."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import Cfg, Port, det_normal
from paper_2602_02108_b200.sharding import KVGroupShard, combine_votes, fixed_order_sum


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def group_partials(q, kav, cfg, groups):
    """Per-group partial votes from the oracle: score_pages restricted to a group's heads."""
    G = cfg.n_q_heads // cfg.n_kv_heads
    out = []
    for g in groups:
        c = Cfg(n_layers=1, n_q_heads=G, n_kv_heads=1, head_dim=cfg.head_dim, chunk_size=cfg.chunk_size,
                page_size=cfg.page_size, retrieval_budget=cfg.retrieval_budget)
        out.append(Port(c, 4).score_pages(q[:, g * G:(g + 1) * G], kav[:, g:g + 1]))
    return torch.from_numpy(np.stack(out))


def _worker(rank, world, port, q, kav, cfg_d, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = Cfg(**cfg_d)
    sh = KVGroupShard(rank, world, cfg.n_kv_heads, cfg.n_q_heads)
    a, b = sh.kv_range
    parts = group_partials(q, kav, cfg, range(a, b))
    vote = combine_votes(parts)
    result[rank] = vote.numpy().copy()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_vote_allgather_fixed_order(world):
    cfg = Cfg(n_layers=1, n_q_heads=8, n_kv_heads=4, head_dim=16, chunk_size=32, page_size=8,
              retrieval_budget=24)
    q = det_normal(5, (32, 8, 16))
    kav = det_normal(6, (20, 4, 16))
    mgr = mp.Manager()
    result = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, q, kav, cfg.__dict__, result), nprocs=world, join=True)
    votes = [result[r] for r in range(world)]
    for v in votes[1:]:
        assert v.tobytes() == votes[0].tobytes()          # identical on every rank
    single = fixed_order_sum(group_partials(q, kav, cfg, range(4))).numpy()
    assert single.tobytes() == votes[0].tobytes()         # == the 1-GPU reduction order
    ref = Port(cfg, 4).score_pages(q, kav)                 # the reference's all-head vote
    assert np.max(np.abs(single - ref) / np.maximum(np.abs(ref), 1e-30)) < 1e-5
    for i in range(ref.shape[0]):
        want = Port.select_topk(ref[i].astype(np.float64), 3).tolist()
        row = np.sort(ref[i])[::-1]
        if (row[2] - row[3]) / row[2] > 1e-4:
            assert Port.select_topk(single[i].astype(np.float64), 3).tolist() == want


def test_shard_geometry():
    sh = KVGroupShard(1, 2, 4, 28)
    assert sh.kv_range == (2, 4) and sh.q_range == (14, 28)
    from paper_2602_02108_b200 import ModelConfig
    lc = sh.local_config(ModelConfig(n_q_heads=28, n_kv_heads=4, head_dim=128, chunk_size=4096, page_size=128,
                                     retrieval_budget=8192))
    assert (lc.n_q_heads, lc.n_kv_heads) == (14, 2)
    with pytest.raises(ValueError):
        KVGroupShard(0, 8, 4, 28)
    x = torch.arange(2 * 28 * 3).reshape(2, 28, 3)
    assert torch.equal(sh.shard_q(x), x[:, 14:28])


# ---------------------------------------------------------------------------
# page-range split: ownership partition and the exact LSE merge (host math, gloo world 2)
# ---------------------------------------------------------------------------
def test_page_range_partition_is_exact():
    from paper_2602_02108_b200.sharding import PageRangeShard
    lists = [[0, 3, 5, 8, 13], [], [4, 6, 7, 10, 1], [13, 12]]
    for world in (1, 2, 3, 8):
        shards = [PageRangeShard(r, world) for r in range(world)]
        for i, l in enumerate(lists):
            parts = [sh.split_lists(lists)[i] for sh in shards]
            assert sorted(x for p in parts for x in p) == sorted(l)          # every page exactly once
            for p in parts:                                                   # list order kept
                assert p == [x for x in l if x in p]
        assert [sh.past_only for sh in shards] == [False] + [True] * (world - 1)


def _merge_np(o_parts, lse_parts):
    m = np.max(lse_parts, axis=0)
    w = np.where(np.isneginf(lse_parts), 0.0, np.exp(lse_parts - m))
    L = m + np.log(w.sum(axis=0))
    return (np.exp(lse_parts - L)[..., None] * o_parts).sum(axis=0), L


def _range_worker(rank, world, port, logits, vals, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_02108_b200.sharding import PageRangeShard
        sh = PageRangeShard(rank, world)
        keys = [k for k in range(logits.shape[1]) if sh.owns(k // 4)]  # 4 keys per "page"
        s = logits[:, keys]
        mx = s.max(axis=1)
        p = np.exp(s - mx[:, None])
        o = (p @ vals[keys]) / p.sum(axis=1)[:, None]
        lse = mx + np.log(p.sum(axis=1))
        go = [torch.zeros(o.shape, dtype=torch.float64) for _ in range(world)]
        gl = [torch.zeros(lse.shape, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(go, torch.from_numpy(o))
        dist.all_gather(gl, torch.from_numpy(lse))
        out, L = _merge_np(np.stack([x.numpy() for x in go]), np.stack([x.numpy() for x in gl]))
        result[rank] = (out, L)
    finally:
        dist.destroy_process_group()


def test_page_range_merge_over_gloo_equals_full_softmax():
    rng = np.random.default_rng(0)
    logits = rng.standard_normal((16, 40)) * 3
    vals = rng.standard_normal((40, 8))
    full_p = np.exp(logits - logits.max(axis=1, keepdims=True))
    full_o = (full_p @ vals) / full_p.sum(axis=1)[:, None]
    full_l = logits.max(axis=1) + np.log(full_p.sum(axis=1))
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_range_worker, args=(2, _free_port(), logits, vals, result), nprocs=2, join=True)
    for r in range(2):
        out, L = result[r]
        assert np.allclose(out, full_o, rtol=1e-12, atol=1e-12) and np.allclose(L, full_l, rtol=1e-12, atol=1e-12)
    assert np.array_equal(result[0][0], result[1][0])
