"""Composed KV-group x page-range split (BASELINE configs[3]: Qwen's 4 KV groups on
8 GPUs = 4 KV shards x 2 page ranges) — host logic over gloo, no GPU.

World 4 over 2 KV groups gives 2 x 2: each rank computes, for ITS KV group and ITS pages
(id % 2 == range_idx), the partial attention of a small layer in float64 numpy (rank 0 of each
range group also attends the chunk's own keys, like OOMB_ATTN_PAST_ONLY elsewhere). The vote is
exchanged over the ranks holding the same page range, the (O, LSE) merge and the dQ reduction
over the ranks holding the same KV group, with the proportional exchanges of sharding.TorchComm
(the algorithms of liboomb_comm.so). Checked: the merged outputs equal the unsplit softmax
attention, the ordered reduction equals the rank-ordered sum bitwise on every rank, and the vote
equals the 1-GPU fixed-order reduction bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_02108_b200.sharding import (ShardPlan, TorchComm, comm_bytes, fixed_order_sum,
                                            lse_merge_torch)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plan_geometry():
    # Qwen2.5-7B: 4 KV groups
    assert [(ShardPlan(0, w, 4, 28).kv_world, ShardPlan(0, w, 4, 28).range_world) for w in (1, 2, 4, 8)] == \
        [(1, 1), (2, 1), (4, 1), (4, 2)]
    # Llama-3-8B c5: page ranges across 2/4/8 GPUs
    assert [ShardPlan(0, w, 8, 32, "range").range_world for w in (2, 4, 8)] == [2, 4, 8]
    p = ShardPlan(5, 8, 4, 28)
    assert (p.kv_idx, p.range_idx) == (2, 1)
    assert p.kv_ranks() == [1, 3, 5, 7] and p.range_ranks() == [4, 5]
    assert p.kv.kv_range == (2, 3) and p.kv.q_range == (14, 21)
    assert p.page_owner() == (2, 1)
    # every (rank) is exactly one (kv_idx, range_idx)
    cells = {(ShardPlan(r, 8, 4, 28).kv_idx, ShardPlan(r, 8, 4, 28).range_idx) for r in range(8)}
    assert len(cells) == 8
    with pytest.raises(ValueError):
        ShardPlan(0, 8, 4, 28, "kv")


def test_comm_bytes_are_proportional():
    t = 4096 * 28 * 128  # dQ of one chunk of Qwen, elements
    for w in (2, 4, 8):
        s_ag, _ = comm_bytes(0, w, t, 4)
        s_rs, r_rs = comm_bytes(1, w, t, 4)
        assert s_ag == (w - 1) * t * 4
        assert s_rs <= 2 * t * 4 and r_rs <= 2 * t * 4
        assert s_rs == pytest.approx(2 * t * 4 * (w - 1) / w, rel=1e-6)


def _attn_partial(q, k, v, keys):
    """float64 softmax attention of q [T, H, d] over the key rows `keys` (shared by the heads)."""
    if len(keys) == 0:
        return np.zeros(q.shape), np.full(q.shape[:2], -np.inf)
    s = np.einsum("thd,kd->thk", q, k[keys])
    mx = s.max(axis=2)
    p = np.exp(s - mx[..., None])
    l = p.sum(axis=2)
    return np.einsum("thk,kd->thd", p, v[keys]) / l[..., None], mx + np.log(l)


def _worker(rank, world, port, data, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, k, v, P, n_past, own = data["q"], data["k"], data["v"], data["P"], data["n_past"], data["own"]
        Hkv = k.shape[1]
        plan = ShardPlan(rank, world, Hkv, q.shape[1])
        kv_g, rg = plan.new_groups()
        kv_comm, range_comm = TorchComm(kv_g), TorchComm(rg)
        a, b = plan.kv.q_range
        g = plan.kv.kv_range[0]
        sh = plan.pages
        # attention of this rank's heads over its owned pages (+ own keys on range rank 0)
        keys = [t for t in range(n_past * P) if sh.owns(t // P)]
        if not sh.past_only:
            keys += list(range(n_past * P, n_past * P + own))
        o, lse = _attn_partial(q[:, a:b], k[:, g], v[:, g], keys)
        mo, ml = range_comm.lse_merge(torch.from_numpy(o).float(), torch.from_numpy(lse).float())
        # a partial "dQ" to reduce in rank order
        dq = torch.from_numpy(data["dq_parts"][rank]).float()
        red = range_comm.allreduce_ordered(dq)
        # votes of this rank's groups, exchanged over the ranks holding the same page range
        vote = kv_comm.vote_allgather(torch.from_numpy(data["votes"][plan.kv_idx:plan.kv_idx + 1]).float())
        result[rank] = dict(out=mo.numpy(), lse=ml.numpy(), red=red.numpy(), vote=vote.numpy(),
                            sent=range_comm.bytes_sent)
    finally:
        dist.destroy_process_group()


def test_composed_split_world4_over_gloo():
    rng = np.random.default_rng(7)
    P, n_past, own, Hkv, G, d = 4, 9, 6, 2, 3, 8
    T = n_past * P + own
    k = rng.standard_normal((T, Hkv, d)) * 0.7
    v = rng.standard_normal((T, Hkv, d))
    q = rng.standard_normal((own, Hkv * G, d)) * 0.7
    world = 4
    data = dict(q=q, k=k, v=v, P=P, n_past=n_past, own=own,
                dq_parts=[rng.standard_normal((own, G, d)).astype(np.float32) for _ in range(world)],
                votes=rng.random((Hkv, 3, 11)).astype(np.float32))
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), data, result), nprocs=world, join=True)
    for r in range(world):
        plan = ShardPlan(r, world, Hkv, Hkv * G)
        a, b = plan.kv.q_range
        g = plan.kv.kv_range[0]
        want_o, want_l = _attn_partial(q[:, a:b], k[:, g], v[:, g], list(range(T)))
        got = result[r]
        assert np.allclose(got["out"], want_o, rtol=1e-5, atol=1e-5)
        assert np.allclose(got["lse"], want_l, rtol=1e-5, atol=1e-5)
        # ordered reduction: bitwise the rank-ordered fp32 sum of the range group's parts
        parts = torch.stack([torch.from_numpy(data["dq_parts"][x]) for x in plan.range_ranks()])
        want = fixed_order_sum(parts.reshape(parts.shape[0], 1, -1)).reshape(parts.shape[1:])
        assert got["red"].tobytes() == want.numpy().tobytes()
        # vote: the 1-GPU fixed-order reduction of all groups' partials
        assert got["vote"].tobytes() == fixed_order_sum(torch.from_numpy(data["votes"])).numpy().tobytes()
        assert got["sent"] > 0
    # the two ranks of a range group hold identical merged outputs
    for kv in range(2):
        r0, r1 = kv * 2, kv * 2 + 1
        assert result[r0]["out"].tobytes() == result[r1]["out"].tobytes()


def test_lse_merge_torch_matches_formula():
    rng = np.random.default_rng(3)
    o = torch.from_numpy(rng.standard_normal((3, 5, 4)).astype(np.float32))
    l = torch.from_numpy(rng.standard_normal((3, 5)).astype(np.float32))
    l[2, 1] = float("-inf")
    o[2, 1] = 0
    out, L = lse_merge_torch(o, l)
    m = l.max(0).values
    w = torch.exp(l - m).nan_to_num(0.0)
    want_l = m + torch.log(w.sum(0))
    assert torch.allclose(L, want_l, atol=1e-6)
    want_o = (torch.exp(l - want_l)[..., None] * o).sum(0)
    assert torch.allclose(out, want_o, atol=1e-6)
