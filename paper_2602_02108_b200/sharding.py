"""Sharding of the hot path across the GPUs of one node.

KV-head-group sharding (KVGroupShard) and, when groups run out (Qwen2.5-7B has 4 groups
for 8 GPUs; c5 splits page ranges across 2/4/8 GPUs), the page-range split
(PageRangeShard) with an exact LSE / output merge.

Attention forward / backward and the gradient pool of different KV groups touch
disjoint K/V/dK/dV head slices and disjoint q-heads, so a rank that owns a
contiguous range of KV groups runs them with NO collective: its PagedCache holds
only its heads (same page table on every rank, since every rank appends the same
tokens). The one exchange is the page vote: score_pages sums over ALL q-heads
(attention.hpp:44-64). Each rank computes per-group partial votes
[G_local, m, n]; an all-gather in global group order followed by a sum in that
fixed order gives every rank — and the 1-GPU path, which reduces the same
per-group partials in the same order — the identical vote, hence identical
top-k selections.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from ._lib import call
from .config import ModelConfig


@dataclass
class KVGroupShard:
    rank: int
    world: int
    n_kv_heads: int
    n_q_heads: int

    def __post_init__(self):
        if self.world < 1 or self.n_kv_heads % self.world:
            raise ValueError(f"{self.n_kv_heads} KV groups cannot be split over {self.world} ranks "
                             "(the page-range split is needed for that)")

    @property
    def kv_local(self) -> int:
        return self.n_kv_heads // self.world

    @property
    def kv_range(self) -> tuple[int, int]:
        return self.rank * self.kv_local, (self.rank + 1) * self.kv_local

    @property
    def q_range(self) -> tuple[int, int]:
        g = self.n_q_heads // self.n_kv_heads
        a, b = self.kv_range
        return a * g, b * g

    def local_config(self, cfg: ModelConfig) -> ModelConfig:
        return cfg.replace(n_kv_heads=self.kv_local, n_q_heads=self.kv_local * (cfg.n_q_heads // cfg.n_kv_heads))

    def shard_q(self, x: torch.Tensor) -> torch.Tensor:   # [tokens, Hq, hd] -> local heads
        a, b = self.q_range
        return x[:, a:b].contiguous()

    def shard_kv(self, x: torch.Tensor) -> torch.Tensor:  # [tokens, Hkv, hd] -> local groups
        a, b = self.kv_range
        return x[:, a:b].contiguous()


class OombComm:
    """liboomb_comm.so: an NCCL communicator with the path's deterministic exchange steps
    (include/oomb_comm.h). Rank 0 creates the NCCL id; the process group broadcasts it."""

    def __init__(self, rank: int, world: int, device: int, uid: bytes):
        from ._lib import comm_call
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        comm_call("oomb_comm_init", buf, rank, world, device, C.byref(h))
        self.handle, self.rank, self.world = h, rank, world

    @staticmethod
    def unique_id() -> bytes:
        from ._lib import comm_call
        buf = (C.c_uint8 * 128)()
        comm_call("oomb_comm_get_unique_id", buf)
        return bytes(buf)

    @classmethod
    def from_process_group(cls, group=None, device: int | None = None) -> "OombComm":
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        return cls(rank, world, torch.cuda.current_device() if device is None else device, obj[0])

    def close(self):
        if getattr(self, "handle", None):
            from ._lib import comm_lib
            comm_lib().oomb_comm_destroy(self.handle)
            self.handle = None

    __del__ = close

    def vote_allgather(self, partials_local: torch.Tensor, stream=None, out: torch.Tensor | None = None) -> torch.Tensor:
        """[G_local, m, n] partial votes -> [m, n] summed over all ranks' groups in global order."""
        from ._lib import comm_call
        from .paged_kv import stream_handle
        g, m, n = partials_local.shape
        p = partials_local.contiguous()
        vote = torch.empty((m, n), dtype=torch.float32, device=p.device) if out is None else out
        comm_call("oomb_vote_allgather", self.handle, C.c_void_p(p.data_ptr()), g, m, n, C.c_void_p(vote.data_ptr()),
                  stream_handle(stream))
        return vote

    def lse_merge_allgather(self, o_part: torch.Tensor, lse_part: torch.Tensor, stream=None):
        """partial (O [C, H, hd], LSE [C, H]) of this rank -> the exact merge over all ranks."""
        from ._lib import comm_call
        from .paged_kv import stream_handle
        c, h, hd = o_part.shape
        o, l = o_part.contiguous(), lse_part.contiguous()
        out, lse = torch.empty_like(o), torch.empty_like(l)
        comm_call("oomb_lse_merge_allgather", self.handle, C.c_void_p(o.data_ptr()), C.c_void_p(l.data_ptr()), c * h,
                  hd, 1 if o.dtype == torch.bfloat16 else 0, C.c_void_p(out.data_ptr()), C.c_void_p(lse.data_ptr()),
                  stream_handle(stream))
        return out, lse

    def dq_reduce(self, dq_part: torch.Tensor, stream=None) -> torch.Tensor:
        """sum of every rank's partial dQ in rank order (fp32)."""
        from ._lib import comm_call
        from .paged_kv import stream_handle
        p = dq_part.contiguous()
        out = torch.empty_like(p)
        comm_call("oomb_dq_reduce", self.handle, C.c_void_p(p.data_ptr()), p.numel(), C.c_void_p(out.data_ptr()),
                  stream_handle(stream))
        return out


def fixed_order_sum(parts: torch.Tensor) -> torch.Tensor:
    """vote = ((p_0 + p_1) + p_2) + ... over the group axis: on CUDA the library's
    vote_reduce kernel, elsewhere the same fp32 additions in the same order."""
    g, m, n = parts.shape
    if parts.is_cuda:
        from .paged_kv import stream_handle
        vote = torch.empty((m, n), dtype=torch.float32, device=parts.device)
        call("oomb_vote_reduce", C.c_void_p(parts.data_ptr()), g, m, n, C.c_void_p(vote.data_ptr()),
             stream_handle(None))
        return vote
    out = parts[0].clone()
    for i in range(1, g):
        out += parts[i]
    return out


def combine_votes(partials_local: torch.Tensor, group=None, comm: OombComm | None = None) -> torch.Tensor:
    """All-gather [G_local, m, n] partial votes over the process group (global group
    order = rank order) and reduce them in that fixed order -> [m, n] vote.
    With `comm` the exchange runs in liboomb_comm.so (NCCL) instead of torch.distributed."""
    if comm is not None:
        return comm.vote_allgather(partials_local)
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return fixed_order_sum(partials_local)
    g, m, n = partials_local.shape
    gathered = torch.empty((world * g, m, n), dtype=partials_local.dtype, device=partials_local.device)
    dist.all_gather_into_tensor(gathered, partials_local.contiguous(), group=group)
    return fixed_order_sum(gathered)


def score_pages_partial(cache, layer: int, q_local: torch.Tensor, n_candidates: int, stream=None) -> torch.Tensor:
    """Per-local-group partial votes [G_local, m, n] from the cache's K_avg."""
    from .paged_kv import _ptr, stream_handle
    cfg = cache.cfg
    q_local = cache._dev(q_local)
    m = (q_local.shape[0] + cfg.page_size - 1) // cfg.page_size
    n = min(n_candidates, cache.n_pages(layer))
    parts = torch.empty((cfg.n_kv_heads, m, max(n, 1)), dtype=torch.float32, device=cache.device)
    call("oomb_score_pages_partial", cache.handle, layer, _ptr(q_local), q_local.shape[0], n, _ptr(parts),
         stream_handle(stream))
    return parts[:, :, :n]


def select_pages_topk_sharded(cache, layer: int, q_local: torch.Tensor, n_candidates: int, group=None,
                              out=None, comm: OombComm | None = None):
    """chunk_trainer.hpp:305-311 on a KV-group shard: partial votes -> all-gather ->
    fixed-order sum -> top-k per query page. Identical ids on every rank."""
    from . import attention as A
    parts = score_pages_partial(cache, layer, q_local, n_candidates)
    vote = combine_votes(parts.contiguous(), group, comm)
    sel = A.select_topk_rows(cache, vote, cache.cfg.budget_pages()) if out is None else out
    if out is not None:
        from .paged_kv import _ptr, stream_handle
        call("oomb_select_topk", out.handle, _ptr(vote), vote.shape[0], vote.shape[1], cache.cfg.budget_pages(),
             stream_handle(None))
    sel.vote = vote
    return sel


# ---------------------------------------------------------------------------
# Page-range split (SURVEY §8e "page-range split", c5)
# ---------------------------------------------------------------------------
@dataclass
class PageRangeShard:
    """Rank r of R owns the pages with id % R == r (interleaved ranges keep every rank's share
    of a growing sequence balanced at every chunk) and attends, for every query page, the
    selected pages it owns, in list order. Rank 0 also owns the chunk's own causal keys.

    forward : partial (O_r, LSE_r) -> all-gather in rank order -> exact merge
              LSE = ln sum_r e^{LSE_r}, O = sum_r e^{LSE_r - LSE} O_r   (oomb_lse_merge)
    backward: with the merged (O, LSE) every rank's dK/dV for its own pages are exact and local;
              the partial dQ are all-gathered and summed in rank order (deterministic, equal on
              every rank); dk_cur / dv_cur come from rank 0 (the other ranks' are zero).
    """
    rank: int
    world: int

    def owns(self, page: int) -> bool:
        return page % self.world == self.rank

    def split_lists(self, lists) -> list[list[int]]:
        return [[p for p in l if self.owns(p)] for l in lists]

    @property
    def past_only(self) -> bool:
        return self.rank != 0


def lse_merge(o_parts: torch.Tensor, lse_parts: torch.Tensor):
    """o_parts [R, C, H, hd] (bf16 or fp32), lse_parts [R, C, H] fp32 -> (O [C, H, hd], LSE [C, H])."""
    from .paged_kv import stream_handle
    r, c, h, hd = o_parts.shape
    out = torch.empty((c, h, hd), dtype=o_parts.dtype, device=o_parts.device)
    lse = torch.empty((c, h), dtype=torch.float32, device=o_parts.device)
    dtype = 1 if o_parts.dtype == torch.bfloat16 else 0
    call("oomb_lse_merge", C.c_void_p(o_parts.contiguous().data_ptr()), C.c_void_p(lse_parts.contiguous().data_ptr()),
         r, c * h, hd, dtype, C.c_void_p(out.data_ptr()), C.c_void_p(lse.data_ptr()), stream_handle(None))
    return out, lse


def _gather(x: torch.Tensor, group=None) -> torch.Tensor:
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return x.unsqueeze(0)
    out = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
    dist.all_gather_into_tensor(out, x.contiguous(), group=group)
    return out


def range_forward(shard: PageRangeShard, cfg, q, cache, layer, selected_lists, k_cur, v_cur, group=None,
                  comm: OombComm | None = None):
    """attn_forward on a page-range shard + the collective merge; returns the merged AttnSaved
    (out, lse) and this rank's sub-selection (for the backward)."""
    from . import attention as A
    sub = A.Selection.from_lists(cache, shard.split_lists(selected_lists))
    part = A.attn_forward(cfg, q, cache, layer, sub, k_cur, v_cur, past_only=shard.past_only)
    if comm is not None:
        out, lse = comm.lse_merge_allgather(part.out, part.lse)
    else:
        out, lse = lse_merge(_gather(part.out, group), _gather(part.lse, group))
    return A.AttnSaved(out, lse, sub), sub


def range_backward(shard: PageRangeShard, cfg, dout, q, cache, layer, k_cur, v_cur, saved, group=None,
                   comm: OombComm | None = None):
    """attn_backward on a page-range shard with the merged (O, LSE); dQ summed over ranks in rank
    order, dk_cur / dv_cur from rank 0. The rank's own pages' dK/dV land in its gradient pool."""
    from . import attention as A
    g = A.attn_backward(cfg, dout, q, cache, layer, k_cur, v_cur, saved, past_only=shard.past_only)
    if comm is not None:
        dq = comm.dq_reduce(g.dq)
    else:
        dq_parts = _gather(g.dq, group)
        dq = fixed_order_sum(dq_parts.reshape(dq_parts.shape[0], 1, -1)).reshape(g.dq.shape)
    dk = _gather(g.dk_cur, group)[0].clone()
    dv = _gather(g.dv_cur, group)[0].clone()
    return A.AttnGrads(dq, dk, dv)
