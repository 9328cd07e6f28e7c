"""KV-head-group sharding of the hot path across the GPUs of one node.

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


def combine_votes(partials_local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather [G_local, m, n] partial votes over the process group (global group
    order = rank order) and reduce them in that fixed order -> [m, n] vote."""
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
                              out=None):
    """chunk_trainer.hpp:305-311 on a KV-group shard: partial votes -> all-gather ->
    fixed-order sum -> top-k per query page. Identical ids on every rank."""
    from . import attention as A
    parts = score_pages_partial(cache, layer, q_local, n_candidates)
    vote = combine_votes(parts.contiguous(), group)
    sel = A.select_topk_rows(cache, vote, cache.cfg.budget_pages()) if out is None else out
    if out is not None:
        from .paged_kv import _ptr, stream_handle
        call("oomb_select_topk", out.handle, _ptr(vote), vote.shape[0], vote.shape[1], cache.cfg.budget_pages(),
             stream_handle(None))
    sel.vote = vote
    return sel
