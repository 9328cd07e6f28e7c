"""Sharding of the hot path across the GPUs of one node.

KV-head-group sharding (KVGroupShard) and, when groups run out (Qwen2.5-7B has 4 groups
for 8 GPUs; c5 splits page ranges across 2/4/8 GPUs), the page-range split
(PageRangeShard) with an exact LSE / output merge. ShardPlan composes the two
(world = kv_world x range_world; rank = kv_idx * range_world + range_idx) and
ShardedLayer runs one chunk of a split layer end to end: selection (vote exchange over
the ranks holding the same page range), attention over the rank's own pages, the exact
(O, LSE) merge and the ordered dQ / dk_cur / dv_cur reduction over the ranks holding the
same KV groups. The merge and reductions are proportional (oomb_comm.h: ordered
reduce-scatter by row slices + in-place all-gather of the slices, ~2x the tensor per rank)
and bitwise equal to the all-gather-then-combine versions.

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
import math
from dataclasses import dataclass, field

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

    # ---- proportional exchanges (ordered reduce-scatter by slices + all-gather of the slices)
    def allreduce_ordered(self, part: torch.Tensor, stream=None, out: torch.Tensor | None = None) -> torch.Tensor:
        """out = sum over ranks of `part` in rank order (fp32), bitwise equal to dq_reduce; out may be part."""
        from ._lib import comm_call
        from .paged_kv import stream_handle
        p = part if part.is_contiguous() else part.contiguous()
        o = p if out is None else out
        comm_call("oomb_allreduce_ordered", self.handle, C.c_void_p(p.data_ptr()), p.numel(),
                  C.c_void_p(o.data_ptr()), stream_handle(stream))
        self.bytes_sent += comm_bytes(1, self.world, p.numel(), 4)[0]
        return o

    def lse_merge(self, o_part: torch.Tensor, lse_part: torch.Tensor, stream=None, out=None, lse=None):
        """The exact (O, LSE) merge over all ranks, bitwise equal to lse_merge_allgather."""
        from ._lib import comm_call
        from .paged_kv import stream_handle
        c, h, hd = o_part.shape
        o, l = o_part.contiguous(), lse_part.contiguous()
        out = torch.empty_like(o) if out is None else out
        lse = torch.empty_like(l) if lse is None else lse
        comm_call("oomb_lse_merge_ordered", self.handle, C.c_void_p(o.data_ptr()), C.c_void_p(l.data_ptr()), c * h,
                  hd, 1 if o.dtype == torch.bfloat16 else 0, C.c_void_p(out.data_ptr()), C.c_void_p(lse.data_ptr()),
                  stream_handle(stream))
        self.bytes_sent += comm_bytes(1, self.world, c * h, hd * o.element_size() + 4)[0]
        return out, lse

    bytes_sent = 0


def comm_bytes(op: int, world: int, elems: int, elem_bytes: int) -> tuple[int, int]:
    """Per-rank (sent, received) wire bytes of one exchange of `elems` elements: op 0 = all-gather +
    local combine, op 1 = ordered reduce-scatter by slices + all-gather of the slices (oomb_comm.h).
    Pure arithmetic (the same formula as oomb_comm_bytes), usable without a GPU."""
    if world <= 1:
        return 0, 0
    t = elems * elem_bytes
    if op == 0:
        return t * (world - 1), t * (world - 1)
    chunk = (elems + world - 1) // world
    mine = min(elems, chunk) * elem_bytes
    return (t - mine) + mine * (world - 1), mine * (world - 1) + (t - mine)


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


# ---------------------------------------------------------------------------
# The same exchange steps over torch.distributed (gloo in the CPU tests; CUDA tensors are staged
# through host memory when the backend cannot carry them, e.g. several ranks sharing one GPU)
# ---------------------------------------------------------------------------
def lse_merge_torch(o_parts: torch.Tensor, lse_parts: torch.Tensor):
    """oomb_lse_merge in torch, with the kernel's fp32 operation order (parts in order)."""
    r = o_parts.shape[0]
    lp = lse_parts.float()
    m = lp[0].clone()
    for i in range(1, r):
        m = torch.maximum(m, lp[i])
    l = torch.zeros_like(m)
    for i in range(r):
        l = l + torch.where(lp[i] == float("-inf"), torch.zeros_like(m), torch.exp(lp[i] - m))
    L = torch.where(m == float("-inf"), m, m + torch.log(l))
    acc = torch.zeros(o_parts.shape[1:], dtype=torch.float32, device=o_parts.device)
    for i in range(r):
        w = torch.where(lp[i] == float("-inf"), torch.zeros_like(m), torch.exp(lp[i] - L))
        acc = acc + w[..., None] * o_parts[i].float()
    return acc.to(o_parts.dtype), L


def _on_stream(fn):
    """Run a TorchComm step with `stream` current, so the host staging of CUDA tensors is ordered
    after the work already enqueued there and its results are consumed in stream order."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *a, stream=None, **kw):
        if stream is None or not torch.cuda.is_available():
            return fn(self, *a, **kw)
        with torch.cuda.stream(stream):
            return fn(self, *a, **kw)
    return wrapper


class TorchComm:
    """Exchange steps of the sharded path over a torch.distributed group, with the algorithms of
    liboomb_comm.so: row slices exchanged all-to-all, combined in rank order by the slice's owner,
    then all-gathered. Results equal OombComm's bitwise on fp32 sums (same per-element order)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.bytes_sent = 0
        backend = dist.get_backend(group) if dist.is_initialized() else "gloo"
        self.stage_cuda = backend != "nccl"

    def _host(self, x):
        return x.cpu() if (x.is_cuda and self.stage_cuda) else x

    def _slices(self, rows):
        ch = (rows + self.world - 1) // self.world
        offs = [min(rows, s * ch) for s in range(self.world)]
        lens = [min(rows, (s + 1) * ch) - offs[s] for s in range(self.world)]
        return offs, lens

    def _exchange(self, x2):  # x2 [rows, w] -> packed [world, len(me), w]
        offs, lens = self._slices(x2.shape[0])
        me = lens[self.rank]
        out = torch.empty((self.world * me, x2.shape[1]), dtype=x2.dtype, device=x2.device)
        self.dist.all_to_all_single(out, x2.contiguous(), output_split_sizes=[me] * self.world,
                                    input_split_sizes=lens, group=self.group)
        return out.view(self.world, me, x2.shape[1]), offs, lens

    def _share(self, full, mine, offs, lens):  # all-gather of the slices into full [rows, w]
        ch = max(lens)
        pad = torch.zeros((ch, full.shape[1]), dtype=full.dtype, device=full.device)
        pad[: lens[self.rank]] = mine
        gath = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(gath, pad, group=self.group)
        for s in range(self.world):
            full[offs[s]: offs[s] + lens[s]] = gath[s][: lens[s]]

    @_on_stream
    def vote_allgather(self, partials_local: torch.Tensor, out=None) -> torch.Tensor:
        vote = combine_votes(self._host(partials_local.contiguous()), self.group)
        vote = vote.to(partials_local.device)
        if out is not None:
            out.copy_(vote)
            return out
        return vote

    @_on_stream
    def allreduce_ordered(self, part: torch.Tensor, out=None) -> torch.Tensor:
        dev = part.device
        x = self._host(part.contiguous()).reshape(-1, 1).float()
        if self.world == 1:
            res = x
        else:
            packed, offs, lens = self._exchange(x)
            acc = packed[0].clone()
            for s in range(1, self.world):
                acc = acc + packed[s]
            res = torch.empty_like(x)
            self._share(res, acc, offs, lens)
            self.bytes_sent += comm_bytes(1, self.world, x.shape[0], 4)[0]
        res = res.reshape(part.shape).to(dev)
        if out is not None:
            out.copy_(res)
            return out
        return res

    @_on_stream
    def lse_merge(self, o_part: torch.Tensor, lse_part: torch.Tensor, out=None, lse=None):
        dev = o_part.device
        c, h, hd = o_part.shape
        o2 = self._host(o_part.contiguous()).reshape(c * h, hd)
        l2 = self._host(lse_part.contiguous()).reshape(c * h, 1)
        if self.world == 1:
            mo, ml = o2, l2
        else:
            po, offs, lens = self._exchange(o2)
            pl, _, _ = self._exchange(l2)
            so, sl = lse_merge_torch(po, pl[..., 0])
            mo, ml = torch.empty_like(o2), torch.empty_like(l2)
            self._share(mo, so, offs, lens)
            self._share(ml, sl[:, None], offs, lens)
            self.bytes_sent += comm_bytes(1, self.world, c * h, hd * o2.element_size() + 4)[0]
        mo, ml = mo.reshape(c, h, hd).to(dev), ml.reshape(c, h).to(dev)
        if out is not None:
            out.copy_(mo)
            lse.copy_(ml)
            return out, lse
        return mo, ml


# ---------------------------------------------------------------------------
# Composed split: KV-head groups x page ranges (BASELINE configs[3] on 8 GPUs)
# ---------------------------------------------------------------------------
@dataclass
class ShardPlan:
    """world = kv_world x range_world ranks; rank = kv_idx * range_world + range_idx.

    mode "kv": KV-group split only (world must divide n_kv_heads); "range": page-range split only;
    "kv+range" / "auto": as many KV groups per rank as the world allows (kv_world =
    gcd(world, n_kv_heads)), the rest of the world splits page ranges; "KxR": explicit. Qwen2.5-7B (4 KV groups):
    1/2/4 GPUs -> 1/2/4 x 1, 8 GPUs -> 4 x 2. Llama-3-8B c5 (8 groups) with "range": 1 x N.

    kv_ranks(): the ranks holding the same page range (they exchange the page vote);
    range_ranks(): the ranks holding the same KV groups (they merge O/LSE and reduce dQ and the
    chunk's dK/dV)."""
    rank: int
    world: int
    n_kv_heads: int
    n_q_heads: int
    mode: str = "auto"
    kv_world: int = field(init=False)
    range_world: int = field(init=False)

    def __post_init__(self):
        if self.mode == "kv":
            if self.n_kv_heads % self.world:
                raise ValueError(f"{self.n_kv_heads} KV groups cannot be split over {self.world} ranks")
            self.kv_world, self.range_world = self.world, 1
        elif self.mode == "range":
            self.kv_world, self.range_world = 1, self.world
        elif self.mode in ("auto", "kv+range"):
            self.kv_world = math.gcd(self.world, self.n_kv_heads)
            self.range_world = self.world // self.kv_world
        elif "x" in self.mode:  # explicit "KxR"
            self.kv_world, self.range_world = (int(x) for x in self.mode.split("x"))
            if self.kv_world * self.range_world != self.world or self.n_kv_heads % self.kv_world:
                raise ValueError(f"shard mode {self.mode!r} does not fit world {self.world} / "
                                 f"{self.n_kv_heads} KV groups")
        else:
            raise ValueError(f"unknown shard mode {self.mode!r}")
        if not 0 <= self.rank < self.world:
            raise ValueError("rank out of range")

    @property
    def kv_idx(self) -> int:
        return self.rank // self.range_world

    @property
    def range_idx(self) -> int:
        return self.rank % self.range_world

    @property
    def kv(self) -> KVGroupShard:
        return KVGroupShard(self.kv_idx, self.kv_world, self.n_kv_heads, self.n_q_heads)

    @property
    def pages(self) -> "PageRangeShard":
        return PageRangeShard(self.range_idx, self.range_world)

    def kv_ranks(self) -> list[int]:
        return [k * self.range_world + self.range_idx for k in range(self.kv_world)]

    def range_ranks(self) -> list[int]:
        return [self.kv_idx * self.range_world + j for j in range(self.range_world)]

    def local_config(self, cfg: ModelConfig) -> ModelConfig:
        return self.kv.local_config(cfg)

    def page_owner(self) -> tuple[int, int] | None:
        return (self.range_world, self.range_idx) if self.range_world > 1 else None

    def make_cache(self, cfg: ModelConfig, **kw):
        """The rank's PagedCache: its KV groups' heads, and K/V + gradient storage only for the pages
        its range owns (HBM per rank = 1/range_world of the pages; K_avg kept for every page)."""
        from .paged_kv import PagedCache
        return PagedCache(self.local_config(cfg), page_owner=self.page_owner(), **kw)

    def describe(self) -> str:
        return (f"one sequence split over {self.world} GPU(s): {self.kv_world} KV-head group shard(s) x "
                f"{self.range_world} page-range shard(s)")

    def new_groups(self):
        """(kv_group, range_group) torch.distributed groups of this rank. Every rank must call this
        (new_group is collective over the world); None for a trivial (size-1) group."""
        import torch.distributed as dist
        kv_g = rg = None
        for j in range(self.range_world):  # groups of ranks sharing page range j
            ranks = [k * self.range_world + j for k in range(self.kv_world)]
            g = dist.new_group(ranks) if self.kv_world > 1 else None
            if j == self.range_idx:
                kv_g = g
        for i in range(self.kv_world):  # groups of ranks sharing KV groups i
            ranks = [i * self.range_world + j for j in range(self.range_world)]
            g = dist.new_group(ranks) if self.range_world > 1 else None
            if i == self.kv_idx:
                rg = g
        return kv_g, rg


class ShardedLayer:
    """One attention layer of ONE sequence split by a ShardPlan (chunk_trainer.hpp:292-316, 415-439,
    563-587 on a shard). Per chunk:

      select   per-group partial votes of the rank's groups -> vote exchange over kv_comm (global
               group order, the 1-GPU order) -> top-k (identical on every rank) -> the sub-selection
               of pages this rank's range owns (device filter, list order kept)
      forward  attention over the owned pages (+ the chunk's own keys on range rank 0) -> the exact
               (O, LSE) merge over range_comm
      backward attention backward with the merged (O, LSE): dK/dV of owned pages land in the
               rank's gradient pool; the dM_i read-back adds the owned pages among the chunk's own;
               then dQ and dk_cur / dv_cur are summed over range_comm in rank order.
    With range_world == 1 the comm steps vanish and the layer is the KV-group split (or, at world
    1, the unsplit layer)."""

    def __init__(self, plan: ShardPlan, cfg: ModelConfig, cache=None, kv_comm=None, range_comm=None, layer: int = 0):
        self.plan, self.cfg, self.layer = plan, cfg, layer
        self.kv_comm, self.range_comm = kv_comm, range_comm
        self.m = cfg.chunk_size // cfg.page_size
        self.cache = self.lcfg = None
        if cache is not None:
            self.attach(cache)

    def attach(self, cache):
        """Use `cache` (plan.make_cache(cfg, ...)) as this rank's pool; returns it."""
        self.cache, self.lcfg = cache, cache.cfg
        return cache

    def comm_bytes_per_chunk(self, chunk_tokens: int | None = None) -> dict:
        """Per-rank wire bytes sent per chunk by each exchange (selection vote, (O, LSE) merge, ordered
        [dq | dk_cur | dv_cur] reduction), from the exchange algorithms' formulas."""
        C = chunk_tokens or self.cfg.chunk_size
        hq, hkv, hd = self.lcfg.n_q_heads, self.lcfg.n_kv_heads, self.lcfg.head_dim
        ob = 2 if self.cache.dtype == torch.bfloat16 else 4
        out = {}
        if self.plan.range_world > 1:
            R = self.plan.range_world
            out["olse_merge_bytes"] = comm_bytes(1, R, C * hq, hd * ob + 4)[0]
            out["grad_reduce_bytes"] = comm_bytes(1, R, C * hq * hd + 2 * C * hkv * hd, 4)[0]
            out["olse_merge_bytes_allgather"] = comm_bytes(0, R, C * hq, hd * ob + 4)[0]
            out["grad_reduce_bytes_allgather"] = comm_bytes(0, R, C * hq * hd + 2 * C * hkv * hd, 4)[0]
        return out

    @property
    def split_pages(self) -> bool:
        return self.plan.range_world > 1

    def select(self, i: int, q_local, full, sub=None, vote_buf=None, parts_buf=None, stream=None):
        """Chunk i's selection into `full` (and the owned part into `sub` on a page-range shard)."""
        from . import attention as A
        from .paged_kv import _ptr, stream_handle
        cfg, cache, m = self.cfg, self.cache, self.m
        n_cand = i * m
        mode = cfg.attention_mode[self.layer % len(cfg.attention_mode)]
        if mode == "topk" and n_cand > 0:
            n = min(n_cand, cache.n_pages(self.layer))
            g = self.lcfg.n_kv_heads
            parts = (torch.empty((g, m, n), dtype=torch.float32, device=cache.device) if parts_buf is None
                     else parts_buf.reshape(-1)[: g * m * n].view(g, m, n))
            call("oomb_score_pages_partial", cache.handle, self.layer, _ptr(q_local), q_local.shape[0], n,
                 _ptr(parts), stream_handle(stream))
            vote = (torch.empty((m, n), dtype=torch.float32, device=cache.device) if vote_buf is None
                    else vote_buf.reshape(-1)[: m * n].view(m, n))
            if self.kv_comm is not None and self.plan.kv_world > 1:
                self.kv_comm.vote_allgather(parts, stream=stream, out=vote)
            else:
                call("oomb_vote_reduce", _ptr(parts), g, m, n, _ptr(vote), stream_handle(stream))
            call("oomb_select_topk", full.handle, _ptr(vote), m, n, cfg.budget_pages(), stream_handle(stream))
        elif mode == "local":
            call("oomb_select_recent", full.handle, n_cand, cfg.local_window, m, stream_handle(stream))
        else:  # dense, or no candidates yet (chunk_trainer.hpp:297-304)
            call("oomb_select_all", full.handle, n_cand, m, stream_handle(stream))
        if self.split_pages:
            return full.filter_owned(out=sub, stream=stream)
        return full

    def forward(self, q_local, sel, k_local, v_local, out, lse, o_part=None, lse_part=None, stream=None):
        from . import attention as A
        if not self.split_pages:
            return A.attn_forward(self.lcfg, q_local, self.cache, self.layer, sel, k_local, v_local, stream=stream,
                                  out=out, lse=lse)
        part = A.attn_forward(self.lcfg, q_local, self.cache, self.layer, sel, k_local, v_local, stream=stream,
                              out=o_part, lse=lse_part, past_only=self.plan.range_idx != 0)
        self.range_comm.lse_merge(part.out, part.lse, stream=stream, out=out, lse=lse)
        return A.AttnSaved(out, lse, sel)

    def backward(self, do_local, q_local, k_local, v_local, saved, grads, own_pages, stream=None, flat=None):
        """grads: preallocated AttnGrads; when `flat` is given, grads.dq / dk_cur / dv_cur are views
        of it and one ordered reduction covers all three."""
        from . import attention as A
        A.attn_backward(self.lcfg, do_local, q_local, self.cache, self.layer, k_local, v_local, saved,
                        stream=stream, grads=grads, past_only=self.plan.range_idx != 0)
        if len(own_pages):  # remote pages among them add nothing here (their owners add them)
            self.cache.accumulate_grad_pages(self.layer, own_pages, grads.dk_cur, grads.dv_cur, stream=stream)
        if self.split_pages:
            if flat is not None:
                self.range_comm.allreduce_ordered(flat, stream=stream, out=flat)
            else:
                for t in (grads.dq, grads.dk_cur, grads.dv_cur):
                    self.range_comm.allreduce_ordered(t, stream=stream, out=t)
        return grads
