"""Attention operators — drop-ins for chunktrain/attention.hpp.

score_pages (attention.hpp:32-67), select_topk / select_topk_row (:71-96),
select_recent / select_all (:99-111), attn_forward (:156-208) and
attn_backward (:222-293), computed by the sm_100a kernels in liboomb.so.
A `Selection` is the reference's per-query-page `vector<vector<int32_t>>`,
held as a device CSR with a pinned host mirror.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call
from .config import ModelConfig
from .errors import ShapeError
from .paged_kv import DTYPE_CODE, PagedCache, _ptr, stream_handle


class Selection:
    """Selected page ids per query page (AttnSaved::selected, attention.hpp:117-124)."""

    def __init__(self, cache: PagedCache, max_query_pages: int, max_ids: int):
        self.cache = cache
        h = C.c_void_p()
        call("oomb_selection_create", cache.handle, max_query_pages, max(max_ids, 1), C.byref(h))
        self.handle = h
        self.max_ids = max_ids

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.lib().oomb_selection_destroy(h)
            except Exception:  # interpreter shutdown: module globals may be gone already
                pass
            self.handle = None

    @classmethod
    def from_lists(cls, cache: PagedCache, lists, stream=None) -> "Selection":
        lists = [list(map(int, l)) for l in lists]
        off = np.zeros(len(lists) + 1, np.int32)
        for i, l in enumerate(lists):
            off[i + 1] = off[i] + len(l)
        ids = np.array([x for l in lists for x in l], dtype=np.int32)
        s = cls(cache, max(len(lists), 1), int(off[-1]))
        call("oomb_selection_set_host", s.handle, off.ctypes.data_as(C.c_void_p),
             ids.ctypes.data_as(C.c_void_p) if ids.size else None, len(lists), stream_handle(stream))
        s._keep = (off, ids)
        return s

    def filter_owned(self, out: "Selection | None" = None, stream=None) -> "Selection":
        """The part of this selection the cache's page-range shard owns (list order kept), built on
        the device (oomb_selection_filter_owned); `out` is reused when given."""
        m, nnz = C.c_int(), C.c_int()
        dst = out if out is not None else Selection(self.cache, max(len(self), 1), max(self.max_ids, 1))
        call("oomb_selection_filter_owned", self.cache.handle, self.handle, dst.handle, stream_handle(stream))
        return dst

    def csr(self) -> tuple[np.ndarray, np.ndarray]:
        """(offsets [m+1], ids [nnz]) int32 from the host mirror (waits for the selection's D2H)."""
        m, nnz = C.c_int(), C.c_int()
        call("oomb_selection_get_host", self.handle, None, None, C.byref(m), C.byref(nnz))
        off = np.zeros(m.value + 1, np.int32)
        ids = np.zeros(max(nnz.value, 1), np.int32)
        call("oomb_selection_get_host", self.handle, off.ctypes.data_as(C.c_void_p), ids.ctypes.data_as(C.c_void_p),
             C.byref(m), C.byref(nnz))
        return off, ids[:nnz.value]

    def union(self) -> np.ndarray:
        """Ascending distinct selected page ids (the residency working set of the selection)."""
        return np.unique(self.csr()[1])

    def lists(self) -> list[list[int]]:
        off, ids = self.csr()
        return [ids[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1)]

    def __len__(self) -> int:
        off, ids, m = C.c_void_p(), C.c_void_p(), C.c_int()
        call("oomb_selection_device", self.handle, C.byref(off), C.byref(ids), C.byref(m))
        return m.value


def as_selection(cache: PagedCache, selected, stream=None) -> Selection:
    return selected if isinstance(selected, Selection) else Selection.from_lists(cache, selected, stream)


# ---------------------------------------------------------------------------
# Scoring and selection
# ---------------------------------------------------------------------------
def score_pages(q: torch.Tensor, k_avg: torch.Tensor, page_size: int, gqa_group: int, score_scale: bool = False,
                stream=None) -> torch.Tensor:
    """attention.hpp:32-67 — vote [m, n] fp32 on the device."""
    if q.dim() != 3 or k_avg.dim() != 3:
        raise ShapeError("score_pages: expected rank-3 inputs")
    dev = q.device if q.is_cuda else torch.device("cuda", torch.cuda.current_device())
    dt = q.dtype if q.dtype in (torch.bfloat16, torch.float32, torch.float64) else torch.float32
    acc = torch.float64 if dt == torch.float64 else torch.float32
    q = q.to(dev, dt).contiguous()
    k_avg = k_avg.to(dev, acc).contiguous()
    tokens, qh, hd = q.shape
    n, kvh = k_avg.shape[0], k_avg.shape[1]
    if qh != gqa_group * kvh:
        raise ShapeError("score_pages: head counts do not match the GQA group")
    m = (tokens + page_size - 1) // page_size
    vote = torch.empty((m, max(n, 1)), dtype=acc, device=dev)
    call("oomb_score_pages", _ptr(q), tokens, qh, hd, _ptr(k_avg), n, kvh, page_size, int(score_scale),
         DTYPE_CODE[dt], _ptr(vote), stream_handle(stream))
    return vote[:, :n]


def select_all(n_pages: int) -> list[int]:
    return list(range(n_pages))


def select_recent(n_pages: int, window: int) -> list[int]:
    if window < 0:
        raise ShapeError("select_recent: negative window")
    take = min(n_pages, window)
    return list(range(n_pages - take, n_pages))


def select_topk_rows(cache: PagedCache, vote: torch.Tensor, k: int, stream=None) -> Selection:
    """select_topk_row for every row of a device vote matrix, on the device."""
    vote = vote.to(cache.device, cache.acc_dtype).contiguous()
    m, n = vote.shape
    kk = min(max(k, 0), n)
    sel = Selection(cache, max(m, 1), m * kk)
    call("oomb_select_topk", sel.handle, _ptr(vote), m, n, k, stream_handle(stream))
    return sel


def select_topk(score_row, budget_pages: int, cache: PagedCache | None = None) -> list[int]:
    """attention.hpp:71-88 on the device (ties -> lower id, ascending)."""
    if budget_pages < 0:
        raise ShapeError("select_topk: negative budget")
    c = cache if cache is not None else _scratch_cache()
    # the reference compares the row as double (attention.hpp:71-88): the scratch pool is fp64
    row = torch.as_tensor(np.asarray(score_row, dtype=np.float64 if c.acc_dtype == torch.float64 else np.float32))
    row = row.reshape(1, -1)
    return select_topk_rows(c, row, budget_pages).lists()[0]


def select_topk_row(score: torch.Tensor, row: int, budget_pages: int, cache: PagedCache | None = None) -> list[int]:
    return select_topk(score[row].detach().double().cpu().numpy(), budget_pages, cache)


_SCRATCH = {}


def _scratch_cache() -> PagedCache:
    dev = torch.cuda.current_device()
    if dev not in _SCRATCH:
        _SCRATCH[dev] = PagedCache(ModelConfig(n_layers=1, n_q_heads=1, n_kv_heads=1, head_dim=2, chunk_size=1,
                                               page_size=1, retrieval_budget=0), dtype="fp64", max_tokens=1)
    return _SCRATCH[dev]


def select_pages_topk(cache: PagedCache, layer: int, q: torch.Tensor, n_candidates: int, stream=None,
                      out: Selection | None = None, vote: torch.Tensor | None = None) -> Selection:
    """chunk_trainer.hpp:305-311: K_avg (pinned metadata) -> score_pages -> select_topk_row
    per query page, all on the device. `out` / `vote` let a caller reuse buffers."""
    cfg = cache.cfg
    q = cache._dev(q)
    m = (q.shape[0] + cfg.page_size - 1) // cfg.page_size
    n = min(n_candidates, cache.n_pages(layer))
    k = min(cfg.budget_pages(), max(n, 0))
    sel = out if out is not None else Selection(cache, max(m, 1), m * k)
    if vote is None or vote.numel() < m * max(n, 1):
        vote = torch.empty((m, max(n, 1)), dtype=cache.acc_dtype, device=cache.device)
    else:
        vote = vote.reshape(-1)[: m * max(n, 1)].view(m, max(n, 1))
    call("oomb_select_pages_topk", cache.handle, layer, _ptr(q), q.shape[0], n_candidates, sel.handle, _ptr(vote),
         stream_handle(stream))
    sel.vote = vote[:, :max(n, 0)]
    return sel


# ---------------------------------------------------------------------------
# Streaming attention forward / exact backward
# ---------------------------------------------------------------------------
@dataclass
class AttnSaved:
    out: torch.Tensor        # [C, qh, hd] pool dtype
    lse: torch.Tensor        # [C, qh] fp32, natural log
    selected: Selection      # cached ids, reused verbatim by the backward


@dataclass
class AttnGrads:
    dq: torch.Tensor         # [C, qh, hd] fp32
    dk_cur: torch.Tensor     # [C, kvh, hd] fp32
    dv_cur: torch.Tensor


PAST_ONLY = 1  # OOMB_ATTN_PAST_ONLY: a page-range shard that does not own the chunk's own keys
DEFER_DQ = 2   # OOMB_ATTN_DEFER_DQ: dq keeps running on the library's side stream (join_dq)


def attn_forward(cfg: ModelConfig, q, cache: PagedCache, layer: int, selected, k_cur, v_cur,
                 stream=None, out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                 past_only: bool = False) -> AttnSaved:
    """attention.hpp:156-208. `out` / `lse` may be preallocated by the caller.
    past_only: page-range shard mode (selected pages only, no chunk keys; see sharding.PageRangeShard)."""
    q, k_cur, v_cur = cache._dev(q), cache._dev(k_cur), cache._dev(v_cur)
    c, qh, hd = q.shape
    if qh != cfg.n_q_heads or hd != cfg.head_dim or k_cur.shape != (c, cfg.n_kv_heads, hd) or \
            v_cur.shape != k_cur.shape:
        raise ShapeError("attn_forward: q / k_cur / v_cur shape mismatch")
    sel = as_selection(cache, selected, stream)
    out = torch.empty_like(q) if out is None else out
    lse = torch.empty((c, qh), dtype=cache.acc_dtype, device=q.device) if lse is None else lse
    if out.shape != q.shape or out.dtype != q.dtype or lse.shape != (c, qh) or lse.dtype != cache.acc_dtype:
        raise ShapeError("attn_forward: preallocated out / lse have the wrong shape or dtype")
    # under residency enforcement the library checks the selected pages on the host before the
    # launch (ResidencyError, paged_kv.hpp:301-312); the kernels' device flag is read by
    # cache.check_device_errors() without draining the stream on every chunk
    call("oomb_attn_forward_ex", cache.handle, layer, _ptr(q), c, sel.handle, _ptr(k_cur), _ptr(v_cur), _ptr(out),
         _ptr(lse), PAST_ONLY if past_only else 0, stream_handle(stream))
    return AttnSaved(out, lse, sel)


def attn_backward(cfg: ModelConfig, dout, q, cache: PagedCache, layer: int, k_cur, v_cur, saved: AttnSaved,
                  stream=None, grads: AttnGrads | None = None, past_only: bool = False,
                  selected=None, defer_dq: bool = False, own_first_page: int | None = None) -> AttnGrads:
    """attention.hpp:222-293 — past-page dK/dV go into the cache's gradient pages.
    `grads` may carry preallocated fp32 output buffers. defer_dq: the stream does not wait for dq
    (it overlaps the caller's next backward); join_dq(cache, stream) before reading it.
    own_first_page: dk_cur / dv_cur also receive the pool gradients of the chunk's own pages
    own_first_page .. + C / P - 1 (the dM_i read-back, PagedCache.accumulate_grad_pages of those
    pages, chunk_trainer.hpp:575-587) within the same call (oomb_attn_backward_readback)."""
    dout, q = cache._dev(dout), cache._dev(q)
    k_cur, v_cur = cache._dev(k_cur), cache._dev(v_cur)
    if dout.shape != saved.out.shape:
        raise ShapeError("attn_backward: dO shape mismatch")
    c = q.shape[0]
    if grads is None:
        dq = torch.empty((c, cfg.n_q_heads, cfg.head_dim), dtype=cache.acc_dtype, device=q.device)
        dk = torch.empty((c, cfg.n_kv_heads, cfg.head_dim), dtype=cache.acc_dtype, device=q.device)
        dv = torch.empty_like(dk)
    else:
        dq, dk, dv = grads.dq, grads.dk_cur, grads.dv_cur
        if dq.shape != (c, cfg.n_q_heads, cfg.head_dim) or dk.shape != (c, cfg.n_kv_heads, cfg.head_dim) or \
                dv.shape != dk.shape or {dq.dtype, dk.dtype, dv.dtype} != {cache.acc_dtype}:
            raise ShapeError("attn_backward: preallocated gradients have the wrong shape or dtype")
    sel = saved.selected if selected is None else as_selection(cache, selected, stream)
    flags = (PAST_ONLY if past_only else 0) | (DEFER_DQ if defer_dq else 0)
    args = (cache.handle, layer, _ptr(dout), _ptr(q), c, sel.handle, _ptr(k_cur), _ptr(v_cur), _ptr(saved.out),
            _ptr(saved.lse), _ptr(dq), _ptr(dk), _ptr(dv), flags)
    if own_first_page is None:
        call("oomb_attn_backward_ex", *args, stream_handle(stream))
    else:
        call("oomb_attn_backward_readback", *args, own_first_page, stream_handle(stream))
    return AttnGrads(dq, dk, dv)


def join_dq(cache: PagedCache, stream=None) -> None:
    """Make `stream` wait for every dq deferred by attn_backward(..., defer_dq=True)."""
    call("oomb_attn_join_dq", cache.handle, stream_handle(stream))


def rope(x: torch.Tensor, pos_offset: int, base: float = 10000.0, sign: int = 1, out=None,
         out_dtype=None) -> torch.Tensor:
    """ops.hpp:192-225 (sign -1: rope_backward, ops.hpp:227-230) on the device, [rows, heads, hd]."""
    if x.dim() != 3:
        raise ShapeError("rope: expected [t x h x d]")
    x = x.contiguous() if x.is_cuda else x.cuda().contiguous()
    odt = out_dtype or x.dtype
    out = torch.empty(x.shape, dtype=odt, device=x.device) if out is None else out
    code = {torch.float32: 0, torch.bfloat16: 1}
    call("oomb_rope", _ptr(x), x.shape[0], x.shape[1], x.shape[2], int(pos_offset), C.c_float(base), int(sign),
         code[x.dtype], code[odt], _ptr(out), stream_handle(None))
    return out


def debug_tc_gemm(mode: int, a: torch.Tensor, b: torch.Tensor, n: int) -> torch.Tensor:
    """Validation hook for the tcgen05/TMA descriptor builders (tests only)."""
    m, k = a.shape
    c = torch.empty((m, n), dtype=torch.float32, device=a.device)
    call("oomb_debug_tc_gemm", mode, _ptr(a.contiguous()), _ptr(b.contiguous()), _ptr(c), m, n, k,
         stream_handle(None))
    return c
