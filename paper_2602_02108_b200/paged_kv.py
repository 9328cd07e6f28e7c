"""PagedCache — drop-in for chunktrain::PagedCache<Real> (paged_kv.hpp:41-356).

The page pool lives in HBM (K/V pages in the pool dtype, dK/dV pages fp32) and
is owned by liboomb.so; this class keeps the reference's method names and
semantics and moves tensors across the C ABI as raw device pointers. Inputs
may be CPU or CUDA tensors (CPU inputs are copied to the device first);
outputs are CUDA tensors.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import I32P, OombConfig, OombMemoryReport, call
from .config import ModelConfig
from .errors import ShapeError

DEVICE = 0
HOST = 1


def torch_dtype(name: str) -> torch.dtype:
    return {"fp32": torch.float32, "f32": torch.float32, "bf16": torch.bfloat16, "fp64": torch.float64,
            "f64": torch.float64}[name]


DTYPE_CODE = {torch.float32: 0, torch.bfloat16: 1, torch.float64: 2}  # oomb_dtype


def stream_handle(stream: torch.cuda.Stream | None = None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


@dataclass
class SlotRange:
    begin: int
    end: int


@dataclass
class Gathered:
    k: torch.Tensor      # [n_ids*P, kvh, hd]
    v: torch.Tensor
    valid: torch.Tensor  # [n_ids*P] uint8


@dataclass
class MemoryReport:
    device_bytes: int
    host_bytes: int
    grad_bytes: int
    pages: int
    reallocs: int
    copied_bytes: int
    arena_blocks: int
    free_list: int


class PagedCache:
    """Per-layer logical page tables over a device page pool.

    dtype: "bf16" (tensor-core path), "fp32" (1e-5 parity path) or "fp64" (the reference's Real = double:
    exact SIMT kernels in double; K_avg, gradient pages, lse, dq and votes are double too).
    max_tokens: per-layer capacity of the device page table.
    device_capacity_pages: KV page slots on the device (all layers); default = all (the owned share).
    page_owner: (stride R, rank r) of a page-range shard: this pool stores K/V and
        gradients only for pages with id % R == r; the others are REMOTE (tier 2): appends still
        add their rows to K_avg (so every shard scores every candidate), reads raise ResidencyError.
    """

    def __init__(self, cfg: ModelConfig, dtype: str = "bf16", max_tokens: int | None = None,
                 device: int | None = None, device_capacity_pages: int = -1,
                 page_owner: tuple[int, int] | None = None):
        cfg.validate()
        self.cfg = cfg
        self.dtype_name = dtype
        self.dtype = torch_dtype(dtype)
        # accumulation type of K_avg, gradient pages, lse / dq / dk_cur / dv_cur and votes
        self.acc_dtype = torch.float64 if self.dtype == torch.float64 else torch.float32
        self.device_index = torch.cuda.current_device() if device is None else device
        self.device = torch.device("cuda", self.device_index)
        self.max_tokens = max_tokens if max_tokens is not None else 64 * cfg.chunk_size
        c = OombConfig(cfg.n_layers, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.chunk_size, cfg.page_size,
                       cfg.retrieval_budget, cfg.local_window, int(cfg.score_scale),
                       DTYPE_CODE[self.dtype], self.max_tokens, device_capacity_pages,
                       *(page_owner if page_owner is not None else (0, 0)))
        self.owner_stride, self.owner_rank = (max(1, page_owner[0]), page_owner[1]) if page_owner else (1, 0)
        h = C.c_void_p()
        call("oomb_pool_create", C.byref(c), self.device_index, C.byref(h))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.lib().oomb_pool_destroy(h)
            except Exception:  # interpreter shutdown: module globals may be gone already
                pass
            self.handle = None

    # ------------------------------------------------------------------ helpers
    def _dev(self, t, dtype=None) -> torch.Tensor:
        if isinstance(t, np.ndarray):
            t = torch.from_numpy(t)
        return t.to(device=self.device, dtype=dtype or self.dtype).contiguous()

    def _ids(self, ids) -> np.ndarray:
        return np.ascontiguousarray(np.asarray(list(ids) if not isinstance(ids, np.ndarray) else ids,
                                               dtype=np.int32).reshape(-1))

    # ------------------------------------------------------------------ reference API
    def page_size(self) -> int:
        return self.cfg.page_size

    @property
    def n_layers(self) -> int:
        return self.cfg.n_layers

    def page_elems(self) -> int:
        return self.cfg.page_size * self.cfg.n_kv_heads * self.cfg.head_dim

    def page_buffer_bytes(self) -> int:
        return self.page_elems() * (2 if self.dtype == torch.bfloat16 else 4)

    def page_kv_bytes(self) -> int:
        return 2 * self.page_buffer_bytes()

    def filled(self, layer: int) -> int:
        out = C.c_int64()
        call("oomb_filled", self.handle, layer, C.byref(out))
        return out.value

    def n_pages(self, layer: int) -> int:
        out = C.c_int()
        call("oomb_n_pages", self.handle, layer, C.byref(out))
        return out.value

    def owns(self, page: int) -> bool:
        """Page-range shard ownership: True when this pool stores the page's K/V and gradients."""
        return self.owner_stride <= 1 or page % self.owner_stride == self.owner_rank

    def owned(self, ids) -> np.ndarray:
        """The ids this pool stores, order kept (all of them without page ownership)."""
        a = self._ids(ids)
        return a if self.owner_stride <= 1 else np.ascontiguousarray(a[a % self.owner_stride == self.owner_rank])

    @staticmethod
    def full_pages_before(tokens: int, page_size: int) -> int:
        return tokens // page_size

    def append_chunk(self, layer: int, k, v, stream=None, rope_base: float | None = None) -> SlotRange:
        """paged_kv.hpp:73-108 — write rows into tail-page slots, update K_avg sums.
        rope_base: k is the PRE-RoPE projection; it is rotated at its absolute positions on the
        way into the page (the fused epilogue of chunk_trainer.hpp:424-432)."""
        k, v = self._dev(k), self._dev(v)
        cfg = self.cfg
        if k.dim() != 3 or k.shape[1] != cfg.n_kv_heads or k.shape[2] != cfg.head_dim or k.shape != v.shape:
            raise ShapeError("append_chunk: expected [rows x kvh x hd] K/V of equal shape")
        b, e = C.c_int64(), C.c_int64()
        if rope_base is None:
            call("oomb_append_chunk", self.handle, layer, _ptr(k), _ptr(v), k.shape[0], stream_handle(stream),
                 C.byref(b), C.byref(e))
        else:
            call("oomb_append_chunk_rope", self.handle, layer, _ptr(k), _ptr(v), k.shape[0], C.c_float(rope_base),
                 stream_handle(stream), C.byref(b), C.byref(e))
        return SlotRange(b.value, e.value)

    def gather_pages(self, layer: int, page_ids, stream=None) -> Gathered:
        return self._gather(layer, page_ids, False, stream)

    def gather_grad_pages(self, layer: int, page_ids, stream=None) -> Gathered:
        return self._gather(layer, page_ids, True, stream)

    def _gather(self, layer, page_ids, grads, stream):
        ids = self._ids(page_ids)
        rows = len(ids) * self.cfg.page_size
        dt = self.acc_dtype if grads else self.dtype
        k = torch.zeros((rows, self.cfg.n_kv_heads, self.cfg.head_dim), dtype=dt, device=self.device)
        v = torch.zeros_like(k)
        valid = torch.zeros(rows, dtype=torch.uint8, device=self.device)
        call("oomb_gather_pages", self.handle, layer, ids.ctypes.data_as(C.c_void_p), len(ids), int(grads), _ptr(k),
             _ptr(v), _ptr(valid), stream_handle(stream))
        return Gathered(k, v, valid)

    def scatter_add_grads(self, layer: int, page_ids, dk, dv, stream=None) -> None:
        """paged_kv.hpp:135-164 — lazily allocated, zeroed grad pages; valid slots add in place."""
        ids = self._ids(page_ids)
        dk, dv = self._dev(dk, self.acc_dtype), self._dev(dv, self.acc_dtype)
        want = len(ids) * self.cfg.page_size
        if (dk.dim() != 3 or dk.shape[0] != want or dk.shape[1] != self.cfg.n_kv_heads
                or dk.shape[2] != self.cfg.head_dim or dk.shape != dv.shape):
            raise ShapeError("scatter_add_grads: gradient shape does not match gather layout")
        call("oomb_scatter_add_grads", self.handle, layer, ids.ctypes.data_as(C.c_void_p), len(ids), _ptr(dk),
             _ptr(dv), stream_handle(stream))

    def page_mean_keys(self, layer: int, n_candidates: int = -1, stream=None) -> torch.Tensor:
        """paged_kv.hpp:170-183 — fp32 [n, kvh, hd]."""
        cap = max(self.n_pages(layer), 1)
        out = torch.empty((cap, self.cfg.n_kv_heads, self.cfg.head_dim), dtype=self.acc_dtype, device=self.device)
        n = C.c_int()
        call("oomb_page_mean_keys", self.handle, layer, n_candidates, _ptr(out), stream_handle(stream), C.byref(n))
        return out[: n.value]

    def kavg_raw(self, layer: int):
        n = self.n_pages(layer)
        s = torch.zeros((max(n, 1), self.cfg.n_kv_heads, self.cfg.head_dim), dtype=self.acc_dtype, device=self.device)
        cnt = torch.zeros(max(n, 1), dtype=torch.int32, device=self.device)
        call("oomb_kavg_raw", self.handle, layer, _ptr(s), _ptr(cnt), stream_handle(None))
        return s[:n], cnt[:n]

    def memory_report(self) -> MemoryReport:
        r = OombMemoryReport()
        call("oomb_memory_report_get", self.handle, C.byref(r))
        return MemoryReport(r.device_bytes, r.host_bytes, r.grad_bytes, r.pages, r.reallocs, r.copied_bytes,
                            r.arena_blocks, r.free_list)

    def tier(self, layer: int, page: int) -> int:
        out = C.c_int()
        call("oomb_get_tier", self.handle, layer, page, C.byref(out))
        return out.value

    def set_tier(self, layer: int, page: int, tier: int) -> None:
        call("oomb_set_tier", self.handle, layer, page, int(tier))

    def grads_allocated(self, layer: int, page: int) -> bool:
        out = C.c_int()
        call("oomb_grads_allocated", self.handle, layer, page, C.byref(out))
        return bool(out.value)

    def set_residency_enforced(self, on: bool) -> None:
        call("oomb_set_residency_enforced", self.handle, int(on))
        self._enforced = bool(on)

    def residency_enforced(self) -> bool:
        return getattr(self, "_enforced", False)

    def zero_grad_pages(self, stream=None) -> None:
        call("oomb_zero_grad_pages", self.handle, stream_handle(stream))

    def reset(self, stream=None) -> None:
        call("oomb_pool_reset", self.handle, stream_handle(stream))

    # ------------------------------------------------------------------ introspection
    def page_table(self, layer: int) -> np.ndarray:
        """Reference arena ids per logical page: [n, 4] = k_phys, v_phys, gk_phys, gv_phys."""
        n = self.n_pages(layer)
        out = np.zeros((max(n, 1), 4), np.int32)
        call("oomb_page_table_get", self.handle, layer, out.ctypes.data_as(C.c_void_p))
        return out[:n]

    def device_slots(self, layer: int) -> np.ndarray:
        n = self.n_pages(layer)
        out = np.zeros((max(n, 1), 2), np.int32)
        call("oomb_device_slots_get", self.handle, layer, out.ctypes.data_as(C.c_void_p))
        return out[:n]

    def accumulate_grad_pages(self, layer: int, page_ids, dk: torch.Tensor, dv: torch.Tensor, stream=None) -> None:
        """dM_i read-back (chunk_trainer.hpp:575-587): dk += gather_grad_pages(ids).k, same for dv."""
        ids = self._ids(page_ids)
        if dk.dtype != self.acc_dtype or not dk.is_cuda or not dk.is_contiguous() or dk.shape != dv.shape:
            raise ShapeError("accumulate_grad_pages: fp32 contiguous CUDA dk/dv of equal shape required")
        call("oomb_accumulate_grad_pages", self.handle, layer, ids.ctypes.data_as(C.c_void_p), len(ids), _ptr(dk),
             _ptr(dv), stream_handle(stream))

    def accumulate_grad_pages_rope(self, layer: int, page_ids, dk: torch.Tensor, dv: torch.Tensor, pos_offset: int,
                                   rope_base: float = 10000.0, stream=None) -> None:
        """The dM_i read-back fused with rope_backward of dK (chunk_trainer.hpp:575-592):
        dk <- rope^-1(dk + grad_k(ids)), dv += grad_v(ids); row r at position pos_offset + r."""
        ids = self._ids(page_ids)
        if dk.dtype != self.acc_dtype or not dk.is_cuda or not dk.is_contiguous() or dk.shape != dv.shape:
            raise ShapeError("accumulate_grad_pages_rope: fp32 contiguous CUDA dk/dv of equal shape required")
        call("oomb_accumulate_grad_pages_rope", self.handle, layer, ids.ctypes.data_as(C.c_void_p), len(ids),
             _ptr(dk), _ptr(dv), int(pos_offset), C.c_float(rope_base), stream_handle(stream))

    PROFILE_KINDS = ("append", "score", "topk", "attn_fwd", "bwd_prep", "bwd_dq", "bwd_dkdv", "bwd_simt",
                     "grad_init", "gather_scatter", "other", "bwd_pair")

    def profile_enable(self, on: bool = True) -> None:
        call("oomb_profile_enable", self.handle, int(on))

    def profile_collect(self) -> dict:
        """Per kernel kind: (launches, device ms) since the last collect (synchronises)."""
        n = len(self.PROFILE_KINDS)
        counts = np.zeros(n, np.int64)
        ms = np.zeros(n, np.float64)
        call("oomb_profile_collect", self.handle, counts.ctypes.data_as(C.c_void_p), ms.ctypes.data_as(C.c_void_p), n)
        return {k: (int(c), float(t)) for k, c, t in zip(self.PROFILE_KINDS, counts, ms) if c}

    def check_device_errors(self) -> None:
        call("oomb_check_device_errors", self.handle)

    def set_kernel_policy(self, policy: str) -> None:
        call("oomb_set_kernel_policy", self.handle, {"auto": 0, "simt": 1, "tcgen05": 2}[policy])
