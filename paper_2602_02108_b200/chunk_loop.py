"""The hot path's own call sequence for one attention layer over a sequence.

This is the attention-only slice of ChunkTrainer::train_step
(chunk_trainer.hpp:131-186): for every chunk in order, select pages (top-k on
the device, or dense / local), append the chunk's K/V, run the forward; then for
every chunk in reverse order run the backward (past-page dK/dV into the paged
gradient pool) and the dM_i read-back (chunk_trainer.hpp:575-587). With a
TieredEngine the residency protocol of run_chunk_ is followed: fetch right after
selection (the q-projection point for top-k, :414-419), on_pages_appended,
ensure_resident_ (wait + fill fetch + record_access, :356-363), end_layer_use
after the layer (:455-462), and in the backward a one-step-ahead prefetch of the
next (earlier) chunk's cached ids plus its own grad pages (:328-351, :531-541).
Projections / MLP are not on the path; their inputs (q, k, v, dO per chunk) are
supplied by the caller.
"""
from __future__ import annotations

import numpy as np
import torch

from . import attention as A
from ._lib import call
from .paged_kv import PagedCache, _ptr, stream_handle


class AttentionChunkLoop:
    def __init__(self, cache: PagedCache, layer: int = 0, engine=None, max_chunks: int = 0):
        self.cache = cache
        self.cfg = cache.cfg
        self.layer = layer
        self.engine = engine
        c = self.cfg
        self.m = c.chunk_size // c.page_size
        self.mode = c.mode_for_layer(layer)
        self.sels: list[A.Selection] = []
        self.saved: list[A.AttnSaved] = []
        self.max_chunks = max_chunks
        self._presel: dict[int, A.Selection] = {}  # selections issued one chunk ahead (forward_chunk next_q)
        self._sel_stream = None
        self._votes = None
        # per-chunk residency statistics when an engine is attached: (phase, chunk, pages the chunk
        # needs resident, H2D bytes and D2H bytes the engine moved during the chunk's call)
        self.chunk_stats: list[tuple[str, int, int, int, int]] = []

    def _io(self) -> tuple[int, int]:
        e = self.engine
        return (e.h2d_bytes(0) + e.h2d_bytes(1), e.d2h_bytes()) if e is not None else (0, 0)

    # ---- selection (chunk_trainer.hpp:292-316)
    def _select(self, i: int, q: torch.Tensor, sel: A.Selection, stream=None) -> A.Selection:
        n_cand = i * self.m
        if self.mode == "topk" and n_cand > 0:
            return A.select_pages_topk(self.cache, self.layer, q, n_cand, stream=stream, out=sel)
        if self.mode == "local" and n_cand > 0:
            call("oomb_select_recent", sel.handle, n_cand, self.cfg.local_window, self.m, stream_handle(stream))
        else:
            call("oomb_select_all", sel.handle, n_cand, self.m, stream_handle(stream))
        return sel

    def own_pages(self, i: int) -> np.ndarray:
        return np.arange(i * self.m, (i + 1) * self.m, dtype=np.int32)

    @staticmethod
    def union(sel: A.Selection) -> np.ndarray:
        return sel.union()

    def _selection(self, i: int) -> A.Selection:
        while i >= len(self.sels):
            kmax = self.m * (self.cfg.budget_pages() if self.mode == "topk" else
                             (self.cfg.local_window if self.mode == "local" else self.cache.max_tokens //
                              self.cfg.page_size))
            self.sels.append(A.Selection(self.cache, self.m, max(kmax, 1)))
        return self.sels[i]

    def _preselect(self, i: int, q, stream) -> None:
        """Issue chunk i's page selection on a side stream right after chunk i-1's append (it reads
        only K_avg of chunks < i, chunk_trainer.hpp:297-311), so it runs under chunk i-1's attention
        and the host's wait for the ids (the fetch decision) does not drain the compute stream."""
        if self._sel_stream is None:
            # high priority: the selection's CTAs go ahead of the running attention's remaining ones
            self._sel_stream = torch.cuda.Stream(device=self.cache.device, priority=-1)
            n = self.m * max(self.cache.max_tokens // self.cfg.page_size, 1)
            self._votes = [torch.empty(n, dtype=torch.float32, device=self.cache.device) for _ in range(2)]
        ss = self._sel_stream
        ss.wait_stream(torch.cuda.current_stream() if stream is None else stream)
        sel = self._selection(i)
        n_cand = i * self.m
        if self.mode == "topk" and n_cand > 0:
            A.select_pages_topk(self.cache, self.layer, q, n_cand, stream=ss, out=sel, vote=self._votes[i & 1])
        else:
            self._select(i, q, sel, ss)
        self._presel[i] = sel

    def forward_chunk(self, i: int, q, k, v, stream=None, next_q=None, out=None, lse=None) -> A.AttnSaved:
        """One chunk of the forward. next_q: the next chunk's queries; its selection is then issued
        on a side stream as soon as this chunk's pages are appended (same engine call order).
        out / lse: caller-owned output buffers (the saved activations of the chunk)."""
        sel = self._presel.pop(i, None)
        if sel is None:
            sel = self._select(i, q, self._selection(i), stream)
        else:  # the compute stream must not read the selection before the side stream wrote it
            (torch.cuda.current_stream() if stream is None else stream).wait_stream(self._sel_stream)
        eng = self.engine
        h = None
        io0 = self._io()
        if eng is not None:
            h = eng.fetch_async(self.layer, self.union(sel), i)
        r = self.cache.append_chunk(self.layer, k, v, stream=stream)
        if next_q is not None:
            self._preselect(i + 1, next_q, stream)
        if eng is not None:
            eng.on_pages_appended(self.layer, r)
            ids = self.union(sel)
            eng.wait(h)
            eng.wait(eng.fetch_async(self.layer, ids, i))
            eng.record_access(self.layer, ids, i)
        saved = A.attn_forward(self.cfg, q, self.cache, self.layer, sel, k, v, stream=stream, out=out, lse=lse)
        if eng is not None:
            eng.end_layer_use(self.layer, np.concatenate([ids, self.own_pages(i)]))
            io1 = self._io()
            self.chunk_stats.append(("fwd", i, len(ids), io1[0] - io0[0], io1[1] - io0[1]))
        if i < len(self.saved):
            self.saved[i] = saved
        else:
            self.saved.append(saved)
        return saved

    def backward_chunk(self, i: int, dout, q, k, v, stream=None, prefetch_next: bool = True,
                       grads: A.AttnGrads | None = None) -> A.AttnGrads:
        eng = self.engine
        sel = self.sels[i]
        io0 = self._io()
        if eng is not None:
            ids = np.union1d(self.union(sel), self.own_pages(i)).astype(np.int32)
            eng.wait(eng.fetch_async(self.layer, ids, i))
            eng.record_access(self.layer, ids, i)
            if prefetch_next and i > 0:  # step-ahead prefetch with cached ids + own grad pages
                nxt = np.union1d(self.union(self.sels[i - 1]), self.own_pages(i - 1)).astype(np.int32)
                self._pending = eng.fetch_async(self.layer, nxt, i - 1, best_effort=True)
        g = A.attn_backward(self.cfg, dout, q, self.cache, self.layer, k, v, self.saved[i], stream=stream, grads=grads)
        if eng is not None:
            eng.on_grads_scattered(self.layer, self.union(sel))
        self.cache.accumulate_grad_pages(self.layer, self.own_pages(i), g.dk_cur, g.dv_cur, stream=stream)
        if eng is not None:
            eng.end_layer_use(self.layer, ids)
            io1 = self._io()
            self.chunk_stats.append(("bwd", i, len(ids), io1[0] - io0[0], io1[1] - io0[1]))
        return g

    def check_device_errors(self) -> None:
        """The kernels' device-side residency / page-id flags (the host check in front of every
        launch raises ResidencyError first; this confirms no kernel saw a non-resident slot)."""
        self.cache.check_device_errors()

    def begin_backward(self):
        if self.engine is not None:
            self.check_device_errors()
            from .tiered_memory import BACKWARD
            self.engine.release_all_reservations()
            self.engine.begin_phase(BACKWARD)


MODES = {"dense": 0, "topk": 1, "local": 2}  # OOMB_MODE_*


def layer_step(cache: PagedCache, layer: int, q, k, v, dout, out, lse, grads: A.AttnGrads, mode: str | None = None,
               grad_stride_chunks: int = 0, phase: str = "both", stream=None) -> None:
    """The attention layer's whole chunk-recurrent step as ONE native call (oomb_layer_step): the
    same select -> append -> attend forward and reverse backward + dM_i read-back as
    AttentionChunkLoop without an engine, with the bench's overlaps (selection one chunk ahead on a
    high-priority stream, two forward streams, deferred dQ). q / dout: [Rq][C][Hq][hd] (chunk i uses
    block i % Rq), k / v: [S][C][Hkv][hd]; out [S][C][Hq][hd], lse [S][C][Hq]; grads.dq / dk_cur /
    dv_cur hold one chunk (grad_stride_chunks = 0: every chunk reuses it) or S chunks (= 1).
    phase: "both", "forward" (OOMB_LAYER_FORWARD_ONLY) or "backward" (the backward of the pool's
    last forward of the same chunks, OOMB_LAYER_BACKWARD_ONLY). With a TieredEngine attached to the
    cache the native loop runs AttentionChunkLoop's residency protocol (forward_chunk /
    begin_backward / backward_chunk with an engine) call for call; `stream` must then be the
    engine's compute stream, and layer_stats() returns its per-chunk records."""
    cfg = cache.cfg
    mode = mode or cfg.mode_for_layer(layer)
    S = k.shape[0]
    for t, want in ((q, cache.dtype), (k, cache.dtype), (v, cache.dtype), (dout, cache.dtype), (out, cache.dtype),
                    (lse, cache.acc_dtype), (grads.dq, cache.acc_dtype), (grads.dk_cur, cache.acc_dtype),
                    (grads.dv_cur, cache.acc_dtype)):
        if t.dtype != want or not t.is_cuda or not t.is_contiguous():
            raise ValueError("layer_step: contiguous device tensors of the pool / accumulation dtype expected")
    call("oomb_layer_step", cache.handle, layer, S, MODES[mode], _ptr(q), q.shape[0], _ptr(k), _ptr(v), _ptr(dout),
         dout.shape[0], _ptr(out), _ptr(lse), _ptr(grads.dq), _ptr(grads.dk_cur), _ptr(grads.dv_cur),
         grad_stride_chunks, {"both": 0, "forward": 1, "backward": 2}[phase], stream_handle(stream))


def layer_stats(cache: PagedCache) -> list[tuple[str, int, int, int, int]]:
    """Per-chunk residency records of the cache's last engine-attached layer_step, in the format of
    AttentionChunkLoop.chunk_stats: (phase, chunk, pages needed resident, H2D bytes, D2H bytes)."""
    import ctypes as C
    n = C.c_int64()
    call("oomb_layer_stats", cache.handle, None, 0, C.byref(n))
    buf = np.zeros((max(n.value, 1), 5), np.int64)
    call("oomb_layer_stats", cache.handle, buf.ctypes.data_as(C.c_void_p), n.value, C.byref(n))
    return [("fwd" if r[0] == 0 else "bwd", int(r[1]), int(r[2]), int(r[3]), int(r[4])) for r in buf[:n.value]]
