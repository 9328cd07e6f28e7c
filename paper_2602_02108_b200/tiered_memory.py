"""TieredEngine — drop-in for chunktrain::TieredEngine (tiered_memory.hpp:99-432).

On a `PagedCache` the engine really moves pages: dirty K/V (and dK/dV) pages are
written back D2H into pinned host memory on eviction and fetched H2D into fresh
device slots, on side streams, with the compute stream waiting only in `wait`.
On a `HostPageTable` (no device) it runs the reference's simulated clock and its
ScheduleLog matches the reference event for event.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import OombMemoryReport, call

FORWARD, BACKWARD = 0, 1
EVENT_KINDS = ("fetch_issued", "fetch_done", "evict", "compute_begin", "compute_end", "access")


class OombTierConfig(C.Structure):
    _fields_ = [("device_capacity_pages", C.c_int64), ("bandwidth_bytes_per_s", C.c_double),
                ("fixed_s_per_layer", C.c_double), ("s_per_attended_token", C.c_double)]


class OombEvent(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layer", C.c_int32), ("page", C.c_int32), ("chunk", C.c_int32),
                ("phase", C.c_int32), ("pad", C.c_int32), ("bytes", C.c_uint64), ("t", C.c_double)]


@dataclass
class ComputeCostModel:  # tiered_memory.hpp:58-72
    fixed_s_per_layer: float = 1e-3
    s_per_attended_token: float = 1e-6
    kQFrac = 0.25
    kKvFrac = 0.25
    kPostFrac = 0.50

    def q_time(self):
        return self.fixed_s_per_layer * self.kQFrac

    def kv_time(self):
        return self.fixed_s_per_layer * self.kKvFrac

    def post_time(self):
        return self.fixed_s_per_layer * self.kPostFrac

    def attn_time(self, attended_tokens: int):
        return self.s_per_attended_token * attended_tokens


@dataclass
class TierConfig:  # tiered_memory.hpp:74-78
    device_capacity_pages: int = -1
    bandwidth_bytes_per_s: float = 16e9
    compute: ComputeCostModel = field(default_factory=ComputeCostModel)


@dataclass
class ScheduleEvent:
    kind: str
    t: float
    layer: int
    page: int
    chunk: int
    bytes: int
    phase: str


@dataclass
class ScheduleLog:
    bandwidth_bytes_per_s: float
    events: list


@dataclass
class ValidationReport:
    violations: list  # messages, as the reference's ValidationReport::violations (tiered_memory.hpp:84-97)
    stall_seconds: float
    transfer_bytes: int
    h2d_bytes_forward: int
    h2d_bytes_backward: int
    d2h_bytes: int
    overlap_fraction: float


def _ids(ids):
    a = np.ascontiguousarray(np.asarray(list(ids) if not isinstance(ids, np.ndarray) else ids, np.int32).reshape(-1))
    return a, a.ctypes.data_as(C.c_void_p)


class HostPageTable:
    """The page-table bookkeeping of PagedCache without a device (simulation mode)."""

    def __init__(self, n_layers, page_size, n_kv_heads, head_dim, kv_elem_bytes=4, grad_elem_bytes=4):
        h = C.c_void_p()
        call("oomb_pagetable_create", n_layers, page_size, n_kv_heads, head_dim, kv_elem_bytes, grad_elem_bytes,
             C.byref(h))
        self.handle = h
        self.P = page_size
        self.page_kv_bytes_ = 2 * page_size * n_kv_heads * head_dim * kv_elem_bytes

    def __del__(self):
        if getattr(self, "handle", None):
            _lib.lib().oomb_pagetable_destroy(self.handle)
            self.handle = None

    def append_chunk(self, layer, rows):
        b, e = C.c_int64(), C.c_int64()
        call("oomb_pagetable_append", self.handle, layer, rows, C.byref(b), C.byref(e))
        return b.value, e.value

    def scatter_add_grads(self, layer, ids):
        a, p = _ids(ids)
        call("oomb_pagetable_scatter", self.handle, layer, p, len(a))

    def set_tier(self, layer, page, tier):
        call("oomb_pagetable_set_tier", self.handle, layer, page, int(tier))

    def n_pages(self, layer):
        n = C.c_int()
        call("oomb_pagetable_n_pages", self.handle, layer, C.byref(n))
        return n.value

    def page_kv_bytes(self):
        return self.page_kv_bytes_

    def memory_report(self):
        r = OombMemoryReport()
        call("oomb_pagetable_memory_report", self.handle, C.byref(r))
        return r


class TieredEngine:
    def __init__(self, cache, cfg: TierConfig, stream=None):
        c = OombTierConfig(cfg.device_capacity_pages, cfg.bandwidth_bytes_per_s, cfg.compute.fixed_s_per_layer,
                           cfg.compute.s_per_attended_token)
        h = C.c_void_p()
        if isinstance(cache, HostPageTable):
            call("oomb_tier_create_sim", cache.handle, C.byref(c), C.byref(h))
        else:
            from .paged_kv import stream_handle
            call("oomb_tier_create", cache.handle, C.byref(c), stream_handle(stream), C.byref(h))
            cache._enforced = True
        self.handle = h
        self.cache = cache
        self.cfg = cfg

    def close(self, discard: bool = False):
        """Detach (tiered_memory.hpp:110-113). A real engine brings its host-tier pages back into free
        device slots first; pages it cannot bring back (no room) lose their data and are tagged lost
        (tier 3: every later read raises ResidencyError), and close raises ResidencyError saying so
        unless `discard` (the caller drops the pool's contents anyway, e.g. before reset())."""
        if getattr(self, "handle", None):
            L = _lib.lib()
            rc = L.oomb_tier_destroy(self.handle)
            self.handle = None
            if hasattr(self.cache, "_enforced"):
                self.cache._enforced = False
            if rc != 0 and not discard:
                from .errors import raise_for_status
                raise_for_status(rc, L.oomb_last_error().decode(errors="replace"))

    def __del__(self):
        try:
            self.close(discard=True)
        except Exception:  # interpreter shutdown
            pass

    def begin_phase(self, phase: int):
        call("oomb_tier_begin_phase", self.handle, int(phase))

    def set_prefetch_headroom_pages(self, pages: int):
        call("oomb_tier_set_prefetch_headroom", self.handle, pages)

    def on_pages_appended(self, layer: int, slot_range):
        b, e = (slot_range.begin, slot_range.end) if hasattr(slot_range, "begin") else slot_range
        call("oomb_tier_on_pages_appended", self.handle, layer, b, e)

    def on_grads_scattered(self, layer: int, ids):
        a, p = _ids(ids)
        call("oomb_tier_on_grads_scattered", self.handle, layer, p, len(a))

    def fetch_async(self, layer: int, ids, chunk: int = -1, best_effort: bool = False) -> int:
        a, p = _ids(ids)
        h = C.c_int64()
        call("oomb_tier_fetch_async", self.handle, layer, p, len(a), chunk, int(best_effort), C.byref(h))
        return h.value

    def wait(self, handle: int):
        call("oomb_tier_wait", self.handle, handle)

    def record_access(self, layer: int, ids, chunk: int = -1):
        a, p = _ids(ids)
        call("oomb_tier_record_access", self.handle, layer, p, len(a), chunk)

    def advance_compute(self, seconds: float, chunk: int, layer: int):
        call("oomb_tier_advance_compute", self.handle, C.c_double(seconds), chunk, layer)

    def end_layer_use(self, layer: int, ids):
        a, p = _ids(ids)
        call("oomb_tier_end_layer_use", self.handle, layer, p, len(a))

    def release_all_reservations(self):
        call("oomb_tier_release_all", self.handle)

    def restore_all(self):
        """Real engine: bring every host-tier page back to the device (ConfigError without room).
        close() does this when the pool has room, so detaching keeps every page's data."""
        call("oomb_tier_restore_all", self.handle)

    def _stats(self):
        out = (C.c_double * 5)()
        call("oomb_tier_stats", self.handle, out)
        return list(out)

    def now(self):
        return self._stats()[0]

    def stall_seconds(self):
        return self._stats()[1]

    def h2d_bytes(self, phase: int):
        return int(self._stats()[2 + (1 if phase == BACKWARD else 0)])

    def d2h_bytes(self):
        return int(self._stats()[4])

    def _moved(self) -> tuple[int, int]:
        h, d = C.c_int64(), C.c_int64()
        call("oomb_tier_moved_bytes", self.handle, C.byref(h), C.byref(d))
        return h.value, d.value

    def h2d_bytes_moved(self) -> int:
        """Real engine: host->device bytes actually copied (h2d_bytes counts every fetch decision, as the
        reference does; a page fetched back into its still-unused victim slots moves nothing)."""
        return self._moved()[0]

    def d2h_bytes_moved(self) -> int:
        """Real engine: device->host bytes actually copied (d2h_bytes counts every write-back decision;
        a write-back is deferred until the freed slot is about to be reused, and dropped if the page is
        fetched back first)."""
        return self._moved()[1]

    def raw_log(self) -> np.ndarray:
        n = C.c_int64()
        call("oomb_tier_log", self.handle, None, 0, C.byref(n))
        arr = (OombEvent * max(n.value, 1))()
        call("oomb_tier_log", self.handle, arr, n.value, C.byref(n))
        return arr[: n.value]

    def log(self) -> ScheduleLog:
        evs = [ScheduleEvent(EVENT_KINDS[e.kind], e.t, e.layer, e.page, e.chunk, e.bytes,
                             "forward" if e.phase == 0 else "backward") for e in self.raw_log()]
        return ScheduleLog(self.cfg.bandwidth_bytes_per_s, evs)


def validate_schedule(log, bandwidth: float | None = None) -> ValidationReport:
    """tiered_memory.cpp:47-138 over a ScheduleLog or a raw oomb_event array."""
    if isinstance(log, ScheduleLog):
        bw = log.bandwidth_bytes_per_s if bandwidth is None else bandwidth
        arr = (OombEvent * max(len(log.events), 1))()
        for i, e in enumerate(log.events):
            arr[i] = OombEvent(EVENT_KINDS.index(e.kind), e.layer, e.page, e.chunk,
                               0 if e.phase == "forward" else 1, 0, e.bytes, e.t)
        n = len(log.events)
    else:
        arr, n, bw = log, len(log), bandwidth
        arr = (OombEvent * max(n, 1))(*log)
    out = (C.c_double * 6)()
    nv = C.c_int()
    cap = max(n, 1) + 1
    vev = (C.c_int64 * cap)()
    vcode = (C.c_int32 * cap)()
    call("oomb_validate_schedule", arr, n, C.c_double(bw), out, C.byref(nv), vev, vcode, cap)
    msgs = []
    for i in range(min(nv.value, cap)):
        e = arr[vev[i]] if vev[i] >= 0 else None
        msgs.append(_violation_message(vcode[i], e))
    return ValidationReport(msgs, out[0], int(out[1]), int(out[2]), int(out[3]), int(out[4]), out[5])


def _violation_message(code: int, e) -> str:
    """The reference's violation strings (tiered_memory.cpp:50-126)."""
    if code == 1:
        return f"evict of non-resident page layer={e.layer} page={e.page} t={e.t:g}"
    if code == 2:
        return f"access before fetch_done (or after evict): layer={e.layer} page={e.page} t={e.t:g}"
    return {3: "compute stream timestamps decrease", 4: "nested compute_begin", 5: "compute_end without begin",
            6: "compute segment ends before it begins", 7: "unterminated compute segment"}[code]
