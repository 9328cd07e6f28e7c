"""The offload engine's policy on CPU: driven by the same operation scripts, the
simulation-mode engine (liboomb.so, no device) and the reference TieredEngine
(oracle/_ref, tiered_memory.hpp:99-432) must produce identical ScheduleLogs —
same events, pages, byte counts and simulated timestamps — and validate_schedule
must agree with the reference validator (tiered_memory.cpp:47-138)."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import Cfg, Ref, RefEvent
from paper_2602_02108_b200.tiered_memory import (BACKWARD, FORWARD, HostPageTable, OombEvent, TierConfig,
                                                 TieredEngine, validate_schedule)

pytestmark = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref (reference build) not present")


class RefTierCfg(C.Structure):
    _fields_ = [("device_capacity_pages", C.c_int64), ("bandwidth_bytes_per_s", C.c_double),
                ("fixed_s_per_layer", C.c_double), ("s_per_attended_token", C.c_double)]


class RefEngine:
    """The reference TieredEngine over a reference PagedCache, via the shim."""

    def __init__(self, cfg: Cfg, tier: TierConfig):
        self.c = Ref(cfg, 4)
        self.L = self.c.L
        self.cfg = cfg
        self.tier = tier

    def start(self):
        t = RefTierCfg(self.tier.device_capacity_pages, self.tier.bandwidth_bytes_per_s,
                       self.tier.compute.fixed_s_per_layer, self.tier.compute.s_per_attended_token)
        self.c._chk(self.L.ref_tier_new(self.c.h, C.byref(t)))

    def _ids(self, ids):
        a = np.ascontiguousarray(np.asarray(ids, np.int32))
        return a, a.ctypes.data_as(C.c_void_p), len(a)

    def append(self, layer, rows):
        z = np.zeros((rows, self.cfg.n_kv_heads, self.cfg.head_dim), np.float32)
        return self.c.append(layer, z, z)

    def scatter(self, layer, ids):
        g = np.zeros((len(ids) * self.cfg.page_size, self.cfg.n_kv_heads, self.cfg.head_dim), np.float32)
        self.c.scatter(layer, ids, g, g)

    def set_tier(self, layer, page, tier):
        self.c.set_tier(layer, page, tier)

    def n_pages(self, layer):
        return self.c.n_pages(layer)

    def op(self, name, *args):
        L, h = self.L, self.c.h
        if name == "begin_phase":
            rc = L.ref_tier_begin_phase(h, args[0])
        elif name == "headroom":
            rc = L.ref_tier_set_headroom(h, C.c_int64(args[0]))
        elif name == "appended":
            rc = L.ref_tier_on_pages_appended(h, args[0], C.c_int64(args[1]), C.c_int64(args[2]))
        elif name == "grads_scattered":
            a, p, n = self._ids(args[1])
            rc = L.ref_tier_on_grads_scattered(h, args[0], p, n)
        elif name == "fetch":
            a, p, n = self._ids(args[1])
            hh = C.c_int64()
            rc = L.ref_tier_fetch_async(h, args[0], p, n, args[2], int(args[3]), C.byref(hh))
            return rc, hh.value
        elif name == "wait":
            rc = L.ref_tier_wait(h, C.c_int64(args[0]))
        elif name == "access":
            a, p, n = self._ids(args[1])
            rc = L.ref_tier_record_access(h, args[0], p, n, args[2])
        elif name == "compute":
            rc = L.ref_tier_advance_compute(h, C.c_double(args[0]), args[1], args[2])
        elif name == "end_use":
            a, p, n = self._ids(args[1])
            rc = L.ref_tier_end_layer_use(h, args[0], p, n)
        elif name == "release":
            rc = L.ref_tier_release_all(h)
        return rc, None

    def log(self):
        n = self.L.ref_tier_log_size(self.c.h)
        arr = (RefEvent * max(n, 1))()
        self.c._chk(self.L.ref_tier_log(self.c.h, arr))
        return [(e.kind, e.layer, e.page, e.chunk, e.phase, e.bytes, e.t) for e in arr[:n]]

    def stats(self):
        out = (C.c_double * 5)()
        self.L.ref_tier_stats(self.c.h, out)
        return list(out)


class OurEngine:
    def __init__(self, cfg: Cfg, tier: TierConfig):
        self.pt = HostPageTable(cfg.n_layers, cfg.page_size, cfg.n_kv_heads, cfg.head_dim)
        self.cfg = cfg
        self.tier = tier

    def start(self):
        self.e = TieredEngine(self.pt, self.tier)

    def append(self, layer, rows):
        return self.pt.append_chunk(layer, rows)

    def scatter(self, layer, ids):
        self.pt.scatter_add_grads(layer, ids)

    def set_tier(self, layer, page, tier):
        self.pt.set_tier(layer, page, tier)

    def n_pages(self, layer):
        return self.pt.n_pages(layer)

    def op(self, name, *args):
        e = self.e
        try:
            if name == "begin_phase":
                e.begin_phase(args[0])
            elif name == "headroom":
                e.set_prefetch_headroom_pages(args[0])
            elif name == "appended":
                e.on_pages_appended(args[0], (args[1], args[2]))
            elif name == "grads_scattered":
                e.on_grads_scattered(args[0], args[1])
            elif name == "fetch":
                return 0, e.fetch_async(args[0], args[1], args[2], args[3])
            elif name == "wait":
                e.wait(args[0])
            elif name == "access":
                e.record_access(args[0], args[1], args[2])
            elif name == "compute":
                e.advance_compute(args[0], args[1], args[2])
            elif name == "end_use":
                e.end_layer_use(args[0], args[1])
            elif name == "release":
                e.release_all_reservations()
        except Exception as ex:  # error code parity
            return type(ex).__name__, None
        return 0, None

    def log(self):
        return [(e.kind, e.layer, e.page, e.chunk, e.phase, e.bytes, e.t) for e in self.e.raw_log()]

    def stats(self):
        e = self.e
        return [e.now(), e.stall_seconds(), e.h2d_bytes(FORWARD), e.h2d_bytes(BACKWARD), e.d2h_bytes()]


def trainer_script(cfg: Cfg, n_chunks: int, mode: str, seed: int):
    """A chunk-recurrent schedule in the shape of ChunkTrainer::train_step
    (chunk_trainer.hpp:131-186, 328-363, 388-462, 531-571) for the engine alone."""
    rng = np.random.default_rng(seed)
    P, m, L = cfg.page_size, cfg.chunk_size // cfg.page_size, cfg.n_layers
    ops = [("headroom", m), ("begin_phase", FORWARD)]
    sels = {}
    for c in range(n_chunks):
        for l in range(L):
            n_cand = c * m
            if mode == "dense":
                sel = list(range(n_cand))
            elif mode == "local":
                sel = list(range(max(0, n_cand - cfg.local_window), n_cand))
            else:
                k = cfg.budget_pages
                sel = sorted(rng.choice(n_cand, size=min(k, n_cand), replace=False).tolist()) if n_cand else []
            sels[(c, l)] = sel
            ops.append(("compute", 0.25e-3, c, l))
            ops.append(("fetch", l, sel, c, False))
            ops.append(("compute", 0.25e-3, c, l))
            ops.append(("append_rows", l, cfg.chunk_size))
            ops.append(("wait_last",))
            ops.append(("access", l, sel, c))
            ops.append(("compute", 1e-6 * (len(sel) * P + cfg.chunk_size), c, l))
            own = list(range(c * m, (c + 1) * m))
            ops.append(("compute", 0.5e-3, c, l))
            ops.append(("end_use", l, sel + own))
            if l + 1 < L:  # best-effort prefetch of the next layer's cached pages
                ops.append(("fetch", l + 1, sels.get((c, l + 1), sel), c, True))
    ops.append(("release",))
    ops.append(("begin_phase", BACKWARD))
    for c in reversed(range(n_chunks)):
        for l in reversed(range(L)):
            sel = sels[(c, l)]
            own = list(range(c * m, (c + 1) * m))
            ops.append(("fetch", l, sorted(set(sel + own)), c, False))
            ops.append(("wait_last",))
            ops.append(("access", l, sorted(set(sel + own)), c))
            ops.append(("compute", 2e-6 * (len(sel) * P + cfg.chunk_size), c, l))
            if sel:
                ops.append(("scatter", l, sel))
                ops.append(("grads_scattered", l, sel))
            ops.append(("end_use", l, sorted(set(sel + own))))
            if c > 0:
                ops.append(("fetch", l, sels[(c - 1, l)], c - 1, True))
    return ops


def run(engine, ops, pre=None):
    out = []
    last = None
    if pre:
        pre(engine)
    engine.start()
    for op in ops:
        name = op[0]
        if name == "append_rows":
            r = engine.append(op[1], op[2])
            rc, _ = engine.op("appended", op[1], r[0], r[1])
        elif name == "scatter":
            engine.scatter(op[1], op[2])
            rc = 0
        elif name == "wait_last":
            rc, _ = engine.op("wait", last)
        elif name == "fetch":
            rc, h = engine.op("fetch", op[1], op[2], op[3], op[4])
            if rc == 0:
                last = h
        else:
            rc, _ = engine.op(name, *op[1:])
        out.append(0 if rc == 0 else 1)
        if rc != 0:
            break
    return out, engine.log(), engine.stats()


CFG = Cfg(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=8, chunk_size=32, page_size=8, retrieval_budget=16,
          local_window=2)


@pytest.mark.parametrize("mode", ["dense", "local", "topk"])
@pytest.mark.parametrize("capacity", [-1, 24, 14])
@pytest.mark.parametrize("bw", [1e15, 2e7])
def test_schedule_log_matches_reference(mode, capacity, bw):
    tier = TierConfig(device_capacity_pages=capacity, bandwidth_bytes_per_s=bw)
    ops = trainer_script(CFG, 5, mode, seed=capacity + 100)
    a_rc, a_log, a_st = run(OurEngine(CFG, tier), ops)
    b_rc, b_log, b_st = run(RefEngine(CFG, tier), ops)
    assert a_rc == b_rc
    assert len(a_log) == len(b_log)
    for x, y in zip(a_log, b_log):
        assert x == y
    assert a_st == b_st


def test_capacity_error_and_bad_handles_match_reference():
    tier = TierConfig(device_capacity_pages=2, bandwidth_bytes_per_s=1e9)
    ops = trainer_script(CFG, 3, "dense", 0)
    a_rc, _, _ = run(OurEngine(CFG, tier), ops)
    b_rc, _, _ = run(RefEngine(CFG, tier), ops)
    assert a_rc == b_rc and a_rc[-1] == 1  # ConfigError: capacity below the working set
    e = OurEngine(CFG, TierConfig())
    e.start()
    assert e.op("wait", 7)[0] == "StateError"
    assert e.op("fetch", 0, [5], 0, False)[0] == "StateError"


def test_transfer_arithmetic_and_validator():
    """test_tiered_memory.cpp:141-161: 64 host pages over a 1 MB/s link."""
    tier = TierConfig(bandwidth_bytes_per_s=1e6)
    ours, ref = OurEngine(CFG, tier), RefEngine(CFG, tier)

    def pre(e):
        e.append(0, 64 * 8)
        for p in range(64):
            e.set_tier(0, p, 1)

    ops = [("fetch", 0, list(range(64)), -1, False), ("wait_last",)]
    _, la, sa = run(ours, ops, pre)
    _, lb, sb = run(ref, ops, pre)
    assert la == lb and sa == sb
    expect = 64.0 * ours.pt.page_kv_bytes() / 1e6
    assert abs(sa[0] - expect) <= 1e-12 * expect and sa[2] == 64 * ours.pt.page_kv_bytes()
    rep = validate_schedule(ours.e.log())
    refv = (C.c_double * 6)()
    nv = C.c_int()
    arr = (RefEvent * len(lb))(*[RefEvent(k, l, p, c, ph, 0, b, t) for (k, l, p, c, ph, b, t) in lb])
    assert ref.L.ref_validate_schedule(arr, len(lb), C.c_double(1e6), refv, C.byref(nv)) == 0
    assert len(rep.violations) == nv.value == 0
    assert [rep.stall_seconds, rep.transfer_bytes, rep.h2d_bytes_forward, rep.h2d_bytes_backward, rep.d2h_bytes,
            rep.overlap_fraction] == list(refv)


def test_validator_flags_access_before_fetch():
    """test_tiered_memory.cpp:180-205 and the randomized corruption property."""
    rng = np.random.default_rng(0)
    for seed in range(10):
        evs, resident, t = [], {}, 0.0
        accesses = []
        for _ in range(50):
            page = int(rng.integers(0, 6))
            t += 0.001 + 0.001 * rng.random()
            if not resident.get(page):
                evs.append(OombEvent(1, 0, page, -1, 0, 0, 64, t))
                resident[page] = True
            elif rng.random() < 0.3:
                evs.append(OombEvent(2, 0, page, -1, 0, 0, 0, t))
                resident[page] = False
            else:
                evs.append(OombEvent(5, 0, page, -1, 0, 0, 0, t))
                accesses.append(evs[-1])
        assert validate_schedule(evs, 1e9).violations == []
        if accesses:
            rogue = accesses[int(rng.integers(0, len(accesses)))]
            bad = [OombEvent(5, 0, rogue.page, -1, 0, 0, 0, 0.0)] + evs
            v = validate_schedule(bad, 1e9).violations
            assert v and v[0].startswith("access before fetch_done") and f"page={rogue.page}" in v[0]


def test_reports_in_reference_formats():
    """memory_report_to_json (paged_kv.cpp:13-22) and the CLI's retrieval.csv (chunktrain.cpp:115-130)."""
    import io
    from paper_2602_02108_b200.reports import emit_retrieval_csv, memory_report_to_json
    from paper_2602_02108_b200.tiered_memory import HostPageTable
    pt = HostPageTable(n_layers=2, page_size=4, n_kv_heads=1, head_dim=2)
    pt.append_chunk(0, 8)
    pt.scatter_add_grads(0, [1])
    rep = pt.memory_report()
    s = memory_report_to_json(rep)
    assert s == ('{"copied_bytes":0,"device_bytes":%d,"grad_bytes":%d,"host_bytes":0,"pages":2,"reallocs":0}'
                 % (rep.device_bytes, rep.grad_bytes))
    assert rep.device_bytes == 2 * pt.page_kv_bytes() and rep.grad_bytes > 0
    buf = io.StringIO()
    emit_retrieval_csv(buf, 7, [(0, [[[], []], [[], []]]), (1, [[[0, 1], [1]], [[0], []]])])
    assert buf.getvalue() == "7,1,0,2,0\n7,1,0,2,1\n7,1,0,3,1\n7,1,1,2,0\n"


def test_schedule_jsonl_matches_reference_dump():
    """dump_schedule_jsonl (tiered_memory.cpp:28-45) of a simulated engine log, byte for byte the
    reference's own dump of the same events (when the reference shim is built)."""
    import ctypes as C
    import io
    from oracle.oracle import Ref, build_ref
    from paper_2602_02108_b200.reports import dump_schedule_jsonl
    from paper_2602_02108_b200.tiered_memory import HostPageTable, TierConfig, TieredEngine
    pt = HostPageTable(n_layers=1, page_size=4, n_kv_heads=1, head_dim=2)
    eng = TieredEngine(pt, TierConfig(device_capacity_pages=5, bandwidth_bytes_per_s=1e6))
    for chunk in range(4):
        b, e = pt.append_chunk(0, 8)
        eng.on_pages_appended(0, (b, e))
        ids = list(range(max(0, pt.n_pages(0) - 4), pt.n_pages(0) - 2))
        if ids:
            eng.wait(eng.fetch_async(0, ids, chunk))
            eng.record_access(0, ids, chunk)
        eng.advance_compute(1e-4, chunk, 0)
        eng.end_layer_use(0, list(range(pt.n_pages(0))))
    buf = io.StringIO()
    dump_schedule_jsonl(eng.log(), buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == '{"bandwidth_bytes_per_s":1000000.0}' and len(lines) == len(eng.raw_log()) + 1
    if not Ref.available():
        pytest.skip("reference shim not built (oracle/_ref)")
    raw = eng.raw_log()
    L = C.CDLL(build_ref())
    arr = (type(raw[0]) * len(raw))(*raw)
    n = C.c_int64()
    assert L.ref_dump_schedule_jsonl(arr, len(raw), C.c_double(1e6), None, 0, C.byref(n)) == 0
    out = C.create_string_buffer(n.value)
    assert L.ref_dump_schedule_jsonl(arr, len(raw), C.c_double(1e6), out, n.value, C.byref(n)) == 0
    ref = out.raw[: n.value].decode()
    # nlohmann writes the header's double as 1000000.0 too; compare every line exactly
    assert buf.getvalue() == ref, (buf.getvalue()[:300], ref[:300])
