#!/usr/bin/env python
"""bench.py — the OOMB hot path on B200 (BASELINE.json metric).

Workload (BASELINE configs[2], "c3"): Qwen2.5-7B attention shape (28 Q / 4 KV
heads, head_dim 128), page 128, chunk 4096, 1M-token context, page-level top-k
(64 pages per query page = the 8192-token budget). One *step* = one attention
layer over the whole sequence, exactly the unit of SURVEY §8(d):
    for each of the 256 chunks in order: score -> top-k -> append -> forward
    for each chunk in reverse order:     backward (D preprocess, dQ, dK/dV into
                                         the paged fp32 gradient pool) + dM_i read
tokens/s = context / step time. `value` has every input resident in HBM;
`e2e` drives the same public API from pinned HOST buffers with the H2D of each
chunk's q/k/v/dO and the D2H of its out/dq/dk/dv inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5] [--impl reference]
                    [--shard replica|kv] [--offload-cap F] [--no-e2e] [--no-cpu]

The step keeps every dependency of the sequential loop and overlaps what it does not need:
chunk i+1's selection runs on a high-priority stream under chunk i's attention, consecutive
chunks attend on two streams (OOMB_FWD_STREAMS, default 2), and the backward defers dQ joins
(OOMB_BWD_DEFER=1: chunk i-1's dK/dV runs under chunk i's dQ). Results are bitwise those of the
sequential loop (tests/test_gpu_concurrency.py).

Under torchrun (N > 1) every rank runs its own layer-sequence by default (weak scaling: per-GPU
work fixed), timed on the device and reported as the max over ranks; --shard kv splits one
sequence across the ranks by KV-head group instead (strong scaling, NCCL vote all-gather).
The CPU baseline and the offload regime are N = 1 measurements.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train tokens/sec (attn fwd+bwd) at 1M ctx, Qwen2.5-7B shape; % bf16 tensor peak"

CONFIGS = {
    "c3": dict(desc="BASELINE configs[2]: Qwen2.5-7B attention (28Q/4KV, hd 128), page 128, chunk 4096, "
                    "1M context, top-k 64 pages per query page", Hq=28, Hkv=4, hd=128, P=128, C=4096, T=1 << 20,
               mode="topk", budget=8192),
    "c2": dict(desc="BASELINE configs[1]: Qwen2.5-7B attention, page 128, chunk 4096, 128K context, dense",
               Hq=28, Hkv=4, hd=128, P=128, C=4096, T=1 << 17, mode="dense", budget=0),
    "c4": dict(desc="BASELINE configs[3] on one GPU: Qwen2.5-7B attention, page 128, chunk 4096, 4M context, "
                    "top-k 64 pages per query page (the 8-GPU KV-group split is weak-scaled by --gpus)",
               Hq=28, Hkv=4, hd=128, P=128, C=4096, T=1 << 22, mode="topk", budget=8192),
    "c5": dict(desc="BASELINE configs[4] on one GPU: Llama-3-8B attention (32Q/8KV, hd 128), page 256, "
                    "chunk 4096, 512K context, dense", Hq=32, Hkv=8, hd=128, P=256, C=4096, T=1 << 19,
               mode="dense", budget=0),
    "c1": dict(desc="BASELINE configs[0]: tiny 4Q/1KV, hd 64, page 64, chunk 256, 8K context, dense",
               Hq=4, Hkv=1, hd=64, P=64, C=256, T=8192, mode="dense", budget=0),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), \
            float(d["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def workload(cfg):
    """Exact algorithmic counts per chunk."""
    C, P, Hq, hd, T = cfg["C"], cfg["P"], cfg["Hq"], cfg["hd"], cfg["T"]
    m = C // P
    S = T // C
    k = cfg["budget"] // P if cfg["mode"] == "topk" else None
    chunks = []
    for i in range(S):
        n_cand = i * C // P
        per_qp = n_cand if k is None else min(k, n_cand)
        pairs = P * P * m * per_qp + C * (C + 1) // 2          # per head
        triples = C * Hq * n_cand if (k is not None and n_cand > 0) else 0
        chunks.append(dict(n_cand=n_cand, sel=per_qp, pairs=pairs, fwd=4 * hd * Hq * pairs,
                           bwd=10 * hd * Hq * pairs, score=2 * hd * triples, triples=triples))
    return chunks


# ---------------------------------------------------------------------------
# nvidia-smi clock sampler (runs DURING the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[5 + j].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(rows), "reasons": reasons}


# ---------------------------------------------------------------------------
# offload regime (SURVEY §8d "Offload regime")
# ---------------------------------------------------------------------------
OFFLOAD_SLACK = int(os.environ.get("OOMB_OFFLOAD_SLACK", "-1"))  # physical slots above the tier capacity


def low_locality_keys(run, seed: int = 77):
    """Keys whose page means all have the same norm: every page's rows are re-centred on c * u_p
    (u_p a random unit direction, c = 1), so no page wins the vote by its norm and each query
    page's top-k is close to a random draw (the union of a chunk's 32 selections approaches
    SURVEY 8(d)'s ~1,817 pages at 1M), the worst case for residency."""
    import torch
    cfg = run.cfg
    T, P, Hkv, hd = cfg["T"], cfg["P"], cfg["Hkv"], cfg["hd"]
    g = torch.Generator(device=run.dev).manual_seed(seed)
    out = torch.empty(T, Hkv, hd, device=run.dev, dtype=torch.bfloat16)
    step = 1 << 16  # tokens per block (a multiple of P): bounded fp32 temporaries
    for t0 in range(0, T, step):
        n = min(step, T - t0)
        k = torch.randn(n // P, P, Hkv, hd, device=run.dev, generator=g)
        k -= k.mean(1, keepdim=True)
        u = torch.randn(n // P, 1, Hkv, hd, device=run.dev, generator=g)
        k += u / u.norm(dim=-1, keepdim=True)
        out[t0:t0 + n] = k.view(n, Hkv, hd).to(torch.bfloat16)
    return out


def offload_measure(run, cap_frac: float, repeats: int = 5):
    """One layer step through the reference's residency protocol (AttentionChunkLoop +
    TieredEngine, chunk_trainer.hpp:328-363) with the device page pool capped at cap_frac of the
    layer's pages, against the same protocol with an unlimited tier (every page resident, the same
    host decisions, no copies). Exposed copy % = (capped - resident) / capped step time, from the
    MEDIAN of `repeats` alternating runs (all runs reported). The step runs as one native call
    (oomb_layer_step with the engine attached; OOMB_NATIVE_LOOP=0: the Python AttentionChunkLoop,
    the same calls) and is timed with CUDA events on the compute stream, so the host's per-chunk
    wait for the selection's ids shows up as idle time in both arms; the wall clock is reported
    beside it. Two data regimes: the bench's own N(0,1) keys, and
    low-locality keys (low_locality_keys). The capped pool allocates only the tier capacity plus a
    small slack of device slots (the memory the offload saves is real), and the per-chunk union
    of selected pages and the pages the engine moved are reported."""
    import torch
    from paper_2602_02108_b200 import PagedCache
    from paper_2602_02108_b200.chunk_loop import AttentionChunkLoop, layer_stats, layer_step
    from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine
    cfg, C, P = run.cfg, run.cfg["C"], run.cfg["P"]
    n_pages = cfg["T"] // P
    cap = int(cap_frac * n_pages)
    # device slots above the tier capacity: room for one chunk's appends plus the in-flight fetches of
    # the step-ahead prefetch (measured at c3: 4 chunks' pages is too few, 16 is enough)
    slack = OFFLOAD_SLACK if OFFLOAD_SLACK >= 0 else 16 * (C // P)
    slots = min(n_pages, cap + slack)
    # device bytes of one page slot: K + V (bf16) and the dK + dV gradient block (fp32)
    slot_bytes = P * cfg["Hkv"] * cfg["hd"] * (2 * 2 + 2 * 4)

    def step(frac, K, slots=slots):
        use = frac < 1.0
        cache = PagedCache(run.mc, dtype="bf16", max_tokens=cfg["T"], device_capacity_pages=slots if use else -1)
        eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap if use else -1, bandwidth_bytes_per_s=55e9))
        eng.set_prefetch_headroom_pages(C // P)
        loop = AttentionChunkLoop(cache, engine=eng)
        comp = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(comp)
        if NATIVE_LOOP:  # the same protocol in one native call (oomb_layer_step with the engine attached)
            kv = (run.S, C, cfg["Hkv"], cfg["hd"])
            layer_step(cache, 0, run.q_all, K.view(kv), run.v_all.view(kv), run.do_all, run.o_all, run.lse_all,
                       run.grads, mode=cfg["mode"])
        else:
            for i in range(run.S):
                nq = run.q[(i + 1) % run.RQ] if i + 1 < run.S else None  # selection one chunk ahead
                loop.forward_chunk(i, run.q[i % run.RQ], K[i * C:(i + 1) * C], run.v_all[i * C:(i + 1) * C],
                                   next_q=nq, out=run.o_all[i], lse=run.lse_all[i])
            loop.begin_backward()
            for i in reversed(range(run.S)):
                loop.backward_chunk(i, run.do[i % run.RQ], run.q[i % run.RQ], K[i * C:(i + 1) * C],
                                    run.v_all[i * C:(i + 1) * C], grads=run.grads)
        e1.record(comp)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        # device time of the step on the compute stream (the host's per-chunk fetch decisions show up
        # as idle gaps in it); the wall clock is reported beside it
        out = {"wall_s": wall, "gpu_s": e0.elapsed_time(e1) / 1e3}
        kv_page = cache.page_kv_bytes()
        st = layer_stats(cache) if NATIVE_LOOP else loop.chunk_stats
        fw = [x for x in st if x[0] == "fwd" and x[1] > 0]
        bw = [x for x in st if x[0] == "bwd"]
        out.update(h2d_bytes=eng.h2d_bytes(0) + eng.h2d_bytes(1), d2h_bytes=eng.d2h_bytes(),
                   h2d_bytes_moved=eng.h2d_bytes_moved(), d2h_bytes_moved=eng.d2h_bytes_moved(),
                   fwd_union=[x[2] for x in fw], fwd_fetch_pages=[x[3] / kv_page for x in fw],
                   bwd_h2d=[x[3] for x in bw], bwd_d2h=[x[4] for x in bw],
                   device_bytes=(slots if use else n_pages) * slot_bytes)
        eng.release_all_reservations()
        eng.close(discard=True)  # the measurement is over: host-tier pages are not needed
        del loop, eng, cache
        torch.cuda.empty_cache()
        return out

    def regime(K, slots=slots):
        step(1.0, K)  # warm-up of the loop path
        step(cap_frac, K, slots)  # and of the engine path (first pinned-tier use)
        runs = [(step(1.0, K), step(cap_frac, K, slots)) for _ in range(repeats)]  # alternating
        res = [r["gpu_s"] for r, _ in runs]
        off = [o["gpu_s"] for _, o in runs]
        o = runs[-1][1]
        mres, moff = statistics.median(res), statistics.median(off)
        fu = o["fwd_union"]
        return {"step_s_capped_runs": off, "step_s_resident_runs": res,
                "step_s_capped_median": moff, "step_s_resident_median": mres,
                "wall_s_capped_runs": [x["wall_s"] for _, x in runs],
                "wall_s_resident_runs": [x["wall_s"] for x, _ in runs],
                "resident_moved_bytes": runs[-1][0]["h2d_bytes"] + runs[-1][0]["d2h_bytes"],
                "exposed_pct": 100.0 * (moff - mres) / moff,
                "exposed_pct_runs": [100.0 * (a - b) / a for a, b in zip(off, res)],
                "h2d_bytes": o["h2d_bytes"], "d2h_bytes": o["d2h_bytes"], "h2d_bytes_moved": o["h2d_bytes_moved"],
                "d2h_bytes_moved": o["d2h_bytes_moved"],
                "fwd_union_pages_per_chunk": {"mean": statistics.mean(fu), "median": statistics.median(fu),
                                              "max": max(fu), "last": fu[-1]} if fu else None,
                "fwd_fetched_pages_per_chunk": {"mean": statistics.mean(o["fwd_fetch_pages"]),
                                                "max": max(o["fwd_fetch_pages"])} if fu else None,
                "bwd_bytes_per_chunk": {"h2d_mean": statistics.mean(o["bwd_h2d"]),
                                        "d2h_mean": statistics.mean(o["bwd_d2h"])},
                "pool_bytes_capped": o["device_bytes"], "pool_bytes_resident": runs[-1][0]["device_bytes"]}

    bench_data = regime(run.k_all)
    lowloc, sweep = None, []
    if cfg["mode"] == "topk":
        K = low_locality_keys(run)
        lowloc = regime(K)
        # more physical slots than the tier's capacity: the extra slots keep evicted pages' data as
        # victims (a page fetched back before its slot is reused moves nothing), trading device memory
        # for copies at the same engine decisions
        for extra in (2, 3):
            sl = min(n_pages, cap + extra * slack)
            if sl < n_pages:
                r = regime(K, sl)
                sweep.append({"device_slots": sl, "pool_bytes": sl * slot_bytes, "exposed_pct": r["exposed_pct"],
                              "exposed_pct_runs": r["exposed_pct_runs"], "h2d_bytes_moved": r["h2d_bytes_moved"],
                              "d2h_bytes_moved": r["d2h_bytes_moved"]})
        del K
        torch.cuda.empty_cache()
    return {"capacity_frac": cap_frac, "capacity_pages": cap, "device_slots": slots, "layer_pages": n_pages,
            "exposed_pct": bench_data["exposed_pct"], "h2d_bytes": bench_data["h2d_bytes"],
            "d2h_bytes": bench_data["d2h_bytes"], "bench_data": bench_data, "low_locality": lowloc,
            "low_locality_slot_sweep": sweep,
            "note": "exposed_pct = median capped vs median resident (unlimited tier, same protocol) step time, "
                    "CUDA events on the compute stream, over alternating runs (all runs listed). "
                    "The capped pool holds capacity + slack device page slots (pool_bytes_capped vs "
                    "pool_bytes_resident). bench_data: the bench's N(0,1) keys, whose K_avg norms make a "
                    "shared hot set that LRU keeps resident; low_locality: every page mean at the same norm, "
                    "near-random selections. Pinned-host page moves on side streams (one batched copy per "
                    "engine operation); each chunk's selection is issued one chunk ahead. h2d_bytes counts every "
                    "fetch decision (the reference's accounting); h2d_bytes_moved what was copied (a page fetched "
                    "back into its not-yet-reused victim slots moves nothing). low_locality_slot_sweep: the same "
                    "tier capacity with more physical slots."}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
SEL_PRIORITY = os.environ.get("OOMB_SEL_PRIORITY", "1") != "0"
# consecutive chunks' attention forwards on two streams (they are independent: see forward_pass)
FWD_STREAMS = int(os.environ.get("OOMB_FWD_STREAMS", "2"))
# backward with deferred dQ joins: chunk i-1's dK/dV overlaps chunk i's dQ (OOMB_ATTN_DEFER_DQ)
BWD_DEFER = os.environ.get("OOMB_BWD_DEFER", "1") != "0"
# the unsplit layer step through the native loop (oomb_layer_step); 0: the Python chunk loop
NATIVE_LOOP = os.environ.get("OOMB_NATIVE_LOOP", "1") != "0"


def bench_inputs(cfg, seed: int, device, rq: int = 16):
    """The bench's synthetic inputs: N(0,1) keys / values for the whole context and `rq` distinct
    query / dO chunks, rounded to bf16 (tests/test_gpu_bench_data.py checks selection on exactly these)."""
    import torch
    C, Hq, Hkv, hd, T = cfg["C"], cfg["Hq"], cfg["Hkv"], cfg["hd"], cfg["T"]
    g = torch.Generator(device=device).manual_seed(seed)
    bf = torch.bfloat16
    k_all = torch.randn(T, Hkv, hd, device=device, generator=g).to(bf)
    v_all = torch.randn(T, Hkv, hd, device=device, generator=g).to(bf)
    q = torch.empty(rq, C, Hq, hd, device=device, dtype=bf)  # contiguous: the native loop's [Rq][C][Hq][hd]
    do = torch.empty(rq, C, Hq, hd, device=device, dtype=bf)
    for i in range(rq):
        q[i] = torch.randn(C, Hq, hd, device=device, generator=g).to(bf)
    for i in range(rq):
        do[i] = torch.randn(C, Hq, hd, device=device, generator=g).to(bf)
    return k_all, v_all, q, do


class Run:
    RQ = 16  # distinct q / dO chunk buffers (K/V are distinct for every chunk)

    def __init__(self, cfg, seed: int, device, layer=None):
        import torch
        from paper_2602_02108_b200 import ModelConfig, PagedCache
        from paper_2602_02108_b200 import attention as A
        self.torch, self.A = torch, A
        self.cfg = cfg
        self.dev = device
        C, P, Hq, Hkv, hd, T = cfg["C"], cfg["P"], cfg["Hq"], cfg["Hkv"], cfg["hd"], cfg["T"]
        self.S, self.m = T // C, C // P
        self.mc = ModelConfig(n_layers=1, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=hd, chunk_size=C, page_size=P,
                              retrieval_budget=cfg["budget"], attention_mode=[cfg["mode"]])
        # a rank of a split sequence (sharding.ShardedLayer): its KV groups' heads, and K/V + gradient
        # storage only for its page range's pages
        self.layer = layer
        self.cache = (PagedCache(self.mc, dtype="bf16", max_tokens=T) if layer is None else
                      layer.attach(layer.plan.make_cache(layer.cfg, dtype="bf16", max_tokens=T)))
        self.k_all, self.v_all, self.q_all, self.do_all = bench_inputs(cfg, seed, device, self.RQ)
        self.q, self.do = list(self.q_all), list(self.do_all)  # per-chunk views
        bf = torch.bfloat16
        self.o_all = torch.empty(self.S, C, Hq, hd, device=device, dtype=bf)
        self.lse_all = torch.empty(self.S, C, Hq, device=device, dtype=torch.float32)
        kmax = self.m * (cfg["budget"] // P if cfg["mode"] == "topk" else T // P)
        self.sels = [A.Selection(self.cache, self.m, kmax) for _ in range(self.S)]
        self.vote = torch.empty(self.m * max(T // P, 1), device=device, dtype=torch.float32)
        self.grads = A.AttnGrads(torch.empty(C, Hq, hd, device=device), torch.empty(C, Hkv, hd, device=device),
                                 torch.empty(C, Hkv, hd, device=device))
        self.own = [np.arange(i * self.m, (i + 1) * self.m, dtype=np.int32) for i in range(self.S)]
        if layer is not None:
            # per-group partial votes (exchanged over the ranks of the same page range), the owned part
            # of each selection, partial (O, LSE) buffers per attention stream and a ring of two flat
            # [dq | dk | dv] buffers whose ordered reduction overlaps the next chunk's backward
            self.parts = torch.empty(Hkv * self.m * max(T // P, 1), device=device, dtype=torch.float32)
            self.subs = [A.Selection(self.cache, self.m, kmax) for _ in range(self.S)]
            self.o_part = [torch.empty(C, Hq, hd, device=device, dtype=bf) for _ in range(2)]
            self.lse_part = [torch.empty(C, Hq, device=device, dtype=torch.float32) for _ in range(2)]
            n_flat = C * Hq * hd + 2 * C * Hkv * hd
            self.flat = [torch.empty(n_flat, device=device) for _ in range(2)]
            self.flat_grads = [A.AttnGrads(f[:C * Hq * hd].view(C, Hq, hd),
                                           f[C * Hq * hd:C * Hq * hd + C * Hkv * hd].view(C, Hkv, hd),
                                           f[C * Hq * hd + C * Hkv * hd:].view(C, Hkv, hd)) for f in self.flat]
            self.comm_stream = torch.cuda.Stream(device=device)
            self.ev_part = [None, None]   # merge that last read o_part[b]
            self.ev_flat = [None, None]   # reduction that last used flat[b]
        self.fwd_phase = []  # (start, end) CUDA events of every step's forward pass
        self.bwd_phase = []  # and of its backward pass

    def _select(self, i, q, stream=None):
        from paper_2602_02108_b200._lib import call
        from paper_2602_02108_b200.paged_kv import stream_handle
        n_cand = i * self.m
        if self.layer is not None:
            self.layer.select(i, q, self.sels[i], self.subs[i], vote_buf=self.vote, parts_buf=self.parts,
                              stream=stream)
        elif self.cfg["mode"] == "topk" and n_cand > 0:
            self.A.select_pages_topk(self.cache, 0, q, n_cand, stream=stream, out=self.sels[i], vote=self.vote)
        else:  # dense (select_all) or no candidates yet (chunk_trainer.hpp:297-304)
            call("oomb_select_all", self.sels[i].handle, n_cand, self.m, stream_handle(stream))

    def fwd_chunk(self, i, q, k, v, out=None, stream=None):
        self._select(i, q, stream)
        self.cache.append_chunk(0, k, v, stream=stream)
        return self.attend(i, q, k, v, stream, out=self.o_all[i] if out is None else out)

    def attend(self, i, q, k, v, stream, out=None):
        """Chunk i's attention forward on `stream`; on a page-range shard the partial (O, LSE) of the
        rank's pages is merged over its range group on the comm stream (writes o_all[i] / lse_all[i])."""
        torch = self.torch
        out = self.o_all[i] if out is None else out
        if self.layer is None or not self.layer.split_pages:
            sel = self.sels[i]
            return self.A.attn_forward(self.mc, q, self.cache, 0, sel, k, v, stream=stream, out=out,
                                       lse=self.lse_all[i])
        b = i & 1
        st = stream if stream is not None else torch.cuda.current_stream()
        if self.ev_part[b] is not None:
            st.wait_event(self.ev_part[b])  # the merge that last read this partial buffer is done
        part = self.A.attn_forward(self.mc, q, self.cache, 0, self.subs[i], k, v, stream=st, out=self.o_part[b],
                                   lse=self.lse_part[b], past_only=self.layer.plan.range_idx != 0)
        cs = self.comm_stream
        cs.wait_stream(st)
        self.layer.range_comm.lse_merge(part.out, part.lse, stream=cs, out=out, lse=self.lse_all[i])
        ev = torch.cuda.Event()
        ev.record(cs)
        self.ev_part[b] = ev
        return self.A.AttnSaved(out, self.lse_all[i], self.subs[i])

    def bwd_chunk(self, i, do, q, k, v, grads=None, stream=None, defer_dq=False):
        torch = self.torch
        if self.layer is not None and self.layer.split_pages:
            # page-range shard: backward into a ring buffer, then the ordered reduction of
            # [dq | dk_cur | dv_cur] over the range group on the comm stream (it waits for the deferred dQ)
            b = i & 1
            st = stream if stream is not None else torch.cuda.current_stream()
            if self.ev_flat[b] is not None:
                st.wait_event(self.ev_flat[b])
            g = self.flat_grads[b]
            saved = self.A.AttnSaved(self.o_all[i], self.lse_all[i], self.subs[i])
            self.A.attn_backward(self.mc, do, q, self.cache, 0, k, v, saved, stream=st, grads=g,
                                 defer_dq=defer_dq, past_only=self.layer.plan.range_idx != 0)
            self.cache.accumulate_grad_pages(0, self.own[i], g.dk_cur, g.dv_cur, stream=st)
            cs = self.comm_stream
            cs.wait_stream(st)
            if defer_dq:
                self.A.join_dq(self.cache, cs)
            self.layer.range_comm.allreduce_ordered(self.flat[b], stream=cs, out=self.flat[b])
            ev = torch.cuda.Event()
            ev.record(cs)
            self.ev_flat[b] = ev
            return g
        g = self.grads if grads is None else grads
        saved = self.A.AttnSaved(self.o_all[i], self.lse_all[i], self.sels[i])
        self.A.attn_backward(self.mc, do, q, self.cache, 0, k, v, saved, stream=stream, grads=g, defer_dq=defer_dq)
        self.cache.accumulate_grad_pages(0, self.own[i], g.dk_cur, g.dv_cur, stream=stream)
        return g

    def join_comm(self, stream):
        if self.layer is not None and self.layer.split_pages:
            stream.wait_stream(self.comm_stream)

    def forward_pass(self):
        """All chunks' [select -> append -> attend], with chunk i+1's page selection (score + top-k,
        which needs only the K_avg of chunks <= i) on a second stream, overlapping chunk i's attention.
        Same work and dependencies as the sequential loop."""
        torch, C = self.torch, self.cfg["C"]
        comp = torch.cuda.current_stream()
        if not hasattr(self, "sel_stream"):
            # high priority: the selection's CTAs are scheduled ahead of the running attention's
            # remaining ones, so chunk i+1's ids are ready before chunk i's attention drains
            self.sel_stream = torch.cuda.Stream(priority=-1 if SEL_PRIORITY else 0)
            self.ev_app = [torch.cuda.Event() for _ in range(2)]
            self.ev_sel = [torch.cuda.Event() for _ in range(2)]
        ss = self.sel_stream
        ss.wait_stream(comp)  # the cache reset / previous work precede this step's selections
        if FWD_STREAMS > 1 and not hasattr(self, "att_streams"):
            self.att_streams = [torch.cuda.Stream() for _ in range(FWD_STREAMS)]
            self.ev_att = [torch.cuda.Event() for _ in range(FWD_STREAMS)]
        for st in getattr(self, "att_streams", []):
            st.wait_stream(comp)
        for i in range(self.S):
            q, k, v = self.q[i % self.RQ], self.k_all[i * C:(i + 1) * C], self.v_all[i * C:(i + 1) * C]
            if i > 0:
                ss.wait_event(self.ev_app[(i - 1) & 1])  # K_avg of every earlier chunk is in
            self._select(i, q, stream=ss)
            self.ev_sel[i & 1].record(ss)
            self.cache.append_chunk(0, k, v, stream=comp)
            self.ev_app[i & 1].record(comp)
            # chunk i's attention reads pages of chunks < i (appended above, before the selection
            # that chose them) and its own k/v: it does not depend on chunk i-1's attention, so with
            # FWD_STREAMS > 1 consecutive chunks attend concurrently and fill each other's tail wave
            ast = comp if FWD_STREAMS <= 1 else self.att_streams[i % FWD_STREAMS]
            if ast is not comp:
                ast.wait_event(self.ev_app[i & 1])
            ast.wait_event(self.ev_sel[i & 1])
            self.attend(i, q, k, v, ast)
        for st in getattr(self, "att_streams", []):
            comp.wait_stream(st)
        comp.wait_stream(ss)
        self.join_comm(comp)

    def step(self):
        torch, C = self.torch, self.cfg["C"]
        self.cache.reset()
        comp = torch.cuda.current_stream()
        f0, b0, b1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        if NATIVE_LOOP and self.layer is None:
            # the whole layer step in native code (oomb_layer_step): the same work, streams and order
            # as forward_pass + the reverse bwd_chunk loop below, without ~10 host calls per chunk
            from paper_2602_02108_b200.chunk_loop import layer_step
            cfg = self.cfg
            kv = (self.S, C, cfg["Hkv"], cfg["hd"])
            args = (self.cache, 0, self.q_all, self.k_all.view(kv), self.v_all.view(kv), self.do_all, self.o_all,
                    self.lse_all, self.grads)
            f0.record(comp)
            layer_step(*args, mode=cfg["mode"], phase="forward")
            b0.record(comp)
            layer_step(*args, mode=cfg["mode"], phase="backward")
            b1.record(comp)
            self.fwd_phase.append((f0, b0))
            self.bwd_phase.append((b0, b1))
            return
        f0.record(comp)
        self.forward_pass()
        b0.record(comp)
        for i in reversed(range(self.S)):
            # with BWD_DEFER the stream does not wait for chunk i's dQ (it runs on the library's
            # side stream): chunk i-1's prep and dK/dV start under it; the grads buffers are
            # reused, so only the last chunk's dQ survives the step (it is not read here)
            self.bwd_chunk(i, self.do[i % self.RQ], self.q[i % self.RQ], self.k_all[i * C:(i + 1) * C],
                           self.v_all[i * C:(i + 1) * C], defer_dq=BWD_DEFER)
        if BWD_DEFER:
            self.A.join_dq(self.cache, comp)
        self.join_comm(comp)
        b1.record(comp)
        self.fwd_phase.append((f0, b0))
        self.bwd_phase.append((b0, b1))


NB = 3  # e2e staging depth


class E2E:
    """Same step through the public API, inputs from pinned host memory: per chunk
    H2D(q, k, v) before the forward, D2H(out) after it; H2D(dO, q, k, v) before the
    backward, D2H(dq, dk_cur, dv_cur) after it. Copies run on side streams one chunk
    ahead (NB-deep device staging, so a slow read-out of chunk i-NB is the only thing chunk i's
    kernels can wait for) so they overlap the kernels."""

    def __init__(self, run: Run):
        torch = run.torch
        self.r = run
        self.torch = torch
        cfg = run.cfg
        C, Hq, Hkv, hd = cfg["C"], cfg["Hq"], cfg["Hkv"], cfg["hd"]
        pin = dict(pin_memory=True)
        self.k_h = run.k_all.cpu().pin_memory()
        self.v_h = run.v_all.cpu().pin_memory()
        self.q_h = [x.cpu().pin_memory() for x in run.q]
        self.do_h = [x.cpu().pin_memory() for x in run.do]
        bf = torch.bfloat16
        self.out_h = [torch.empty(C, Hq, hd, dtype=bf, **pin) for _ in range(NB)]
        self.dq_h = [torch.empty(C, Hq, hd, **pin) for _ in range(NB)]
        self.dk_h = [torch.empty(C, Hkv, hd, **pin) for _ in range(NB)]
        self.dv_h = [torch.empty(C, Hkv, hd, **pin) for _ in range(NB)]
        d = run.dev
        self.qd = [torch.empty(C, Hq, hd, dtype=bf, device=d) for _ in range(NB)]
        self.dod = [torch.empty(C, Hq, hd, dtype=bf, device=d) for _ in range(NB)]
        self.kd = [torch.empty(C, Hkv, hd, dtype=bf, device=d) for _ in range(NB)]
        self.vd = [torch.empty(C, Hkv, hd, dtype=bf, device=d) for _ in range(NB)]
        self.gd = [run.A.AttnGrads(torch.empty(C, Hq, hd, device=d), torch.empty(C, Hkv, hd, device=d),
                                   torch.empty(C, Hkv, hd, device=d)) for _ in range(NB)]
        self.h2d = torch.cuda.Stream(device=d)
        self.d2h = torch.cuda.Stream(device=d)
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        # small steps (c1: 32 chunks of 256 tokens) through the native layer loop with whole-step
        # copies: the per-chunk Python loop above would make the host, not the copies, the bound
        S = run.S
        self.native = (NATIVE_LOOP and run.layer is None and
                       S * C * (Hq + 2 * Hkv) * hd * 4 <= (256 << 20))
        if self.native:
            RQ = run.RQ
            self.qa_h = run.q_all.cpu().pin_memory()
            self.doa_h = run.do_all.cpu().pin_memory()
            self.qa_d, self.doa_d = torch.empty_like(run.q_all), torch.empty_like(run.do_all)
            self.ka_d, self.va_d = torch.empty_like(run.k_all), torch.empty_like(run.v_all)
            self.ga = run.A.AttnGrads(torch.empty(S, C, Hq, hd, device=d), torch.empty(S, C, Hkv, hd, device=d),
                                      torch.empty(S, C, Hkv, hd, device=d))
            self.oa_h = torch.empty(S, C, Hq, hd, dtype=bf, **pin)
            self.lsea_h = torch.empty(S, C, Hq, **pin)
            self.ga_h = [torch.empty(S, C, Hq, hd, **pin), torch.empty(S, C, Hkv, hd, **pin),
                         torch.empty(S, C, Hkv, hd, **pin)]
            self.ev_in = torch.cuda.Event()

    def step_native(self):
        """Every step: H2D of the step's q / dO blocks and K / V from pinned memory, the native layer
        step (chunk_loop.layer_step, every chunk's dq / dk_cur / dv_cur kept), D2H of out, lse and
        the gradients."""
        from paper_2602_02108_b200.chunk_loop import layer_step
        torch, r = self.torch, self.r
        cfg, C, S = r.cfg, r.cfg["C"], r.S
        comp = torch.cuda.current_stream()
        r.cache.reset()
        with torch.cuda.stream(self.h2d):
            self.h2d.wait_stream(comp)
            for dst, src in ((self.qa_d, self.qa_h), (self.doa_d, self.doa_h), (self.ka_d, self.k_h),
                             (self.va_d, self.v_h)):
                dst.copy_(src, non_blocking=True)
            self.ev_in.record(self.h2d)
        comp.wait_event(self.ev_in)
        kv = (S, C, cfg["Hkv"], cfg["hd"])
        layer_step(r.cache, 0, self.qa_d, self.ka_d.view(kv), self.va_d.view(kv), self.doa_d, r.o_all, r.lse_all,
                   self.ga, mode=cfg["mode"], grad_stride_chunks=1)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_stream(comp)
            for dst, src in ((self.oa_h, r.o_all), (self.lsea_h, r.lse_all), (self.ga_h[0], self.ga.dq),
                             (self.ga_h[1], self.ga.dk_cur), (self.ga_h[2], self.ga.dv_cur)):
                dst.copy_(src, non_blocking=True)
        comp.wait_stream(self.d2h)
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in (self.qa_h, self.doa_h, self.k_h, self.v_h))
        self.d2h_bytes = sum(t.numel() * t.element_size() for t in (self.oa_h, self.lsea_h, *self.ga_h))

    def step(self):
        if self.native:
            return self.step_native()
        torch, r = self.torch, self.r
        C = r.cfg["C"]
        comp = torch.cuda.current_stream()
        S = r.S
        r.cache.reset()
        h2d_b = d2h_b = 0
        ev_in = [torch.cuda.Event() for _ in range(NB)]
        ev_used = [torch.cuda.Event() for _ in range(NB)]
        ev_out = [torch.cuda.Event() for _ in range(NB)]
        for e in ev_used + ev_out:
            e.record(comp)

        def load_fwd(i):
            nonlocal h2d_b
            b = i % NB
            with torch.cuda.stream(self.h2d):
                self.h2d.wait_event(ev_used[b])
                self.qd[b].copy_(self.q_h[i % r.RQ], non_blocking=True)
                self.kd[b].copy_(self.k_h[i * C:(i + 1) * C], non_blocking=True)
                self.vd[b].copy_(self.v_h[i * C:(i + 1) * C], non_blocking=True)
                ev_in[b].record(self.h2d)
            h2d_b += 2 * (self.qd[b].numel() + 2 * self.kd[b].numel())

        load_fwd(0)
        # as Run.forward_pass: chunk i+1's selection on a second stream overlaps chunk i's attention
        if not hasattr(self, "ss"):
            self.ss = torch.cuda.Stream(device=r.dev, priority=-1 if SEL_PRIORITY else 0)
            self.att = [torch.cuda.Stream(device=r.dev) for _ in range(max(FWD_STREAMS, 1))]
        ss = self.ss
        for st in self.att:
            st.wait_stream(comp)
        ev_app = [torch.cuda.Event() for _ in range(NB)]
        ev_sel = [torch.cuda.Event() for _ in range(NB)]
        ss.wait_stream(comp)
        for i in range(S):
            b = i % NB
            if i + 1 < S:
                load_fwd(i + 1)
            ss.wait_event(ev_in[b])
            if i > 0:
                ss.wait_event(ev_app[(i - 1) % NB])  # K_avg of every earlier chunk is in
            r._select(i, self.qd[b], stream=ss)
            ev_sel[b].record(ss)
            comp.wait_event(ev_in[b])
            comp.wait_event(ev_out[b])  # the D2H that last read out slot b finished
            r.cache.append_chunk(0, self.kd[b], self.vd[b], stream=comp)
            ev_app[b].record(comp)
            # as Run.forward_pass: consecutive chunks attend on alternating streams
            ast = self.att[i % len(self.att)]
            ast.wait_event(ev_app[b])
            ast.wait_event(ev_sel[b])  # (the selection read qd[b] too: ev_used below covers it)
            r.attend(i, self.qd[b], self.kd[b], self.vd[b], ast)
            ev_used[b].record(ast)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(ev_used[b])
                r.join_comm(self.d2h)  # a page-range shard's merged out is written on the comm stream
                self.out_h[b].copy_(r.o_all[i], non_blocking=True)
                ev_out[b].record(self.d2h)
            d2h_b += 2 * r.o_all[i].numel()
        for st in self.att:
            comp.wait_stream(st)
        r.join_comm(comp)

        def load_bwd(i):
            nonlocal h2d_b
            b = i % NB
            with torch.cuda.stream(self.h2d):
                self.h2d.wait_event(ev_used[b])
                if BWD_DEFER:  # the deferred dQ of the chunk that last used slot b read its inputs too
                    r.A.join_dq(r.cache, self.h2d)
                self.dod[b].copy_(self.do_h[i % r.RQ], non_blocking=True)
                self.qd[b].copy_(self.q_h[i % r.RQ], non_blocking=True)
                self.kd[b].copy_(self.k_h[i * C:(i + 1) * C], non_blocking=True)
                self.vd[b].copy_(self.v_h[i * C:(i + 1) * C], non_blocking=True)
                ev_in[b].record(self.h2d)
            h2d_b += 2 * (2 * self.qd[b].numel() + 2 * self.kd[b].numel())

        order = list(reversed(range(S)))
        load_bwd(order[0])
        for n, i in enumerate(order):
            b = i % NB
            if n + 1 < S:
                load_bwd(order[n + 1])
            comp.wait_event(ev_in[b])
            comp.wait_event(ev_out[b])
            g = r.bwd_chunk(i, self.dod[b], self.qd[b], self.kd[b], self.vd[b], grads=self.gd[b], defer_dq=BWD_DEFER)
            ev_used[b].record(comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(ev_used[b])
                if BWD_DEFER:
                    r.A.join_dq(r.cache, self.d2h)  # dq(i) ran on the library's side stream
                r.join_comm(self.d2h)  # a page-range shard reduces its grads on the comm stream
                self.dq_h[b].copy_(g.dq, non_blocking=True)
                self.dk_h[b].copy_(g.dk_cur, non_blocking=True)
                self.dv_h[b].copy_(g.dv_cur, non_blocking=True)
                ev_out[b].record(self.d2h)
            d2h_b += 4 * (g.dq.numel() + 2 * g.dk_cur.numel())
        if BWD_DEFER:
            r.A.join_dq(r.cache, comp)
        r.join_comm(comp)
        comp.wait_stream(self.d2h)
        self.h2d_bytes, self.d2h_bytes = h2d_b, d2h_b


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the reference's own code; else the C port)
# ---------------------------------------------------------------------------
def _cpu_sample(args):
    """One bounded slice of the c3 workload through the reference functions: the
    last query page of a chunk over 64 selected pages + its causal prefix, one KV
    group (7 q-heads), fwd + bwd; and score_pages of 128 tokens x 7 heads over 512
    candidates. Returns (attn seconds, pair-heads, score seconds, triples)."""
    seed, hd, P, G, n_sel, n_score, kind = args
    sys.path.insert(0, ROOT)
    from oracle.oracle import Cfg, Port, Ref, det_normal
    B = Ref if kind == "reference" else Port
    c = Cfg(n_layers=1, n_q_heads=G, n_kv_heads=1, head_dim=hd, chunk_size=P, page_size=P,
            retrieval_budget=n_sel * P)
    o = B(c, 4)
    pk = det_normal(seed * 8 + 1, (n_sel * P, 1, hd))
    o.append(0, pk, det_normal(seed * 8 + 2, (n_sel * P, 1, hd)))
    q = det_normal(seed * 8 + 3, (P, G, hd))
    kc = det_normal(seed * 8 + 4, (P, 1, hd))
    vc = det_normal(seed * 8 + 5, (P, 1, hd))
    do = det_normal(seed * 8 + 6, (P, G, hd))
    o.append(0, kc, vc)
    sel = [list(range(n_sel))]
    t0 = time.perf_counter()
    out, lse = o.attn_forward(0, q, sel, kc, vc)
    o.attn_backward(0, do, q, sel, kc, vc, out, lse)
    t_attn = time.perf_counter() - t0
    pair_heads = G * (P * n_sel * P + P * (P + 1) // 2)
    kav = det_normal(seed * 8 + 7, (n_score, 1, hd))
    t0 = time.perf_counter()
    o.score_pages(q, kav)
    t_score = time.perf_counter() - t0
    return t_attn, pair_heads, t_score, P * G * n_score


def cpu_baseline(cfg, max_workers=None, n_sel=64, n_score=512):
    """Time the reference CPU path on this host's cores and scale by the exact
    pair / triple counts of the workload. Returns the cpu_baseline object."""
    import multiprocessing as mp
    from oracle.oracle import Ref, build_port
    kind = "reference" if Ref.available() else "port"
    build_port()
    cores = os.cpu_count() or 1
    workers = max(1, min(cores, max_workers or cores))
    G = cfg["Hq"] // cfg["Hkv"]
    P = min(cfg["P"], 128)
    n_sel = min(n_sel, max(1, cfg["T"] // cfg["P"] // 4))
    jobs = [(s, cfg["hd"], P, G, n_sel, n_score, kind) for s in range(workers)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(workers) as pool:
        res = pool.map(_cpu_sample, jobs)
    wall = time.perf_counter() - t0
    # per-core effective costs under full load
    c_pair = statistics.mean(r[0] / r[1] for r in res)
    c_tri = statistics.mean(r[2] / r[3] for r in res)
    chunks = workload(cfg)
    core_seconds = sum(ch["pairs"] * cfg["Hq"] * c_pair + ch["triples"] * c_tri for ch in chunks)
    tok_s = cfg["T"] / (core_seconds / workers)
    return {"value": tok_s, "unit": "tokens/s", "cores": workers, "kind": kind,
            "sample": (f"{workers} parallel processes x [1 query page (P={P}) x {G} q-heads over {n_sel} selected "
                       f"pages + causal prefix, fwd+bwd; score_pages {P} tokens x {G} heads x {n_score} pages], "
                       f"scaled by the exact pair/triple counts of the workload"),
            "ns_per_pair_head": c_pair * 1e9, "ns_per_score_triple": c_tri * 1e9, "sample_wall_s": wall}


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="oomb", choices=["oomb", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-workers", type=int, default=None)
    ap.add_argument("--tokens", type=int, default=None, help="override the context length (debug)")
    ap.add_argument("--shard", default="auto",
                    help="auto (default): at N > 1 ONE sequence is split across the ranks by KV-head group and, "
                         "when the groups run out, by page range (sharding.ShardPlan: Qwen 8 GPUs = 4 x 2; strong "
                         "scaling); kv | range | kv+range | KxR: that split explicitly; replica: every rank runs its "
                         "own sequence (weak scaling)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "torch"],
                    help="exchange steps over liboomb_comm.so (NCCL, default) or torch.distributed (gloo, CUDA "
                         "tensors staged through the host: lets several ranks share one GPU in tests)")
    ap.add_argument("--same-device", action="store_true", help="every rank on cuda:0 (tests; with --comm torch)")
    ap.add_argument("--offload-cap", type=float, default=0.75,
                    help="device capacity (fraction of the layer's pages) of the offload measurement; 0 = skip")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.tokens:
        cfg["T"] = args.tokens
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    chunks = workload(cfg)
    # one sequence split across the ranks (the north-star partition) unless replicas are asked for;
    # at N = 1 "auto" is the unsplit layer
    sharded = args.shard != "replica" and (world > 1 or args.shard != "auto")
    plan = None
    if sharded:
        from paper_2602_02108_b200.sharding import ShardPlan
        plan = ShardPlan(rank, world, cfg["Hkv"], cfg["Hq"], args.shard)
    base_config = {"workload": f"{args.config}: {cfg['desc']}", "context_tokens": cfg["T"],
                   "chunk": cfg["C"], "page": cfg["P"], "q_heads": cfg["Hq"], "kv_heads": cfg["Hkv"],
                   "head_dim": cfg["hd"], "selection": cfg["mode"],
                   "pages_per_query_page": cfg["budget"] // cfg["P"] if cfg["mode"] == "topk" else "all",
                   "layers_per_step": 1,
                   "parallelism": (plan.describe() if sharded
                                   else f"{world} independent replica(s), one sequence each")}

    if args.impl == "reference":
        if rank != 0:
            return
        vals = []
        for s in range(args.warmup + args.steps):
            cb = cpu_baseline(cfg, args.cpu_workers)
            if s >= args.warmup:
                vals.append(cb["value"])
        v = statistics.mean(vals)
        line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": cfg["T"] / v * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic N(0,1)",
                "impl": "reference", "config": base_config,
                "cpu_baseline": {**cb, "value": v},
                "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    if world > 1:
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(0 if args.same_device else local)
        dist.init_process_group("nccl" if args.comm == "nccl" else "gloo")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    from paper_2602_02108_b200 import _lib

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    run_cfg = cfg
    layer = None
    if sharded:
        from paper_2602_02108_b200 import ModelConfig
        from paper_2602_02108_b200.sharding import OombComm, ShardedLayer, TorchComm
        kv_g, rg = plan.new_groups() if world > 1 else (None, None)

        def make_comm(group, size):
            if size <= 1:
                return None
            return OombComm.from_process_group(group) if args.comm == "nccl" else TorchComm(group)

        gcfg = ModelConfig(n_layers=1, n_q_heads=cfg["Hq"], n_kv_heads=cfg["Hkv"], head_dim=cfg["hd"],
                           chunk_size=cfg["C"], page_size=cfg["P"], retrieval_budget=cfg["budget"],
                           attention_mode=[cfg["mode"]])
        layer = ShardedLayer(plan, gcfg, None, make_comm(kv_g, plan.kv_world), make_comm(rg, plan.range_world))
        run_cfg = dict(cfg, Hq=cfg["Hq"] // plan.kv_world, Hkv=cfg["Hkv"] // plan.kv_world)
        args.offload_cap = 0.0  # the offload regime is a one-GPU, unsplit measurement
    # the ranks of one page-range group hold the same heads: they must see the same q / k / v / dO
    run = Run(run_cfg, seed=1234 + (plan.kv_idx if sharded else rank), device=dev, layer=layer)
    for _ in range(args.warmup):
        run.step()
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs
    clocks = Clocks(dev.index)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = _lib.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run.fwd_phase.clear()
    run.bwd_phase.clear()
    e0.record()
    for _ in range(args.steps):
        run.step()
    e1.record()
    torch.cuda.synchronize()
    bwd_phase_ms = sum(a.elapsed_time(b) for a, b in run.bwd_phase) / args.steps
    fwd_phase_ms = sum(a.elapsed_time(b) for a, b in run.fwd_phase) / args.steps
    launches = _lib.kernel_launches() - launches0
    barrier()
    clk = clocks.stop()
    # per-kernel breakdown: as many steps again with the library's event profiler on (two timing
    # events per launch add host work that a 2 ms c1 step notices), so the timed steps above run
    # without it
    run.cache.profile_enable(True)
    run.cache.profile_collect()
    for _ in range(args.steps):
        run.step()
    torch.cuda.synchronize()
    prof = run.cache.profile_collect()
    run.cache.profile_enable(False)
    run.fwd_phase.clear()
    run.bwd_phase.clear()
    barrier()
    ms_step = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    seqs = 1 if sharded else world  # sequences processed by the whole job per step
    value = seqs * cfg["T"] / (ms_step / 1e3)

    # ---- e2e: same API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        ee = E2E(run)
        ee.step()
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            ee.step()
        f1.record()
        torch.cuda.synchronize()
        ms_e2e = max_over_ranks(f0.elapsed_time(f1) / args.steps)
        e2e = {"value": seqs * cfg["T"] / (ms_e2e / 1e3), "unit": "tokens/s", "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": ee.h2d_bytes, "d2h_bytes_per_step": ee.d2h_bytes,
               "path": ("native layer loop (chunk_loop.layer_step), whole-step copies" if ee.native else
                        "public per-chunk API, copies one chunk ahead on side streams")}

    offload = None
    # the offload regime is a one-GPU measurement (wall clock, pinned host tier per process)
    if args.offload_cap and 0 < args.offload_cap < 1 and cfg["mode"] == "topk" and world == 1:
        try:
            offload = offload_measure(run, args.offload_cap)
        except Exception as ex:  # the offload measurement never blocks the line
            offload = {"error": repr(ex)}

    if rank != 0:
        return
    peak, peak_sus, hbm, peak_src = peaks()
    fwd_fl = sum(c["fwd"] for c in chunks)
    bwd_fl = sum(c["bwd"] for c in chunks)
    # per-GPU algorithmic TFLOP/s: a shard of a split sequence does 1/world of its work
    tflops = (fwd_fl + bwd_fl) / (ms_step / 1e3) / 1e12 / (world if sharded else 1)
    if sharded:
        fwd_fl, bwd_fl = fwd_fl / world, bwd_fl / world
    kernels = {}
    for k, (n, ms) in prof.items():
        kernels[k] = {"launches_per_step": n / args.steps, "ms_per_step": ms / args.steps}
    for k in ("bwd_dq", "bwd_dkdv"):
        if k in kernels and "bwd_pair" in kernels:
            kernels[k]["note"] = "overlaps the other backward kernel; see bwd_pair for their joint span"
    for k in ("bwd_dq", "bwd_dkdv", "bwd_prep", "gather_scatter", "grad_init"):
        if k in kernels and BWD_DEFER:
            kernels[k]["note"] = ("chunk i's dQ runs on the library's side stream under chunk i-1's prep, dK/dV and "
                                  "dM read-back: these spans overlap each other; see bwd_phase")
    for k in ("score", "topk", "other", "append", "attn_fwd"):
        if k in kernels:
            kernels[k]["note"] = ("chunk i+1's selection (score, topk; the dense CSR fill is 'other') runs on "
                                  "a second stream while chunk i appends and attends: these spans overlap "
                                  "each other, so they are not additive")

    # dominant kernel pair: the tcgen05 backward (dq + dkdv launches per chunk)
    # the dq and dkdv kernels run concurrently (dq on a side stream): their pair is timed as one span
    if BWD_DEFER:  # chunks chain through the dQ side stream: the backward pass is the span
        t_bwd = bwd_phase_ms
        kernels["bwd_phase"] = {"ms_per_step": bwd_phase_ms,
                                "note": "CUDA events around the whole backward pass (dq + dkdv of every chunk, "
                                        "chained; also bwd_prep, grad_init, the dM read-back)"}
    elif "bwd_pair" in prof:
        t_bwd = prof["bwd_pair"][1] / args.steps
    else:
        t_bwd = (prof.get("bwd_dq", (0, 0.0))[1] + prof.get("bwd_dkdv", (0, 0.0))[1]) / args.steps
    kernels["fwd_phase"] = {"ms_per_step": fwd_phase_ms,
                            "note": "CUDA events around the whole forward pass (selection, append and attention of "
                                    "every chunk)"}
    # with two attention streams the per-launch spans overlap: the forward pass span is the honest time
    t_fwd = fwd_phase_ms if FWD_STREAMS > 1 else prof.get("attn_fwd", (0, 0.0))[1] / args.steps
    for name, fl, t in (("attn_fwd", fwd_fl, t_fwd), ("attn_bwd(dq+dkdv)", bwd_fl, t_bwd)):
        if t > 0:
            kernels.setdefault(name, {})
            kernels[name]["achieved_tflops"] = fl / (t / 1e3) / 1e12
            kernels[name]["frac_of_peak"] = fl / (t / 1e3) / 1e12 / peak
    achieved = bwd_fl / (t_bwd / 1e3) / 1e12 if t_bwd > 0 else None
    traffic = None
    try:  # DRAM bytes of the dominant kernel pair from the committed ncu --set full capture
        tf = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
        if not os.path.exists(tf):
            tf = os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")
        with open(tf) as f:
            tr = json.load(f)
        traffic = {"bytes_per_launch": sum(tr[k]["dram_read_bytes"] + tr[k]["dram_write_bytes"]
                                           for k in ("attn_bwd_dq", "attn_bwd_dkdv")),
                   "source": tr["source"]}
    except Exception:
        pass
    roofline = {"bound": "tensor",
                "kernel": ("attn_bwd_dq + attn_bwd_dkdv (tcgen05), every chunk's pair chained through the dQ side "
                           "stream: achieved = backward FLOPs / backward-pass span (CUDA events on the launching "
                           "stream)") if BWD_DEFER else
                          "attn_bwd_dq + attn_bwd_dkdv (tcgen05, run concurrently), per chunk",
                # the pair is timed inside a long step (hundreds of ms at the power cap), so its roofline
                # denominator is the sustained cuBLAS figure; the burst one is kept beside it
                "achieved": achieved, "peak": peak_sus, "unit": "TFLOP/s",
                "frac": achieved / peak_sus if achieved else None,
                "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside a long step)",
                "peak_burst": peak, "frac_of_burst": achieved / peak if achieved else None,
                "algorithmic": "10*hd*Hq*pairs per chunk, pairs = P*P*sum|sel| + C(C+1)/2 (SURVEY 8d)",
                "traffic": traffic["bytes_per_launch"] if traffic else None,
                "traffic_source": traffic["source"] if traffic else None}
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0,1) bf16 q/k/v/dO generated on device (1M-token K/V distinct per chunk; "
                    "16 distinct q/dO chunks cycled); random-init, no checkpoint",
            "config": {**base_config, "l2": "inputs > L2 (KV pool 2 GiB + grad pool 4 GiB + 17 GB of inputs)",
                       "offload": "value / e2e: all pages resident (declared); the `offload` key measures the "
                                  "capped-capacity regime separately; e2e moves chunk inputs/outputs over the host link"},
            "pct_bf16_peak": tflops / peak, "pct_bf16_peak_sustained": tflops / peak_sus,
            "algorithmic_tflops": tflops,
            "model_equiv_tokens_per_s": value / (32 if cfg["Hq"] == 32 else 28),
            "roofline": roofline, "kernels": kernels, "gpu_launches": launches,
            "gpu_launches_per_step": launches // args.steps, "clocks": clk, "e2e": e2e, "offload": offload,
            "train_step_variant": {
                "what": "full train step of SURVEY 3.2: 2 forwards (phase A + recompute) + 1 backward per chunk; "
                        "the recompute forward is charged as a whole forward pass (fwd_phase, selection and append "
                        "included: an upper bound)" if FWD_STREAMS > 1 else
                        "full train step of SURVEY 3.2: 2 forwards (phase A + recompute) + 1 backward per chunk; "
                        "the recompute forward is the same forward kernel, timed above",
                "tokens_per_s": seqs * cfg["T"] / ((ms_step + t_fwd) / 1e3),
                "ms_per_step": ms_step + t_fwd}}
    if sharded:
        from paper_2602_02108_b200.sharding import comm_bytes
        g_loc, m_q = run_cfg["Hkv"], cfg["C"] // cfg["P"]
        n_last = chunks[-1]["n_cand"]
        line["sharding"] = {
            "kv_world": plan.kv_world, "range_world": plan.range_world, "comm": args.comm,
            "pool_pages_per_rank": (cfg["T"] // cfg["P"] + plan.range_world - 1) // plan.range_world,
            "layer_pages": cfg["T"] // cfg["P"],
            "bytes_sent_per_rank_per_chunk": {
                **layer.comm_bytes_per_chunk(),
                "vote_allgather_bytes_last_chunk": (comm_bytes(0, plan.kv_world, g_loc * m_q * n_last, 4)[0]
                                                    if cfg["mode"] == "topk" else 0)},
            "note": "vote exchanged over the ranks of one page range (all-gather, then a fixed-order sum); "
                    "(O, LSE) merge and the [dq | dk_cur | dv_cur] reduction over the ranks of one KV group "
                    "(ordered reduce-scatter by row slices + all-gather of the slices; *_allgather = the "
                    "all-gather-then-combine bytes they replace)"}
    if not args.no_cpu and world == 1:  # rank 0 at N = 1 only (the reference arm covers every N)
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_workers)
        except Exception as ex:  # the baseline never blocks the measurement line
            line["cpu_baseline"] = {"value": None, "error": repr(ex)}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
