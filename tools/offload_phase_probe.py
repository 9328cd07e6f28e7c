"""Where the low-locality offload regime's exposed time goes: forward vs backward phase of the
native loop (engine attached), capped tier vs unlimited tier, CUDA events per phase."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2602_02108_b200 import PagedCache  # noqa: E402
from paper_2602_02108_b200.chunk_loop import layer_stats, layer_step  # noqa: E402
from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine  # noqa: E402

cfg = dict(bench.CONFIGS["c3"])
run = bench.Run(cfg, seed=1234, device=torch.device("cuda", 0))
C, P = cfg["C"], cfg["P"]
n_pages = cfg["T"] // P
cap = int(0.75 * n_pages)
slots = cap + 16 * (C // P)
K = bench.low_locality_keys(run) if "--bench-data" not in sys.argv else run.k_all
kv = (run.S, C, cfg["Hkv"], cfg["hd"])


SLOTS = int(sys.argv[sys.argv.index("--slots") + 1]) if "--slots" in sys.argv else slots


def one(capped):
    cache = PagedCache(run.mc, dtype="bf16", max_tokens=cfg["T"], device_capacity_pages=SLOTS if capped else -1)
    eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap if capped else -1, bandwidth_bytes_per_s=55e9))
    eng.set_prefetch_headroom_pages(C // P)
    comp = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    ev[0].record(comp)
    args = (cache, 0, run.q_all, K.view(kv), run.v_all.view(kv), run.do_all, run.o_all, run.lse_all, run.grads)
    import time
    t0 = time.perf_counter()
    layer_step(*args, mode="topk", phase="forward")
    t1 = time.perf_counter()
    ev[1].record(comp)
    layer_step(*args, mode="topk", phase="backward")
    t2 = time.perf_counter()
    ev[2].record(comp)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    st = layer_stats(cache)
    r = {"fwd_s": ev[0].elapsed_time(ev[1]) / 1e3, "bwd_s": ev[1].elapsed_time(ev[2]) / 1e3,
         "host_fwd_s": t1 - t0, "host_bwd_s": t2 - t1, "host_drain_s": t3 - t2,
         "h2d_fwd": eng.h2d_bytes(0), "h2d_bwd": eng.h2d_bytes(1), "d2h": eng.d2h_bytes(),
         "fwd_fetch_chunks": sum(1 for x in st if x[0] == "fwd" and x[3] > 0),
         "bwd_d2h_in_fwd": sum(x[4] for x in st if x[0] == "fwd")}
    if capped:
        ev_log = eng.raw_log()
        per = {}
        for e in ev_log:
            if e.phase != 1 or e.kind not in (0, 1):
                continue
            d = per.setdefault(e.chunk, [1e30, 0.0, 0])
            if e.kind == 0:
                d[0] = min(d[0], e.t)
            else:
                d[1] = max(d[1], e.t)
                d[2] += e.bytes
        bw = [(c, (v[1] - v[0]) * 1e3, v[2] / max(v[1] - v[0], 1e-9) / 1e9) for c, v in sorted(per.items()) if v[2]]
        r["bwd_fetch_ms_median"] = sorted(x[1] for x in bw)[len(bw) // 2]
        r["bwd_fetch_GBps_median"] = sorted(x[2] for x in bw)[len(bw) // 2]
        r["bwd_fetch_sample"] = [(c, round(ms, 3), round(g, 1)) for c, ms, g in bw[100:106]]
    eng.release_all_reservations()
    eng.close(discard=True)
    del cache
    torch.cuda.empty_cache()
    return r


h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for what, dst, src in (("h2d", d, h), ("d2h", h, d)):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dst.copy_(src, non_blocking=True)
    a.record()
    dst.copy_(src, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    print(what, "1 GiB copy GB/s", round((1 << 30) / (a.elapsed_time(b) / 1e3) / 1e9, 1), flush=True)
del h, d
one(False)
one(True)
for rep in range(2):
    print(json.dumps({"rep": rep, "resident": one(False), "capped": one(True)}), flush=True)
