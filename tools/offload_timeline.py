"""Per-chunk timeline of the capped low-locality backward (diagnostics): compute start / end of every
chunk's attn_backward (OOMB_LAYER_TIMELINE events on the compute stream) against the engine log's
CUDA-event stamps (prefetch H2D issue / done per chunk, write-back batch done), all in ms from the
engine's origin. Prints where the compute stream idles and which copy it was waiting for."""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2602_02108_b200 import PagedCache  # noqa: E402
from paper_2602_02108_b200.chunk_loop import layer_step  # noqa: E402
from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine  # noqa: E402

cfg = dict(bench.CONFIGS["c3"])
run = bench.Run(cfg, seed=1234, device=torch.device("cuda", 0))
C, P = cfg["C"], cfg["P"]
n_pages = cfg["T"] // P
cap = int(0.75 * n_pages)
slots = int(sys.argv[sys.argv.index("--slots") + 1]) if "--slots" in sys.argv else cap + 16 * (C // P)
K = bench.low_locality_keys(run) if "--bench-data" not in sys.argv else run.k_all
kv = (run.S, C, cfg["Hkv"], cfg["hd"])
path = os.path.abspath("gpurun_out/timeline.txt")


def one(capped, timeline):
    cache = PagedCache(run.mc, dtype="bf16", max_tokens=cfg["T"], device_capacity_pages=slots if capped else -1)
    eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap if capped else -1, bandwidth_bytes_per_s=55e9))
    eng.set_prefetch_headroom_pages(C // P)
    if timeline:
        os.environ["OOMB_LOOP_TIMELINE"] = path
    args = (cache, 0, run.q_all, K.view(kv), run.v_all.view(kv), run.do_all, run.o_all, run.lse_all, run.grads)
    layer_step(*args, mode="topk")
    torch.cuda.synchronize()
    os.environ.pop("OOMB_LOOP_TIMELINE", None)
    log = eng.raw_log() if timeline else None
    if capped:
        print(f"h2d reference bytes {eng.h2d_bytes(0) + eng.h2d_bytes(1)}, moved {eng.h2d_bytes_moved()}, "
              f"d2h {eng.d2h_bytes()}, moved {eng.d2h_bytes_moved()}")
    eng.release_all_reservations()
    eng.close(discard=True)
    del cache
    torch.cuda.empty_cache()
    return log


one(True, False)
for capped in (False, True):
    log = one(capped, True)
    tl, host = {}, {}
    for line in open(path):
        c, a, b, *h = line.split()
        tl[int(c)] = (float(a), float(b))
        host[int(c)] = [float(x) for x in h]
    comp = [tl[c][1] - tl[c][0] for c in sorted(tl)]
    order = sorted(tl, reverse=True)
    gaps = [tl[order[j + 1]][0] - tl[order[j]][1] for j in range(len(order) - 1)]
    print(f"== {'capped' if capped else 'resident'}: backward {tl[0][1] - tl[order[0]][0]:.1f} ms, "
          f"compute per chunk median {statistics.median(comp):.3f} ms (sum {sum(comp):.1f}), "
          f"gaps between chunks sum {sum(gaps):.1f} ms, median {statistics.median(gaps):.3f}")
    if not capped:
        continue
    from collections import Counter
    print("log events (kind, phase):", sorted(Counter((e.kind, e.phase) for e in log).items()))
    longest = sorted(((tl[c][1] - tl[c][0], c) for c in tl), reverse=True)[:12]
    print("longest chunk computes (ms, chunk):", [(round(a, 2), c) for a, c in longest])
    print("host ms of those chunks (fetch+wait, prefetch, attn_backward call, rest):",
          [(c, [round(x, 2) for x in host[c]]) for _, c in longest[:6]])
    print("host ms totals (fetch+wait, prefetch, attn_backward call, rest):",
          [round(sum(host[c][k] for c in host), 1) for k in range(4)])
    # engine log, backward phase, in issue order: attribute evictions to the chunk being waited
    pre = {}   # chunk -> [issued min, done max, bytes]
    wb = {}    # chunk context -> write-back batch done (max)
    cur = None
    for e in log:
        if e.phase != 1:
            continue
        if e.kind in (0, 1):
            d = pre.setdefault(e.chunk, [1e30, 0.0, 0])
            if e.kind == 0:
                d[0] = min(d[0], e.t * 1e3)
            else:
                d[1] = max(d[1], e.t * 1e3)
                d[2] += e.bytes
        if e.kind == 5:  # access: the chunk being computed
            cur = e.chunk
        if e.kind == 2 and cur is not None:
            wb[cur] = max(wb.get(cur, 0.0), e.t * 1e3)
    # write-backs of pages already dead for this step (owned by a chunk whose backward, and so its
    # read-back, is done): nothing reads them again before the step ends
    cur, dead_b, all_b, dead_n, all_n = None, 0, 0, 0, 0
    m_ = C // P
    for e in log:
        if e.kind == 5 and e.phase == 1:
            cur = e.chunk
        if e.kind == 2 and e.phase == 1 and e.bytes > 0 and cur is not None:
            all_b += e.bytes
            all_n += 1
            if e.page // m_ > cur:
                dead_b += e.bytes
                dead_n += 1
    print(f"backward write-backs: {all_n} pages {all_b / 1e9:.2f} GB, of dead pages {dead_n} ({dead_b / 1e9:.2f} GB)")
    # victim reuse estimate: fetches (backward) of a page evicted at most D evictions earlier (its old
    # slots would still be unused in a FIFO free list holding ~D slots)
    for D in (128, 256, 400):
        seq, last_ev, hit, tot, hit_b, tot_b = 0, {}, 0, 0, 0, 0
        for e in log:
            if e.kind == 2:
                seq += 1
                last_ev[(e.layer, e.page)] = seq
            elif e.kind == 0:
                k = (e.layer, e.page)
                ok_ = k in last_ev and seq - last_ev[k] < D
                if e.phase == 1:
                    tot_b += 1
                    hit_b += ok_
                tot += 1
                hit += ok_
        print(f"victim reuse within {D} evictions: {hit}/{tot} fetches ({hit_b}/{tot_b} in backward)")
    rows = []
    for j in range(1, len(order)):
        c, prev = order[j], order[j - 1]
        start, end_prev = tl[c][0], tl[prev][1]
        pi = pre.get(c)
        rows.append((c, start - end_prev, (pi[1] - end_prev) if pi else None, (pi[1] - pi[0]) if pi else None,
                     pi[2] / 1e6 if pi else 0, (wb.get(prev, 0) - tl[prev][0]) if prev in wb else None))
    waiting = [r for r in rows if r[1] > 0.05]
    print(f"chunks with a compute gap > 0.05 ms: {len(waiting)} of {len(rows)}; gap sum {sum(r[1] for r in waiting):.1f} ms")
    print("chunk gap_ms  prefetch_done-prev_end  prefetch_dur  prefetch_MB  prev_wb_done-prev_start")
    for r in rows[100:125]:
        print(r[0], *(f"{x:.3f}" if isinstance(x, float) else str(x) for x in r[1:]))
