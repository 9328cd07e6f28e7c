"""oomb_layer_step (the native layer loop) is the Python chunk loop, bitwise.

bench.Run.step runs the unsplit layer through chunk_loop.layer_step (one C call per phase); the
host loop (forward_pass + bwd_chunk, the call sequence AttentionChunkLoop follows) is the
reference for it here. Both run on the same bench inputs: every chunk's out / lse, the last
chunk's dq / dk_cur / dv_cur and the whole gradient pool must match bit for bit, for top-k (c3
shape, 16 chunks), dense (c2 shape, 8 chunks) and the c1 geometry (tcgen05 head dim 64 / page 64,
split-K).
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = {"c3_16chunks": ("c3", 16 * 4096), "c2_8chunks": ("c2", 8 * 4096), "c1": ("c1", None)}


@pytest.mark.parametrize("name", sorted(CASES))
def test_native_loop_bitwise(name):
    import bench
    cfg_name, tokens = CASES[name]
    cfg = dict(bench.CONFIGS[cfg_name])
    if tokens:
        cfg["T"] = tokens
    run = bench.Run(cfg, seed=1234, device=torch.device("cuda", 0))
    res = {}
    for native in (False, True):
        bench.NATIVE_LOOP = native
        run.step()
        torch.cuda.synchronize()
        run.cache.check_device_errors()
        n = run.cache.n_pages(0)
        gp = run.cache.gather_grad_pages(0, list(range(n)))
        res[native] = [run.o_all.clone(), run.lse_all.clone(), run.grads.dq.clone(), run.grads.dk_cur.clone(),
                       run.grads.dv_cur.clone(), gp.k.clone(), gp.v.clone()]
    bench.NATIVE_LOOP = True
    for a, b, what in zip(res[False], res[True], ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v")):
        assert torch.equal(a, b), (name, what)


def _engine_run(run, K, native, cap, slots):
    """One layer step under the residency protocol: the Python AttentionChunkLoop + TieredEngine
    (bench.offload_measure's loop) or the native loop with the same engine attached."""
    import bench
    from paper_2602_02108_b200 import PagedCache
    from paper_2602_02108_b200.chunk_loop import AttentionChunkLoop, layer_stats, layer_step
    from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine
    cfg, C = run.cfg, run.cfg["C"]
    cache = PagedCache(run.mc, dtype="bf16", max_tokens=cfg["T"], device_capacity_pages=slots)
    eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap, bandwidth_bytes_per_s=55e9))
    eng.set_prefetch_headroom_pages(C // cfg["P"])
    run.o_all.zero_()
    run.lse_all.zero_()
    if native:
        kv = (run.S, C, cfg["Hkv"], cfg["hd"])
        layer_step(cache, 0, run.q_all, K.view(kv), run.v_all.view(kv), run.do_all, run.o_all, run.lse_all,
                   run.grads, mode=cfg["mode"])
        stats = layer_stats(cache)
    else:
        loop = AttentionChunkLoop(cache, engine=eng)
        for i in range(run.S):
            nq = run.q[(i + 1) % run.RQ] if i + 1 < run.S else None
            loop.forward_chunk(i, run.q[i % run.RQ], K[i * C:(i + 1) * C], run.v_all[i * C:(i + 1) * C],
                               next_q=nq, out=run.o_all[i], lse=run.lse_all[i])
        loop.begin_backward()
        for i in reversed(range(run.S)):
            loop.backward_chunk(i, run.do[i % run.RQ], run.q[i % run.RQ], K[i * C:(i + 1) * C],
                                run.v_all[i * C:(i + 1) * C], grads=run.grads)
        stats = loop.chunk_stats
    torch.cuda.synchronize()
    cache.check_device_errors()
    io = (eng.h2d_bytes(0), eng.h2d_bytes(1), eng.d2h_bytes())
    eng.release_all_reservations()
    eng.restore_all()  # every page back on the device (the pool has a slot for each) to compare grads
    n = cache.n_pages(0)
    gp = cache.gather_grad_pages(0, list(range(n)))
    res = [run.o_all.clone(), run.lse_all.clone(), run.grads.dq.clone(), run.grads.dk_cur.clone(),
           run.grads.dv_cur.clone(), gp.k.clone(), gp.v.clone()]
    eng.close(discard=True)
    del cache
    assert bench is not None
    return res, stats, io


@pytest.mark.parametrize("regime", ["bench_data", "low_locality"])
def test_native_loop_with_engine_matches_host_loop(regime):
    """The native loop with a TieredEngine attached makes the host loop's engine calls: the same
    outputs and gradients bit for bit, the same per-chunk resident-page counts and the same bytes
    moved, with the tier capped at 75 % of the layer's pages (pages really leave the device)."""
    import bench
    cfg = dict(bench.CONFIGS["c3"])
    # low locality: 64 chunks, so a chunk's working set (the union of 32 near-random top-64 lists
    # plus its own pages) stays under the 75 % tier (at 16 chunks it approaches every page)
    cfg["T"] = (16 if regime == "bench_data" else 64) * 4096
    run = bench.Run(cfg, seed=4321, device=torch.device("cuda", 0))
    K = run.k_all if regime == "bench_data" else bench.low_locality_keys(run)
    n_pages = cfg["T"] // cfg["P"]
    cap = int(0.75 * n_pages)
    host = _engine_run(run, K, False, cap, n_pages)
    nat = _engine_run(run, K, True, cap, n_pages)
    for a, b, what in zip(host[0], nat[0], ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v")):
        assert torch.equal(a, b), (regime, what)
    assert host[1] == nat[1]
    assert host[2] == nat[2]
    assert host[2][0] > 0 and host[2][2] > 0, "the capped tier must move pages both ways"


@pytest.mark.parametrize("lazy", [False, True])
@pytest.mark.parametrize("slack", [512, 768])
def test_victim_slot_reclaim_bitwise(slack, lazy, monkeypatch):
    """Pages fetched back into their victim slots (the slots their eviction freed, not yet handed out
    again) and pages copied in from the host tier mix within one step: every chunk's output, LSE,
    dq and dk_cur / dv_cur (the dM_i read-back of the chunk's own pages: together the whole
    gradient pool) equal the all-resident run bit for bit, and the engine really did both (moved
    fewer bytes than the reference's accounting, but some). lazy: write-backs deferred until a
    freed slot nears reuse and dropped for pages fetched back first (OOMB_TIER_LAZY_WB=1, read at
    engine creation)."""
    import bench
    from paper_2602_02108_b200 import PagedCache
    from paper_2602_02108_b200 import attention as A
    from paper_2602_02108_b200.chunk_loop import layer_step
    monkeypatch.setenv("OOMB_TIER_LAZY_WB", "1" if lazy else "0")
    from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine
    cfg = dict(bench.CONFIGS["c3"])
    cfg["T"] = 128 * 4096  # 4,096 pages: the tier holds 3,072, the pool 3,072 + slack
    dev = torch.device("cuda", 0)
    run = bench.Run(cfg, seed=99, device=dev)
    K = bench.low_locality_keys(run)
    C, P, S = cfg["C"], cfg["P"], run.S
    n_pages = cfg["T"] // P
    cap = int(0.75 * n_pages)
    kv = (S, C, cfg["Hkv"], cfg["hd"])
    grads = A.AttnGrads(torch.empty(S, C, cfg["Hq"], cfg["hd"], device=dev),
                        torch.empty(S, C, cfg["Hkv"], cfg["hd"], device=dev),
                        torch.empty(S, C, cfg["Hkv"], cfg["hd"], device=dev))
    res, moved = {}, None
    for capped in (False, True):
        cache = PagedCache(run.mc, dtype="bf16", max_tokens=cfg["T"],
                           device_capacity_pages=cap + slack if capped else -1)
        eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap if capped else -1, bandwidth_bytes_per_s=55e9))
        eng.set_prefetch_headroom_pages(C // P)
        for t in (run.o_all, run.lse_all, grads.dq, grads.dk_cur, grads.dv_cur):
            t.zero_()
        layer_step(cache, 0, run.q_all, K.view(kv), run.v_all.view(kv), run.do_all, run.o_all, run.lse_all,
                   grads, mode="topk", grad_stride_chunks=1)
        torch.cuda.synchronize()
        cache.check_device_errors()
        if capped:
            moved = (eng.h2d_bytes(0) + eng.h2d_bytes(1), eng.h2d_bytes_moved(), eng.d2h_bytes(),
                     eng.d2h_bytes_moved())
        res[capped] = [x.clone() for x in (run.o_all, run.lse_all, grads.dq, grads.dk_cur, grads.dv_cur)]
        eng.release_all_reservations()
        eng.close(discard=True)
        del cache, eng
        torch.cuda.empty_cache()
    for a, b, what in zip(res[False], res[True], ("out", "lse", "dq", "dk_cur", "dv_cur")):
        assert torch.equal(a, b), (slack, what)
    assert 0 < moved[1] < moved[0], moved
    assert 0 < moved[3] <= moved[2], moved  # deferred write-backs of pages fetched back are dropped
    if lazy:
        assert moved[3] < moved[2], moved


def test_engine_loop_phase_split_equals_whole_step():
    """With an engine attached, the forward-only call followed by the backward-only call is the same
    step as one call: the same outputs, gradients, bytes moved and per-chunk records."""
    import bench
    from paper_2602_02108_b200 import PagedCache
    from paper_2602_02108_b200.chunk_loop import layer_stats, layer_step
    from paper_2602_02108_b200.tiered_memory import TierConfig, TieredEngine
    cfg = dict(bench.CONFIGS["c3"])
    cfg["T"] = 16 * 4096
    run = bench.Run(cfg, seed=2024, device=torch.device("cuda", 0))
    K = run.k_all
    C, P = cfg["C"], cfg["P"]
    n_pages = cfg["T"] // P
    cap = int(0.75 * n_pages)
    kv = (run.S, C, cfg["Hkv"], cfg["hd"])
    res = []
    for split in (False, True):
        cache = PagedCache(run.mc, dtype="bf16", max_tokens=cfg["T"], device_capacity_pages=n_pages)
        eng = TieredEngine(cache, TierConfig(device_capacity_pages=cap, bandwidth_bytes_per_s=55e9))
        eng.set_prefetch_headroom_pages(C // P)
        args = (cache, 0, run.q_all, K.view(kv), run.v_all.view(kv), run.do_all, run.o_all, run.lse_all, run.grads)
        if split:
            layer_step(*args, mode="topk", phase="forward")
            layer_step(*args, mode="topk", phase="backward")
        else:
            layer_step(*args, mode="topk")
        torch.cuda.synchronize()
        cache.check_device_errors()
        res.append(([x.clone() for x in (run.o_all, run.lse_all, run.grads.dq, run.grads.dk_cur, run.grads.dv_cur)],
                    layer_stats(cache), (eng.h2d_bytes(0), eng.h2d_bytes(1), eng.d2h_bytes())))
        eng.release_all_reservations()
        eng.close(discard=True)
        del cache, eng
        torch.cuda.empty_cache()
    for a, b in zip(res[0][0], res[1][0]):
        assert torch.equal(a, b)
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]
    assert res[0][2][0] > 0
