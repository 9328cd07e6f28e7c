"""Generate the golden fixtures for the OOMB hot path FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    make -f oracle/Makefile.ref && python tests/golden/make_golden.py

Every number written here comes out of oracle/_ref/libchunktrain_ref.so, i.e.
the unmodified reference headers (paged_kv.hpp, attention.hpp,
tiered_memory.hpp, oracle.hpp) compiled in place. The fixtures pin:

* known_answers.json — the reference's own known-answer tests
  (test_attention.cpp:54-118), re-derived by calling the reference;
* attn_small_{f32,f64}.npz — full fwd/bwd arrays at the reference test geometry
  (test_attention.cpp:19-31: P=8, C=16, 4Q/2KV, hd=8) incl. scattered grad pages;
* pagetable.npz — a random append / scatter / reset script (page tables,
  K_avg sums, memory reports), test_paged_kv.cpp style;
* select.npz — top-k rows with heavy ties;
* hashes.json — SHA-256 of reference outputs at larger geometries (c1 tiny
  geometry, a Qwen2.5-7B-shaped slice, top-k scoring) whose inputs are re-made
  from det_normal(seed) at test time, so the arrays themselves are not stored.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Cfg, Ref, det_normal  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# ---------------------------------------------------------------------------
# Shared case builders (also imported by the tests to rebuild inputs)
# ---------------------------------------------------------------------------

def attn_case(cfg: Cfg, past_tokens: int, seed: int, dtype, selected=None, layer: int = 0):
    """Deterministic inputs for one chunk over `past_tokens` of cache."""
    P, C = cfg.page_size, cfg.chunk_size
    kvh, hd, qh = cfg.n_kv_heads, cfg.head_dim, cfg.n_q_heads
    pk = det_normal(seed * 16 + 1, (past_tokens, kvh, hd), dtype)
    pv = det_normal(seed * 16 + 2, (past_tokens, kvh, hd), dtype)
    q = det_normal(seed * 16 + 3, (C, qh, hd), dtype)
    kc = det_normal(seed * 16 + 4, (C, kvh, hd), dtype)
    vc = det_normal(seed * 16 + 5, (C, kvh, hd), dtype)
    do = det_normal(seed * 16 + 6, (C, qh, hd), dtype)
    n_past_pages = (past_tokens + P - 1) // P
    if selected is None:
        selected = [list(range(n_past_pages)) for _ in range(C // P)]
    return dict(pk=pk, pv=pv, q=q, kc=kc, vc=vc, do=do, selected=selected)


def run_attn(backend, cfg: Cfg, case, layer: int = 0):
    """append(past) -> append(current chunk) -> forward -> backward, reference order."""
    if len(case["pk"]):
        backend.append(layer, case["pk"], case["pv"])
    n_past = backend.n_pages(layer)
    backend.append(layer, case["kc"], case["vc"])
    out, lse = backend.attn_forward(layer, case["q"], case["selected"], case["kc"], case["vc"])
    dq, dk, dv = backend.attn_backward(layer, case["do"], case["q"], case["selected"], case["kc"], case["vc"],
                                       out, lse)
    gk, gv, _ = backend.gather(layer, list(range(n_past)), grads=True)
    return dict(out=out, lse=lse, dq=dq, dk_cur=dk, dv_cur=dv, grad_k=gk, grad_v=gv,
                page_table=backend.page_table(layer))


def pagetable_script(backend, seed: int):
    """Random append / scatter / reset sequence on a 2-layer cache
    (test_paged_kv.cpp:99-137, 168-219, 251-269 style). Returns snapshots."""
    rng = np.random.default_rng(seed)
    cfg = backend.cfg
    snaps = []
    for step in range(3):
        for layer in range(cfg.n_layers):
            for _ in range(int(rng.integers(1, 5))):
                rows = int(rng.integers(1, 40))
                k = det_normal(seed * 1000 + step * 100 + layer * 10 + rows, (rows, cfg.n_kv_heads, cfg.head_dim),
                               backend.dtype)
                v = det_normal(seed * 1000 + step * 100 + layer * 10 + rows + 5, (rows, cfg.n_kv_heads,
                                                                                   cfg.head_dim), backend.dtype)
                backend.append(layer, k, v)
            n = backend.n_pages(layer)
            ids = sorted(set(int(x) for x in rng.integers(0, n, size=max(1, n // 2))))
            rng.shuffle(ids)
            g = det_normal(seed * 7 + step + layer, (len(ids) * cfg.page_size, cfg.n_kv_heads, cfg.head_dim),
                           backend.dtype)
            backend.scatter(layer, ids, g, -0.5 * g)
        snap = {}
        for layer in range(cfg.n_layers):
            snap[f"pt{layer}"] = backend.page_table(layer)
            s, c = backend.kavg_raw(layer)
            snap[f"kavg_sum{layer}"] = s
            snap[f"kavg_count{layer}"] = c
            snap[f"mean{layer}"] = backend.mean_keys(layer)
            n = backend.n_pages(layer)
            gk, gv, valid = backend.gather(layer, list(range(n)), grads=True)
            snap[f"gk{layer}"] = gk
            snap[f"valid{layer}"] = valid
        rep = backend.memory_report()
        snap["report"] = np.array([rep[k] for k in ("device_bytes", "host_bytes", "grad_bytes", "pages",
                                                    "arena_blocks", "free_list")], np.int64)
        snaps.append(snap)
        backend.reset()
    return snaps


def c1_cfg() -> Cfg:
    """BASELINE config 1 geometry (tiny: 4Q/1KV, hd 64, P 64, C 256)."""
    return Cfg(n_layers=1, n_q_heads=4, n_kv_heads=1, head_dim=64, chunk_size=256, page_size=64,
               retrieval_budget=256, local_window=4)


def qwen_slice_cfg() -> Cfg:
    """Qwen2.5-7B attention shape (28Q/4KV, hd 128, P 128) on a 512-token chunk."""
    return Cfg(n_layers=1, n_q_heads=28, n_kv_heads=4, head_dim=128, chunk_size=512, page_size=128,
               retrieval_budget=512, local_window=4)


def llama_slice_cfg() -> Cfg:
    """Llama-3-8B attention shape (32Q/8KV, hd 128) with page 256 (BASELINE config 5) on a 512-token chunk."""
    return Cfg(n_layers=1, n_q_heads=32, n_kv_heads=8, head_dim=128, chunk_size=512, page_size=256,
               retrieval_budget=512, local_window=4)


def small_cfg() -> Cfg:
    """test_attention.cpp:19-31 attn_config()."""
    return Cfg(n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=8, chunk_size=16, page_size=8,
               retrieval_budget=16, local_window=4)


def topk_case(cfg: Cfg, n_past_pages: int, seed: int, dtype=np.float32):
    """Planted-structure scoring inputs: page-specific offsets on K so votes have margins."""
    P = cfg.page_size
    pk = det_normal(seed * 16 + 1, (n_past_pages * P, cfg.n_kv_heads, cfg.head_dim), dtype)
    dirs = det_normal(seed * 16 + 7, (n_past_pages, cfg.n_kv_heads, cfg.head_dim), dtype)
    pk = (pk + 2.0 * np.repeat(dirs, P, axis=0)).astype(dtype)
    pv = det_normal(seed * 16 + 2, pk.shape, dtype)
    q = det_normal(seed * 16 + 3, (cfg.chunk_size, cfg.n_q_heads, cfg.head_dim), dtype)
    return pk, pv, q


def main():
    Ref.lib()
    fixtures = {}

    # ---- known answers (test_attention.cpp:54-118) -------------------------
    ka = {}
    r = Ref(Cfg(n_layers=1, n_q_heads=1, n_kv_heads=1, head_dim=2, chunk_size=8, page_size=8,
                retrieval_budget=8), 8)
    ka["score_one_token"] = r.score_pages(np.array([[[1.0, 0.0]]]), np.array([[[1.0, 0.0]], [[0.0, 1.0]]])).tolist()
    q = det_normal(11, (8, 2, 8), np.float64)
    kav = np.tile((0.37 * np.arange(8))[None, None, :], (3, 1, 1))
    r2 = Ref(Cfg(n_layers=1, n_q_heads=2, n_kv_heads=1, head_dim=8, chunk_size=8, page_size=4,
                 retrieval_budget=8), 8)
    ka["score_uniform"] = r2.score_pages(q, kav).tolist()
    ka["topk"] = {
        "ties_k1": Ref.select_topk([5.0, 5.0, 1.0], 1).tolist(),
        "k_ge_n": Ref.select_topk([5.0, 5.0, 1.0], 7).tolist(),
        "k0": Ref.select_topk([5.0, 5.0, 1.0], 0).tolist(),
        "subset": Ref.select_topk([0.1, 9.0, 3.0, 7.0, 0.2], 3).tolist(),
    }
    ka["recent"] = {"10_3": Ref.select_recent(10, 3).tolist(), "2_5": Ref.select_recent(2, 5).tolist(),
                    "4_0": Ref.select_recent(4, 0).tolist()}
    with open(os.path.join(OUT, "known_answers.json"), "w") as f:
        json.dump(ka, f, indent=1)

    # ---- small attention geometry, full arrays ------------------------------
    for rb, dt in ((4, np.float32), (8, np.float64)):
        cfg = small_cfg()
        sel_sets = {
            "dense": None,
            "sparse": [[0, 2], [1, 3, 4]],
            "empty_first": [[], [4, 0, 2]],
        }
        arrays = {}
        for name, sel in sel_sets.items():
            case = attn_case(cfg, 5 * cfg.page_size - 3, seed=21 + rb, dtype=dt, selected=sel)
            res = run_attn(Ref(cfg, rb), cfg, case)
            for k, v in res.items():
                arrays[f"{name}/{k}"] = v
            off = np.zeros(len(case["selected"]) + 1, np.int32)
            for i, l in enumerate(case["selected"]):
                off[i + 1] = off[i] + len(l)
            arrays[f"{name}/sel_off"] = off
            arrays[f"{name}/sel_ids"] = np.array([x for l in case["selected"] for x in l], np.int32)
        np.savez_compressed(os.path.join(OUT, f"attn_small_{'f32' if rb == 4 else 'f64'}.npz"), **arrays)

    # ---- page-table script ---------------------------------------------------
    pcfg = Cfg(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=16, chunk_size=64, page_size=16,
               retrieval_budget=32)
    arrays = {}
    for i, snap in enumerate(pagetable_script(Ref(pcfg, 4), seed=5)):
        for k, v in snap.items():
            arrays[f"s{i}/{k}"] = v
    np.savez_compressed(os.path.join(OUT, "pagetable.npz"), **arrays)

    # ---- selection rows with ties --------------------------------------------
    rng = np.random.default_rng(9)
    rows, ks, outs = [], [], []
    for n in (1, 3, 17, 64, 200, 1000):
        for k in (0, 1, 5, 64, 1000):
            row = rng.integers(0, 6, size=n).astype(np.float32) / 4.0  # heavy ties
            rows.append(np.pad(row, (0, 1000 - n), constant_values=np.nan))
            ks.append((n, k))
            outs.append(np.pad(Ref.select_topk(row.astype(np.float64), k), (0, 1000), constant_values=-1)[:1000])
    np.savez_compressed(os.path.join(OUT, "select.npz"), rows=np.array(rows), nk=np.array(ks, np.int32),
                        ids=np.array(outs, np.int32))

    # ---- hashes at larger geometries ---------------------------------------
    hashes = {}
    for label, cfg, past, seed, sel in (
        ("c1_dense_f32", c1_cfg(), 4 * 64, 31, None),
        ("c1_dense_f64", c1_cfg(), 4 * 64, 31, None),
        ("qwen_slice_sparse_f32", qwen_slice_cfg(), 8 * 128, 41, [[0, 3, 5], [1, 2], [7], [0, 4, 6, 7]]),
    ):
        rb = 8 if label.endswith("f64") else 4
        dt = np.float64 if rb == 8 else np.float32
        case = attn_case(cfg, past, seed=seed, dtype=dt, selected=sel)
        res = run_attn(Ref(cfg, rb), cfg, case)
        hashes[label] = {k: sha(v) for k, v in res.items()}
        hashes[label]["_norms"] = {k: float(np.linalg.norm(v)) for k, v in res.items()}

    # scoring + top-k on planted structure (c1 geometry and the Qwen slice)
    for label, cfg, npages, seed in (("score_c1", c1_cfg(), 12, 51), ("score_qwen", qwen_slice_cfg(), 24, 52)):
        pk, pv, q = topk_case(cfg, npages, seed)
        r = Ref(cfg, 4)
        r.append(0, pk, pv)
        kav = r.mean_keys(0)
        score = r.score_pages(q, kav)
        k = 3
        sel = [Ref.select_topk(score[i].astype(np.float64), k).tolist() for i in range(score.shape[0])]
        hashes[label] = {"kavg": sha(kav), "score": sha(score), "selected": sel}

    with open(os.path.join(OUT, "hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
