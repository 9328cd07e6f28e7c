"""The C restatement (oracle/oomb_oracle.c) against golden vectors produced by
the reference itself (tests/golden/make_golden.py). Bit-exact: the oracle uses
the reference's floating-point operation order and is built with
-ffp-contract=off, so every comparison here is on raw bytes."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle.oracle import Cfg, OracleError, Port, Ref, det_normal
from tests.golden.make_golden import (attn_case, c1_cfg, pagetable_script, qwen_slice_cfg, run_attn,
                                      small_cfg, topk_case)

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def test_known_answers():
    ka = json.load(open(os.path.join(G, "known_answers.json")))
    p = Port(Cfg(n_layers=1, n_q_heads=1, n_kv_heads=1, head_dim=2, chunk_size=8, page_size=8,
                 retrieval_budget=8), 8)
    s = p.score_pages(np.array([[[1.0, 0.0]]]), np.array([[[1.0, 0.0]], [[0.0, 1.0]]]))
    assert s.tolist() == ka["score_one_token"]
    assert abs(s[0, 0] - 0.731058578) < 1e-6 and abs(s[0, 1] - 0.268941421) < 1e-6
    q = det_normal(11, (8, 2, 8), np.float64)
    kav = np.tile((0.37 * np.arange(8))[None, None, :], (3, 1, 1))
    p2 = Port(Cfg(n_layers=1, n_q_heads=2, n_kv_heads=1, head_dim=8, chunk_size=8, page_size=4,
                  retrieval_budget=8), 8)
    s2 = p2.score_pages(q, kav)
    assert s2.tolist() == ka["score_uniform"]
    assert np.allclose(s2, 4 * 2 / 3.0, atol=1e-9)  # P * Hq / n (test_attention.cpp:66-83)
    t = ka["topk"]
    assert Port.select_topk([5.0, 5.0, 1.0], 1).tolist() == t["ties_k1"] == [0]
    assert Port.select_topk([5.0, 5.0, 1.0], 7).tolist() == t["k_ge_n"] == [0, 1, 2]
    assert Port.select_topk([5.0, 5.0, 1.0], 0).tolist() == t["k0"] == []
    assert Port.select_topk([0.1, 9.0, 3.0, 7.0, 0.2], 3).tolist() == t["subset"] == [1, 2, 3]
    r = ka["recent"]
    assert Port.select_recent(10, 3).tolist() == r["10_3"] == [7, 8, 9]
    assert Port.select_recent(2, 5).tolist() == r["2_5"] == [0, 1]
    assert Port.select_recent(4, 0).tolist() == r["4_0"] == []
    with pytest.raises(OracleError):
        Port.select_topk([1.0], -1)


@pytest.mark.parametrize("rb", [4, 8])
@pytest.mark.parametrize("name", ["dense", "sparse", "empty_first"])
def test_attention_small_bit_exact(rb, name):
    g = np.load(os.path.join(G, f"attn_small_{'f32' if rb == 4 else 'f64'}.npz"))
    cfg = small_cfg()
    dt = np.float32 if rb == 4 else np.float64
    off, ids = g[f"{name}/sel_off"], g[f"{name}/sel_ids"]
    sel = [ids[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1)]
    case = attn_case(cfg, 5 * cfg.page_size - 3, seed=21 + rb, dtype=dt,
                     selected=None if name == "dense" else sel)
    res = run_attn(Port(cfg, rb), cfg, case)
    for k, v in res.items():
        assert bits_equal(v, g[f"{name}/{k}"]), (name, k)


def test_pagetable_script_bit_exact():
    g = np.load(os.path.join(G, "pagetable.npz"))
    pcfg = Cfg(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=16, chunk_size=64, page_size=16,
               retrieval_budget=32)
    for i, snap in enumerate(pagetable_script(Port(pcfg, 4), seed=5)):
        for k, v in snap.items():
            assert bits_equal(np.asarray(v), g[f"s{i}/{k}"].astype(np.asarray(v).dtype)), (i, k)


def test_select_ties_match_reference():
    g = np.load(os.path.join(G, "select.npz"))
    for row, (n, k), ids in zip(g["rows"], g["nk"], g["ids"]):
        got = Port.select_topk(row[:n].astype(np.float64), k)
        want = ids[ids >= 0]
        assert got.tolist() == want.tolist(), (n, k)


@pytest.mark.parametrize("label", ["c1_dense_f32", "c1_dense_f64", "qwen_slice_sparse_f32"])
def test_attention_hashes(label):
    h = json.load(open(os.path.join(G, "hashes.json")))[label]
    cfg = c1_cfg() if label.startswith("c1") else qwen_slice_cfg()
    rb = 8 if label.endswith("f64") else 4
    dt = np.float64 if rb == 8 else np.float32
    sel = None if label.startswith("c1") else [[0, 3, 5], [1, 2], [7], [0, 4, 6, 7]]
    past = 4 * 64 if label.startswith("c1") else 8 * 128
    seed = 31 if label.startswith("c1") else 41
    res = run_attn(Port(cfg, rb), cfg, attn_case(cfg, past, seed=seed, dtype=dt, selected=sel))
    for k, v in res.items():
        assert sha(v) == h[k], (label, k)


@pytest.mark.parametrize("label", ["score_c1", "score_qwen"])
def test_scoring_hashes(label):
    h = json.load(open(os.path.join(G, "hashes.json")))[label]
    cfg, npages, seed = (c1_cfg(), 12, 51) if label == "score_c1" else (qwen_slice_cfg(), 24, 52)
    pk, pv, q = topk_case(cfg, npages, seed)
    p = Port(cfg, 4)
    p.append(0, pk, pv)
    kav = p.mean_keys(0)
    score = p.score_pages(q, kav)
    assert sha(kav) == h["kavg"]
    assert sha(score) == h["score"]
    sel = [Port.select_topk(score[i].astype(np.float64), 3).tolist() for i in range(score.shape[0])]
    assert sel == h["selected"]


def test_naive_matches_streaming_f64():
    """test_attention.cpp:249-298 on the oracle: the streaming paged path equals
    the independent naive attention within 1e-10 (f64)."""
    cfg = small_cfg()
    past = 3 * cfg.page_size
    case = attn_case(cfg, past, seed=9, dtype=np.float64)
    res = run_attn(Port(cfg, 8), cfg, case)
    allk = np.concatenate([case["pk"], case["kc"]])
    allv = np.concatenate([case["pv"], case["vc"]])
    out, dq, dk, dv = Port(cfg, 8).naive_attention(case["q"], allk, allv, past, case["do"], cfg.gqa_group)

    def rel(a, b):
        return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)

    assert rel(res["out"], out) < 1e-10
    assert rel(res["dq"], dq) < 1e-10
    assert rel(res["grad_k"], dk[:past]) < 1e-10
    assert rel(res["grad_v"], dv[:past]) < 1e-10
    assert rel(res["dk_cur"], dk[past:]) < 1e-10
    assert rel(res["dv_cur"], dv[past:]) < 1e-10


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_port_equals_reference_live_random():
    """When the reference build is present, a fresh random case is also checked live."""
    cfg = Cfg(n_layers=1, n_q_heads=6, n_kv_heads=2, head_dim=16, chunk_size=24, page_size=8,
              retrieval_budget=16)
    case = attn_case(cfg, 7 * 8 - 5, seed=77, dtype=np.float32, selected=[[6, 1], [], [0, 2, 3, 4, 5, 6]])
    a = run_attn(Port(cfg, 4), cfg, case)
    b = run_attn(Ref(cfg, 4), cfg, case)
    for k in a:
        assert bits_equal(a[k], b[k]), k
