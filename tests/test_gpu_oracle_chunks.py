"""Cross-chunk parity at the BASELINE shape against the CPU oracle (oracle/oomb_oracle.c).

One KV group of Qwen2.5-7B attention (7 q-heads over 1 kv head, head dim 128, page 128,
chunk 4096) runs several consecutive chunks through the public API, exactly as the
reference's chunk loop does (chunk_trainer.hpp:409-437 forward: select over the pages of
earlier chunks, append the chunk, attend; backward_from_loss_ in reverse chunk order,
attention.hpp:222-293, every past page's dK/dV accumulating in the paged gradient pool):

* c2-style dense, 3 chunks (chunk 2 attends 64 past pages + its causal prefix);
* c3-style top-k 64 pages per query page, 4 chunks (chunk 3 selects 64 of 96 candidates).

Every output is compared IN FULL with the oracle on the same bf16-rounded inputs: the votes
(1e-4), the selected ids (bit-exact; the planted page structure gives margins far above the
vote tolerance, asserted), out / lse / dq / dk_cur / dv_cur of every chunk and the whole
fp32 gradient pool after the backward (bf16 tolerance 2e-2, BASELINE.json north_star).

The oracle is single-threaded C; it runs one instance per q-head on the host's cores
(ctypes releases the GIL). A head's instance (1 q-head / 1 kv head) computes exactly that
head's rows of out / lse / dq and that head's share of dK / dV; the shares are summed over
the 7 heads in float64. Selection needs all 7 heads (the vote sums over every head,
attention.hpp:43-64), so it comes from one 7-head instance.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G, HD, P, C = 7, 128, 128, 4096
M = C // P
K_SEL = 64
TOL = 2e-2
VOTE_TOL = 1e-4
CASES = {"c2_dense_3chunks": ("dense", 3), "c3_topk_4chunks": ("topk", 4)}


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    n = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / n) if n > 0 else float(np.linalg.norm(a - b))


def _inputs(mode, n_chunks, seed=2602):
    from oracle.oracle import to_bf16
    rng = np.random.default_rng(seed)
    T = n_chunks * C
    K = rng.standard_normal((T, 1, HD), dtype=np.float32)
    if mode == "topk":  # planted page structure: page-specific key offsets give the votes clear margins
        dirs = rng.standard_normal((T // P, 1, HD), dtype=np.float32)
        K = K + 0.5 * np.repeat(dirs, P, axis=0)
    V = rng.standard_normal((T, 1, HD), dtype=np.float32)
    q = rng.standard_normal((n_chunks, C, G, HD), dtype=np.float32)
    do = rng.standard_normal((n_chunks, C, G, HD), dtype=np.float32)
    return dict(K=to_bf16(K), V=to_bf16(V), q=to_bf16(q), do=to_bf16(do), T=T)


def _oracle_selection(mode, n_chunks, x):
    """Per chunk: the oracle's votes and selected lists (7-head instance, reference order)."""
    from oracle.oracle import Cfg, Port
    cfg = Cfg(n_layers=1, n_q_heads=G, n_kv_heads=1, head_dim=HD, chunk_size=C, page_size=P,
              retrieval_budget=K_SEL * P, local_window=4)
    port = Port(cfg, 4)
    votes, sels = [], []
    for i in range(n_chunks):
        n_cand = i * M
        if mode == "topk" and n_cand > 0:
            kavg = port.mean_keys(0, n_cand)
            v = port.score_pages(x["q"][i], kavg)
            votes.append(v)
            sels.append([list(Port.select_topk(v[qp], K_SEL)) for qp in range(M)])
        else:
            votes.append(None)
            sels.append([list(range(n_cand)) for _ in range(M)])
        port.append(0, x["K"][i * C:(i + 1) * C], x["V"][i * C:(i + 1) * C])
    return votes, sels


def _oracle_head(h, n_chunks, x, sels):
    """One q-head's forward (chunks ascending) and backward (descending) through the oracle."""
    from oracle.oracle import Cfg, Port
    cfg = Cfg(n_layers=1, n_q_heads=1, n_kv_heads=1, head_dim=HD, chunk_size=C, page_size=P,
              retrieval_budget=K_SEL * P, local_window=4)
    port = Port(cfg, 4)
    fw = []
    for i in range(n_chunks):
        kc, vc = x["K"][i * C:(i + 1) * C], x["V"][i * C:(i + 1) * C]
        port.append(0, kc, vc)
        q = np.ascontiguousarray(x["q"][i][:, h:h + 1])
        fw.append(port.attn_forward(0, q, sels[i], kc, vc))
    bw = [None] * n_chunks
    for i in reversed(range(n_chunks)):
        kc, vc = x["K"][i * C:(i + 1) * C], x["V"][i * C:(i + 1) * C]
        q = np.ascontiguousarray(x["q"][i][:, h:h + 1])
        do = np.ascontiguousarray(x["do"][i][:, h:h + 1])
        bw[i] = port.attn_backward(0, do, q, sels[i], kc, vc, *fw[i])
    n_pages = port.n_pages(0)
    gk, gv, _ = port.gather(0, list(range(n_pages)), grads=True)
    return fw, bw, gk, gv


@pytest.fixture(scope="module", params=sorted(CASES))
def case(request):
    import torch
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200 import attention as A
    mode, n_chunks = CASES[request.param]
    x = _inputs(mode, n_chunks)
    # ---- the oracle, one instance per q-head on the host's cores
    votes, sels = _oracle_selection(mode, n_chunks, x)
    workers = max(1, min(G, os.cpu_count() or 1))
    with ThreadPoolExecutor(workers) as ex:
        heads = list(ex.map(lambda h: _oracle_head(h, n_chunks, x, sels), range(G)))
    # ---- the device path (public API), the same chunk loop
    dev = torch.device("cuda")
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev, torch.bfloat16)
    cfg = ModelConfig(n_layers=1, n_q_heads=G, n_kv_heads=1, head_dim=HD, chunk_size=C, page_size=P,
                      retrieval_budget=K_SEL * P, attention_mode=[mode])
    cache = PagedCache(cfg, dtype="bf16", max_tokens=x["T"])
    got = dict(votes=[], lists=[], saved=[], grads=[None] * n_chunks)
    for i in range(n_chunks):
        q, kc, vc = bf(x["q"][i]), bf(x["K"][i * C:(i + 1) * C]), bf(x["V"][i * C:(i + 1) * C])
        n_cand = i * M
        if mode == "topk" and n_cand > 0:
            sel = A.select_pages_topk(cache, 0, q, n_cand)
            got["votes"].append(sel.vote.double().cpu().numpy())
            lists = sel.lists()
        else:
            got["votes"].append(None)
            sel = lists = [A.select_all(n_cand) for _ in range(M)]
        got["lists"].append(lists)
        cache.append_chunk(0, kc, vc)
        got["saved"].append(A.attn_forward(cfg, q, cache, 0, sel, kc, vc))
    for i in reversed(range(n_chunks)):
        q, kc, vc = bf(x["q"][i]), bf(x["K"][i * C:(i + 1) * C]), bf(x["V"][i * C:(i + 1) * C])
        g = A.attn_backward(cfg, bf(x["do"][i]), q, cache, 0, kc, vc, got["saved"][i])
        got["grads"][i] = tuple(t.double().cpu().numpy() for t in (g.dq, g.dk_cur, g.dv_cur))
    gp = cache.gather_grad_pages(0, list(range(cache.n_pages(0))))
    got["gk"], got["gv"] = gp.k.double().cpu().numpy(), gp.v.double().cpu().numpy()
    torch.cuda.synchronize()
    cache.check_device_errors()
    got["saved"] = [(s.out.double().cpu().numpy(), s.lse.double().cpu().numpy()) for s in got["saved"]]
    yield dict(mode=mode, n=n_chunks, votes=votes, sels=sels, heads=heads, got=got)
    del cache
    torch.cuda.empty_cache()


def test_chunks_selection(case):
    """Votes within 1e-4 of the oracle; selected ids bit-exact wherever the oracle's k-boundary
    margin exceeds twice the row's largest vote difference (SURVEY 7 hard part 4), and otherwise
    differing only in pages whose votes sit within that distance of the boundary."""
    if case["mode"] != "topk":
        pytest.skip("dense: select_all")
    got = case["got"]
    n_rows = n_exact = 0
    for i in range(case["n"]):
        if case["votes"][i] is None:
            assert got["votes"][i] is None
            continue
        want = case["votes"][i].astype(np.float64)
        assert rel(got["votes"][i], want) < VOTE_TOL, f"chunk {i} votes {rel(got['votes'][i], want):.2e}"
        for qp in range(M):
            g_ids = [int(v) for v in got["lists"][i][qp]]
            w_ids = [int(v) for v in case["sels"][i][qp]]
            n_rows += 1
            if len(want[qp]) <= K_SEL:  # k >= n: every page, ascending
                assert g_ids == w_ids == list(range(len(want[qp])))
                n_exact += 1
                continue
            err = float(np.max(np.abs(got["votes"][i][qp] - want[qp])))
            row = np.sort(want[qp])[::-1]
            boundary = 0.5 * (row[K_SEL - 1] + row[K_SEL])
            if row[K_SEL - 1] - row[K_SEL] > 2 * err:
                assert g_ids == w_ids, f"chunk {i} qp {qp} ids (margin {row[K_SEL - 1] - row[K_SEL]:.3g}, err {err:.3g})"
                n_exact += 1
            else:
                for pg in set(g_ids) ^ set(w_ids):
                    assert abs(want[qp][pg] - boundary) <= 2 * err, f"chunk {i} qp {qp} page {pg} off the boundary"
    assert n_rows >= 3 * M and n_exact >= 0.9 * n_rows, (n_rows, n_exact)


def test_chunks_forward(case):
    """out and lse of every chunk, every head, every row."""
    got, heads = case["got"], case["heads"]
    for i in range(case["n"]):
        out = np.concatenate([heads[h][0][i][0] for h in range(G)], axis=1)
        lse = np.concatenate([heads[h][0][i][1] for h in range(G)], axis=1)
        assert rel(got["saved"][i][0], out) < TOL, f"chunk {i} out {rel(got['saved'][i][0], out):.3e}"
        assert rel(got["saved"][i][1], lse) < TOL, f"chunk {i} lse"


def test_chunks_backward(case):
    """dq of every head, dk_cur / dv_cur summed over the group's heads, every chunk."""
    got, heads = case["got"], case["heads"]
    for i in range(case["n"]):
        dq = np.concatenate([heads[h][1][i][0] for h in range(G)], axis=1)
        dk = sum(heads[h][1][i][1].astype(np.float64) for h in range(G))
        dv = sum(heads[h][1][i][2].astype(np.float64) for h in range(G))
        gq, gk, gv = got["grads"][i]
        for name, a, b in (("dq", gq, dq), ("dk_cur", gk, dk), ("dv_cur", gv, dv)):
            assert rel(a, b) < TOL, f"chunk {i} {name} {rel(a, b):.3e}"


def test_chunks_gradient_pool(case):
    """The whole fp32 gradient pool after the reverse-chunk backward (every page, summed heads)."""
    got, heads = case["got"], case["heads"]
    gk = sum(heads[h][2].astype(np.float64) for h in range(G))
    gv = sum(heads[h][3].astype(np.float64) for h in range(G))
    n_past = (case["n"] - 1) * M  # pages of the last chunk are never a past page of a later chunk
    assert np.all(gk[n_past * P:] == 0) and np.all(got["gk"][n_past * P:] == 0)
    assert rel(got["gk"], gk) < TOL, f"grad_k {rel(got['gk'], gk):.3e}"
    assert rel(got["gv"], gv) < TOL, f"grad_v {rel(got['gv'], gv):.3e}"
    # per page as well: no page may hide a large error inside the whole-pool norm
    for pg in range(n_past):
        sl = slice(pg * P, (pg + 1) * P)
        if np.linalg.norm(gk[sl]) > 0:
            assert rel(got["gk"][sl], gk[sl]) < 3 * TOL, f"page {pg} grad_k"
            assert rel(got["gv"][sl], gv[sl]) < 3 * TOL, f"page {pg} grad_v"
