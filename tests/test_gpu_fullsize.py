"""Parity at BASELINE.json's full sizes — c3 (Qwen2.5-7B attention, 1M context, top-k 64 pages per
query page), c2 (the same shape dense at 128K), c4 (c3 at 4M context) and c5 (Llama-3-8B attention, page 256, 512K context,
dense): the last chunk of the sequence, through the public API, against a float64
restatement of the reference's math (attention.hpp:32-96 scoring/selection, :156-208 forward,
:222-293 backward) evaluated on the GPU for sampled query pages and heads.

The CPU oracle cannot run this size in test time, so the reference here is a direct float64
evaluation of the same formulas on the same bf16 inputs — votes for sampled query pages, the
top-k ids where the vote margin allows, out / lse / dq for sampled (query page, head) rows, and
the fp32 gradient page of a selected past page summed over every query page that selected it.
Tolerances are the bf16 ones of tests/test_gpu_parity.py (2e-2 relative L2); votes 1e-4.
"""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu

C, HD = 4096, 128
CONFIGS = {  # bench.py CONFIGS
    "c2": dict(T=1 << 17, P=128, HQ=28, HKV=4, k=None),  # dense
    "c3": dict(T=1 << 20, P=128, HQ=28, HKV=4, k=64),
    "c4": dict(T=1 << 22, P=128, HQ=28, HKV=4, k=64),
    "c5": dict(T=1 << 19, P=256, HQ=32, HKV=8, k=None),  # dense
}
TOL = 2e-2


def rel(a, b):
    d = torch.linalg.norm((a.double() - b.double()).flatten())
    n = torch.linalg.norm(b.double().flatten())
    return float(d / n) if n > 0 else float(d)


@pytest.fixture(scope="module", params=sorted(CONFIGS))
def run(request):
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200 import attention as A
    T, P, HQ, HKV, K_SEL = (CONFIGS[request.param][k] for k in ("T", "P", "HQ", "HKV", "k"))
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(2602)
    past = T - C
    n_cand = past // P
    # planted page structure (like tests/golden topk_case): page-specific key offsets give the votes
    # clear margins, so the top-k ids are comparable with a float64 restatement
    dirs = torch.randn(T // P, HKV, HD, device=dev, generator=g)
    K = (torch.randn(T, HKV, HD, device=dev, generator=g) + 0.5 * dirs.repeat_interleave(P, 0)).bfloat16()
    V = torch.randn(T, HKV, HD, device=dev, generator=g).bfloat16()
    q = torch.randn(C, HQ, HD, device=dev, generator=g).bfloat16()
    do = torch.randn(C, HQ, HD, device=dev, generator=g).bfloat16()
    cfg = ModelConfig(n_layers=1, n_q_heads=HQ, n_kv_heads=HKV, head_dim=HD, chunk_size=C, page_size=P,
                      retrieval_budget=(K_SEL or 0) * P, attention_mode=["topk" if K_SEL else "dense"])
    cache = PagedCache(cfg, dtype="bf16", max_tokens=T)
    cache.append_chunk(0, K[:past], V[:past])
    if K_SEL:
        sel = A.select_pages_topk(cache, 0, q, n_candidates=n_cand)
        vote = sel.vote.clone()
    else:
        sel, vote = [A.select_all(n_cand) for _ in range(C // P)], None
    lists = sel.lists() if K_SEL else sel
    kc, vc = K[past:], V[past:]
    cache.append_chunk(0, kc, vc)
    saved = A.attn_forward(cfg, q, cache, 0, sel, kc, vc)
    grads = A.attn_backward(cfg, do, q, cache, 0, kc, vc, saved)
    torch.cuda.synchronize()
    cache.check_device_errors()
    yield dict(cache=cache, K=K, V=V, q=q, do=do, past=past, n_cand=n_cand, vote=vote, lists=lists,
               saved=saved, grads=grads, P=P, HQ=HQ, HKV=HKV, G=HQ // HKV, k=K_SEL, name=request.param)
    del cache, K, V, saved, grads
    torch.cuda.empty_cache()


def _kavg(r):
    P, HKV = r["P"], r["HKV"]
    Kp = r["K"][: r["past"]].double().view(r["n_cand"], P, HKV, HD)
    return Kp.sum(1) * (1.0 / P)  # paged_kv.hpp:177-180: sum * (1/count)


def _ref_rows(r, qp, h):
    """float64 forward + backward of the 128 rows of query page qp, q-head h (attention.hpp)."""
    P, HKV, G = r["P"], r["HKV"], r["G"]
    kvh = h // G
    ids = r["lists"][qp]
    past, K, V = r["past"], r["K"], r["V"]
    kp = K[: past].view(-1, P, HKV, HD)[ids, :, kvh].reshape(-1, HD).double()
    vp = V[: past].view(-1, P, HKV, HD)[ids, :, kvh].reshape(-1, HD).double()
    kcur, vcur = K[past:, kvh].double(), V[past:, kvh].double()
    keys, vals = torch.cat([kp, kcur]), torch.cat([vp, vcur])
    rows = torch.arange(qp * P, qp * P + P, device=keys.device)
    n_past = kp.shape[0]
    causal = torch.arange(C, device=keys.device)[None, :] <= rows[:, None]
    mask = torch.cat([torch.ones(P, n_past, dtype=torch.bool, device=keys.device), causal], 1)
    qr = r["q"][rows, h].double()
    scale = 1.0 / math.sqrt(HD)
    s = (qr @ keys.T) * scale
    s = s.masked_fill(~mask, -math.inf)
    lse = torch.logsumexp(s, 1)
    p = torch.exp(s - lse[:, None])
    out = p @ vals
    dor = r["do"][rows, h].double()
    o_saved = r["saved"].out[rows, h].double()  # D uses the saved O (attention.hpp:253-256)
    D = (dor * o_saved).sum(1)
    dp = dor @ vals.T
    ds = p * (dp - D[:, None])
    dq = (ds @ keys) * scale
    return dict(rows=rows, out=out, lse=lse, dq=dq, ds=ds * scale, p=p, dor=dor, qr=qr, n_past=n_past, ids=ids)


def test_fullsize_votes_and_topk(run):
    r = run
    if not r["k"]:
        pytest.skip("dense config: no scoring")
    P, HQ, G, K_SEL = r["P"], r["HQ"], r["G"], r["k"]
    assert len(r["lists"]) == C // P and all(len(x) == K_SEL for x in r["lists"])
    kavg = _kavg(r)
    for qp in (0, 13, 31):
        qr = r["q"][qp * P:(qp + 1) * P].double()  # [128, HQ, HD]
        vote = torch.zeros(r["n_cand"], dtype=torch.float64, device=qr.device)
        for h in range(HQ):
            s = qr[:, h] @ kavg[:, h // G].T  # unscaled (score_scale off), [128, n]
            vote += torch.softmax(s, 1).sum(0)
        got = r["vote"][qp].double()
        assert rel(got, vote) < 1e-4, qp
        order = sorted(range(r["n_cand"]), key=lambda p: (-float(vote[p]), p))
        want = sorted(order[:K_SEL])
        margin = float(vote[order[K_SEL - 1]] - vote[order[K_SEL]]) / float(vote[order[K_SEL - 1]])
        if margin > 1e-3:  # clear boundary: the ids must match exactly
            assert r["lists"][qp] == want, qp
        else:  # near tie at the boundary: everything above it must be selected
            assert set(order[:K_SEL - 1]) <= set(r["lists"][qp]), qp


@pytest.mark.parametrize("qp,h", [(0, 0), (7, 13), (13, 6), (-1, -1)])
def test_fullsize_forward_and_dq_rows(run, qp, h):
    r = run
    qp, h = qp % (C // r["P"]), h % r["HQ"]
    ref = _ref_rows(r, qp, h)
    rows = ref["rows"]
    assert rel(r["saved"].out[rows, h], ref["out"]) < TOL
    assert rel(r["saved"].lse[rows, h], ref["lse"]) < 1e-4
    assert rel(r["grads"].dq[rows, h], ref["dq"]) < TOL


def test_fullsize_grad_page(run):
    """dK / dV of one past page (kv head 1) = sum over every (query page that selected it, q-head
    of the group, row) of dS^T q and P^T dO — the page's gradient block after the backward."""
    r = run
    if not r["k"]:
        pytest.skip("dense config: every query page selects every page (covered by the row checks)")
    P, G = r["P"], r["G"]
    kvh = 1
    counts = {}
    for ids in r["lists"]:
        for p in ids:
            counts[p] = counts.get(p, 0) + 1
    pid = max(counts, key=lambda p: (counts[p], -p))  # the page most query pages selected
    dk = torch.zeros(P, HD, dtype=torch.float64, device="cuda")
    dv = torch.zeros_like(dk)
    for qp, ids in enumerate(r["lists"]):
        if pid not in ids:
            continue
        j = ids.index(pid)
        for h in range(kvh * G, (kvh + 1) * G):
            ref = _ref_rows(r, qp, h)
            cols = slice(j * P, (j + 1) * P)
            dk += ref["ds"][:, cols].T @ ref["qr"]
            dv += ref["p"][:, cols].T @ ref["dor"]
    got = r["cache"].gather_grad_pages(0, [pid])
    assert counts[pid] >= 2
    assert rel(got.k[:, kvh], dk) < TOL
    assert rel(got.v[:, kvh], dv) < TOL
