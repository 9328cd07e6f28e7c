"""Parity of the sm_100a kernels with the CPU oracle (oracle/oomb_oracle.c, itself
pinned bit-exactly to the reference by tests/test_oracle_golden.py).

Tolerances (BASELINE.json north_star): fp32 mode 1e-5 relative L2 per output
tensor; bf16 mode 2e-2 relative L2 against the oracle run on the bf16-rounded
inputs up-cast to fp32. Page tables, K_avg sums and top-k ids are bit-exact.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import Cfg, Port, det_normal, to_bf16
from tests.golden.make_golden import attn_case, c1_cfg, llama_slice_cfg, qwen_slice_cfg, small_cfg, topk_case

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 2e-2


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return d if n == 0 else d / n


def T(x):
    return x.detach().float().cpu().numpy()


def model_cfg(c: Cfg, **kw):
    from paper_2602_02108_b200 import ModelConfig
    return ModelConfig(n_layers=c.n_layers, n_q_heads=c.n_q_heads, n_kv_heads=c.n_kv_heads, head_dim=c.head_dim,
                       chunk_size=c.chunk_size, page_size=c.page_size, retrieval_budget=c.retrieval_budget,
                       local_window=c.local_window, **kw)


def cache_for(c: Cfg, dtype, max_tokens=None, **kw):
    from paper_2602_02108_b200 import PagedCache
    return PagedCache(model_cfg(c), dtype=dtype, max_tokens=max_tokens or 64 * c.chunk_size, **kw)


def run_device(c: Cfg, case, dtype, policy="auto"):
    """append(past) -> append(chunk) -> attn_forward -> attn_backward through the public API."""
    from paper_2602_02108_b200 import attention as A
    cache = cache_for(c, dtype)
    cache.set_kernel_policy(policy)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", tdt)
    if len(case["pk"]):
        cache.append_chunk(0, dev(case["pk"]), dev(case["pv"]))
    n_past = cache.n_pages(0)
    q, kc, vc, do = dev(case["q"]), dev(case["kc"]), dev(case["vc"]), dev(case["do"])
    cache.append_chunk(0, kc, vc)
    saved = A.attn_forward(cache.cfg, q, cache, 0, case["selected"], kc, vc)
    grads = A.attn_backward(cache.cfg, do, q, cache, 0, kc, vc, saved)
    gp = cache.gather_grad_pages(0, list(range(n_past)))
    torch.cuda.synchronize()
    cache.check_device_errors()
    return dict(out=T(saved.out), lse=T(saved.lse), dq=T(grads.dq), dk_cur=T(grads.dk_cur), dv_cur=T(grads.dv_cur),
                grad_k=T(gp.k), grad_v=T(gp.v), page_table=cache.page_table(0)), cache


def run_oracle(c: Cfg, case, rb=4):
    from tests.golden.make_golden import run_attn
    return run_attn(Port(c, rb), c, case)


def bf16_case(case):
    out = dict(case)
    for k in ("pk", "pv", "q", "kc", "vc", "do"):
        out[k] = to_bf16(case[k])
    return out


# ---------------------------------------------------------------------------
# tcgen05 / TMA building blocks
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("mode,n,k", [(0, 128, 128), (0, 256, 64), (0, 64, 128), (1, 128, 128), (1, 256, 64),
                                      (2, 128, 128), (2, 64, 64), (3, 128, 128), (3, 64, 64), (4, 128, 128),
                                      (4, 64, 128)])
def test_tc_gemm_descriptors(mode, n, k):
    from paper_2602_02108_b200.attention import debug_tc_gemm
    g = torch.Generator(device="cuda").manual_seed(mode * 1000 + n + k)
    a = torch.randn(128, k, device="cuda", generator=g).bfloat16()
    if mode in (0, 4):
        b = torch.randn(n, k, device="cuda", generator=g).bfloat16()
        want = a.float() @ b.float().T
    else:
        b = torch.randn(k, n, device="cuda", generator=g).bfloat16()
        want = a.float() @ b.float()
    got = debug_tc_gemm(mode, a, b, n)
    torch.cuda.synchronize()
    assert rel(T(got), T(want)) < 1e-5


# ---------------------------------------------------------------------------
# page manager
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_append_gather_kavg_bit_exact(dtype):
    c = Cfg(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=16, chunk_size=64, page_size=16, retrieval_budget=32)
    cache = cache_for(c, dtype)
    oracle = Port(c, 4)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rng = np.random.default_rng(3)
    for i in range(8):
        layer = i % 2
        rows = int(rng.integers(1, 60))
        k = to_bf16(det_normal(100 + i, (rows, 2, 16)))
        v = to_bf16(det_normal(200 + i, (rows, 2, 16)))
        r = cache.append_chunk(layer, torch.from_numpy(k).to("cuda", tdt), torch.from_numpy(v).to("cuda", tdt))
        assert (r.begin, r.end) == oracle.append(layer, k, v)
    for layer in range(2):
        n = cache.n_pages(layer)
        assert n == oracle.n_pages(layer)
        assert cache.page_table(layer).tolist() == oracle.page_table(layer).tolist()
        s, cnt = cache.kavg_raw(layer)
        os_, ocnt = oracle.kavg_raw(layer)
        assert np.array_equal(T(s), os_) and np.array_equal(cnt.cpu().numpy(), ocnt)
        assert np.array_equal(T(cache.page_mean_keys(layer)), oracle.mean_keys(layer))
        ids = list(rng.permutation(n))
        g = cache.gather_pages(layer, ids)
        ok, ov, ovalid = oracle.gather(layer, ids)
        assert np.array_equal(T(g.k), ok) and np.array_equal(T(g.v), ov)
        assert np.array_equal(g.valid.cpu().numpy(), ovalid)


def test_scatter_lazy_grads_and_reset_reuse():
    c = Cfg(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=16, chunk_size=64, page_size=16, retrieval_budget=32)
    cache = cache_for(c, "fp32")
    oracle = Port(c, 4)
    for step in range(2):
        for layer in range(2):
            z = det_normal(7 + step + layer, (3 * 16 + 5, 2, 16))
            cache.append_chunk(layer, torch.from_numpy(z).cuda(), torch.from_numpy(z).cuda())
            oracle.append(layer, z, z)
        assert cache.memory_report().grad_bytes == 0 or step > 0
        gk = cache.gather_grad_pages(0, [0, 1])
        assert float(gk.k.abs().sum()) == 0.0
        for ids in ([3, 1], [0, 3], [2], [1, 1, 0]):  # a repeated id adds twice, in list order
            dk = det_normal(50 + len(ids) + step, (len(ids) * 16, 2, 16))
            dv = -2 * dk
            cache.scatter_add_grads(0, ids, torch.from_numpy(dk).cuda(), torch.from_numpy(dv).cuda())
            oracle.scatter(0, ids, dk, dv)
        assert cache.page_table(0).tolist() == oracle.page_table(0).tolist()
        g = cache.gather_grad_pages(0, [0, 1, 2, 3])
        ok, ov, _ = oracle.gather(0, [0, 1, 2, 3], grads=True)
        assert np.array_equal(T(g.k), ok) and np.array_equal(T(g.v), ov)
        rep, orep = cache.memory_report(), oracle.memory_report()
        assert (rep.device_bytes, rep.grad_bytes, rep.pages, rep.arena_blocks, rep.free_list) == \
            (orep["device_bytes"], orep["grad_bytes"], orep["pages"], orep["arena_blocks"], orep["free_list"])
        cache.reset()
        oracle.reset()


def test_residency_enforcement():
    from paper_2602_02108_b200 import ResidencyError
    c = Cfg(n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=16, chunk_size=16, page_size=16, retrieval_budget=32)
    cache = cache_for(c, "fp32")
    z = torch.randn(16, 2, 16, device="cuda")
    cache.append_chunk(0, z, z)
    cache.set_tier(0, 0, 1)
    cache.gather_pages(0, [0])  # enforcement off by default
    cache.set_residency_enforced(True)
    with pytest.raises(ResidencyError):
        cache.gather_pages(0, [0])
    cache.set_tier(0, 0, 0)
    cache.gather_pages(0, [0])


# ---------------------------------------------------------------------------
# scoring and selection
# ---------------------------------------------------------------------------
def test_select_known_answers_on_device():
    from paper_2602_02108_b200.attention import select_topk
    assert select_topk([5.0, 5.0, 1.0], 1) == [0]
    assert select_topk([5.0, 5.0, 1.0], 7) == [0, 1, 2]
    assert select_topk([5.0, 5.0, 1.0], 0) == []
    assert select_topk([0.1, 9.0, 3.0, 7.0, 0.2], 3) == [1, 2, 3]
    assert select_topk([0.0, -0.0, 0.0], 2) == [0, 1]


def test_topk_bit_exact_with_ties():
    from paper_2602_02108_b200.attention import select_topk_rows
    from paper_2602_02108_b200 import PagedCache
    cache = cache_for(small_cfg(), "fp32")
    rng = np.random.default_rng(11)
    for n in (1, 7, 64, 1000, 8160, 32768):
        for k in (0, 1, 3, 64, 5000):
            m = 4
            v = (rng.integers(0, 9, size=(m, n)) / 8.0).astype(np.float32)
            v[1] = rng.standard_normal(n).astype(np.float32)
            sel = select_topk_rows(cache, torch.from_numpy(v), k).lists()
            for i in range(m):
                assert sel[i] == Port.select_topk(v[i].astype(np.float64), k).tolist(), (n, k, i)


def test_score_pages_known_answer():
    from paper_2602_02108_b200.attention import score_pages
    s = score_pages(torch.tensor([[[1.0, 0.0]]]), torch.tensor([[[1.0, 0.0]], [[0.0, 1.0]]]), 8, 1)
    assert abs(float(s[0, 0]) - 0.731058578) < 1e-6 and abs(float(s[0, 1]) - 0.268941421) < 1e-6
    q = torch.from_numpy(det_normal(11, (8, 2, 8)))
    kav = torch.tile((0.37 * torch.arange(8.0))[None, None, :], (3, 1, 1))
    u = score_pages(q, kav, 4, 2)
    assert torch.allclose(u.cpu(), torch.full((2, 3), 4 * 2 / 3.0), atol=1e-5)


# relative L2 of the tcgen05 scorer's votes vs the fp32 reference (hi/lo bf16 split of K_avg)
TC_VOTE_TOL = 1e-4


@pytest.mark.parametrize("geom,dtype", [("c1", "fp32"), ("qwen", "fp32"), ("c1", "bf16"), ("qwen", "bf16")])
def test_scoring_and_selection_parity(geom, dtype):
    from paper_2602_02108_b200.attention import select_pages_topk
    c, npages, seed = (c1_cfg(), 12, 51) if geom == "c1" else (qwen_slice_cfg(), 24, 52)
    pk, pv, q = topk_case(c, npages, seed)
    if dtype == "bf16":
        pk, pv, q = to_bf16(pk), to_bf16(pv), to_bf16(q)
    c = Cfg(**{**c.__dict__, "retrieval_budget": 3 * c.page_size})
    cache = cache_for(c, dtype)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    cache.append_chunk(0, torch.from_numpy(pk).to("cuda", tdt), torch.from_numpy(pv).to("cuda", tdt))
    oracle = Port(c, 4)
    oracle.append(0, pk, pv)
    want_vote = oracle.score_pages(q, oracle.mean_keys(0))
    sel = select_pages_topk(cache, 0, torch.from_numpy(q).to("cuda", tdt), npages)
    got_vote = T(sel.vote)
    # fp32 mode (and shapes on the exact SIMT scorer) meet 1e-5; the bf16 tcgen05 scorer
    # multiplies by K_avg split into hi + lo bf16 planes (~16 mantissa bits), fp32 accumulate.
    tc = dtype == "bf16" and geom == "qwen"
    tol = TC_VOTE_TOL if tc else FP32_TOL
    assert rel(got_vote, want_vote) < tol, rel(got_vote, want_vote)
    lists = sel.lists()
    checked = 0
    for i in range(want_vote.shape[0]):
        want = Port.select_topk(want_vote[i].astype(np.float64), 3).tolist()
        row = np.sort(want_vote[i])[::-1]
        margin = (row[2] - row[3]) / max(abs(row[2]), 1e-30)
        if margin > 10 * tol:  # ids are defined bit-exactly only where the k-boundary margin exceeds score tolerance
            assert lists[i] == want
            checked += 1
    assert checked >= 1


@pytest.mark.parametrize("n_pages,tokens", [(300, 512), (1000, 1024), (40, 256), (8300, 256)])  # 8300: long rows (65 candidate blocks)
def test_tc_scorer_matches_exact_scorer(n_pages, tokens):
    """The tcgen05 two-pass scorer against the exact SIMT scorer on the same pool:
    votes within the bf16-operand tolerance, and identical top-k where margins allow."""
    from paper_2602_02108_b200.attention import select_pages_topk
    c = Cfg(n_layers=1, n_q_heads=28, n_kv_heads=4, head_dim=128, chunk_size=tokens, page_size=128,
            retrieval_budget=8 * 128)
    cache = cache_for(c, "bf16", max_tokens=(n_pages + 8) * 128)
    g = torch.Generator(device="cuda").manual_seed(n_pages)
    k = torch.randn(n_pages * 128, 4, 128, device="cuda", generator=g)
    k += 1.5 * torch.randn(n_pages, 1, 4, 128, device="cuda", generator=g).repeat_interleave(128, 0)[:, 0]
    cache.append_chunk(0, k.bfloat16(), torch.randn_like(k).bfloat16())
    q = torch.randn(tokens, 28, 128, device="cuda", generator=g).bfloat16()
    tc = select_pages_topk(cache, 0, q, n_pages)
    v_tc = tc.vote.clone()
    cache.set_kernel_policy("simt")
    ex = select_pages_topk(cache, 0, q, n_pages)
    v_ex = ex.vote.clone()
    torch.cuda.synchronize()
    err = rel(T(v_tc), T(v_ex))
    assert err < TC_VOTE_TOL, err
    a, b = tc.lists(), ex.lists()
    vv = T(v_ex)
    checked = 0
    for i in range(len(a)):
        row = np.sort(vv[i])[::-1]
        if (row[7] - row[8]) / row[7] > 10 * TC_VOTE_TOL:
            assert a[i] == b[i]
            checked += 1
    assert checked >= len(a) // 2, (checked, len(a))


# ---------------------------------------------------------------------------
# attention forward / backward
# ---------------------------------------------------------------------------
ATTN_CASES = {
    "small_dense": (small_cfg, 5 * 8 - 3, 21, None),
    "small_sparse": (small_cfg, 5 * 8 - 3, 22, [[0, 2], [1, 3, 4]]),
    "small_empty": (small_cfg, 5 * 8 - 3, 23, [[], [4, 0, 2]]),
    "c1_dense": (c1_cfg, 4 * 64, 31, None),
    "qwen_sparse": (qwen_slice_cfg, 8 * 128, 41, [[0, 3, 5], [1, 2], [7], [0, 4, 6, 7]]),
    "qwen_nopast": (qwen_slice_cfg, 0, 42, [[], [], [], []]),
    "qwen_partial": (qwen_slice_cfg, 8 * 128 - 37, 44, [[0, 3, 7], [1, 7], [7], [0, 4, 6]]),  # last past page partial
    "llama_sparse": (llama_slice_cfg, 6 * 256, 51, [[0, 3, 5], [1, 2, 4, 0]]),               # P 256, GQA 4
}


@pytest.mark.parametrize("name", list(ATTN_CASES))
def test_attention_fp32_parity(name):
    mk, past, seed, sel = ATTN_CASES[name]
    c = mk()
    case = attn_case(c, past, seed=seed, dtype=np.float32, selected=sel)
    got, _ = run_device(c, case, "fp32")
    want = run_oracle(c, case)
    assert got["page_table"].tolist() == want["page_table"].tolist()
    for k in ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v"):
        assert rel(got[k], want[k]) < FP32_TOL, (name, k, rel(got[k], want[k]))


@pytest.mark.parametrize("name", ["c1_dense", "qwen_sparse", "qwen_nopast", "small_sparse", "qwen_partial",
                                  "llama_sparse"])
@pytest.mark.parametrize("policy", ["auto", "simt"])
def test_attention_bf16_parity(name, policy):
    mk, past, seed, sel = ATTN_CASES[name]
    c = mk()
    case = bf16_case(attn_case(c, past, seed=seed, dtype=np.float32, selected=sel))
    got, _ = run_device(c, case, "bf16", policy)
    want = run_oracle(c, case)
    for k in ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v"):
        assert rel(got[k], want[k]) < BF16_TOL, (name, policy, k, rel(got[k], want[k]))


# tcgen05 path at head dim 64 and / or page size 64 (BASELINE configs[0]): the
# 128-wide tiles carry zeros past hd 64; a 128-row query tile covers two 64-token query pages whose
# lists are merged as 64-key half blocks (equal lists: every row; different lists: each page's rows).
def _hd64_p128():
    return Cfg(n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=64, chunk_size=256, page_size=128,
               retrieval_budget=256, local_window=4)


def _hd128_p64():
    return Cfg(n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=128, chunk_size=256, page_size=64,
               retrieval_budget=256, local_window=4)


TC_SMALL_CASES = {
    "c1_dense": (c1_cfg, 6 * 64, 61, None),
    "c1_nopast": (c1_cfg, 0, 62, [[], [], [], []]),
    "c1_distinct_lists": (c1_cfg, 7 * 64, 63, [[0, 3, 5], [1, 2], [5], [0, 4, 2, 1]]),  # odd half counts
    "c1_equal_pairs": (c1_cfg, 7 * 64, 64, [[0, 2, 4], [0, 2, 4], [1, 3, 6, 5], [1, 3, 6, 5]]),
    "c1_partial": (c1_cfg, 6 * 64 - 17, 65, [[0, 5], [5, 1], [2, 5, 3], [4]]),  # last past page partial
    "c1_one_side_empty": (c1_cfg, 5 * 64, 66, [[], [0, 1, 2], [4, 3], []]),
    "hd64_p128": (_hd64_p128, 5 * 128, 67, [[0, 3], [1, 4, 2]]),
    "hd128_p64": (_hd128_p64, 7 * 64, 68, [[0, 6], [1, 2, 3], [6, 5, 4], [0]]),
}


@pytest.mark.parametrize("name", list(TC_SMALL_CASES))
def test_tc_small_shapes_bf16_parity(name):
    """policy "tcgen05" raises ConfigError if the shape would fall back to SIMT: these run on tensor cores."""
    mk, past, seed, sel = TC_SMALL_CASES[name]
    c = mk()
    case = bf16_case(attn_case(c, past, seed=seed, dtype=np.float32, selected=sel))
    got, _ = run_device(c, case, "bf16", "tcgen05")
    want = run_oracle(c, case)
    for k in ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v"):
        assert rel(got[k], want[k]) < BF16_TOL, (name, k, rel(got[k], want[k]))


def test_tc_c1_multichunk_matches_simt():
    """A whole c1 layer (8K context, 32 chunks of 256, dense) through the public chunk loop on the
    tcgen05 policy tracks the SIMT policy's run (itself 1e-5 to the oracle in fp32 elsewhere)."""
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200 import attention as A
    cfg = ModelConfig(n_layers=1, n_q_heads=4, n_kv_heads=1, head_dim=64, chunk_size=256, page_size=64,
                      retrieval_budget=0, attention_mode=["dense"])
    g = torch.Generator(device="cuda").manual_seed(7)
    S = 32
    q = [torch.randn(256, 4, 64, device="cuda", generator=g).bfloat16() for _ in range(S)]
    k = [torch.randn(256, 1, 64, device="cuda", generator=g).bfloat16() for _ in range(S)]
    v = [torch.randn(256, 1, 64, device="cuda", generator=g).bfloat16() for _ in range(S)]
    do = [torch.randn(256, 4, 64, device="cuda", generator=g).bfloat16() for _ in range(S)]
    res = {}
    for policy in ("tcgen05", "simt"):
        cache = PagedCache(cfg, dtype="bf16", max_tokens=S * 256)
        cache.set_kernel_policy(policy)
        saved = []
        for i in range(S):
            sel = [list(range(4 * i))] * 4
            cache.append_chunk(0, k[i], v[i])
            saved.append(A.attn_forward(cfg, q[i], cache, 0, sel, k[i], v[i]))
        outs = [s.out.float() for s in saved]
        dqs, dks = [], []
        for i in reversed(range(S)):
            gr = A.attn_backward(cfg, do[i], q[i], cache, 0, k[i], v[i], saved[i])
            cache.accumulate_grad_pages(0, list(range(4 * i, 4 * i + 4)), gr.dk_cur, gr.dv_cur)
            dqs.append(gr.dq.clone())
            dks.append(torch.cat([gr.dk_cur, gr.dv_cur]))
        torch.cuda.synchronize()
        cache.check_device_errors()
        res[policy] = (torch.stack(outs), torch.stack(dqs), torch.stack(dks))
    for a, b in zip(res["tcgen05"], res["simt"]):
        assert rel(T(a), T(b)) < BF16_TOL


def test_tc_forward_dense_qwen_chunk():
    """Longer key lists (8 past pages x all 4 query pages) through the tcgen05 forward."""
    c = qwen_slice_cfg()
    case = bf16_case(attn_case(c, 16 * 128, seed=43, dtype=np.float32, selected=[list(range(16))] * 4))
    got, _ = run_device(c, case, "bf16", "tcgen05")
    want = run_oracle(c, case)
    assert rel(got["out"], want["out"]) < BF16_TOL
    assert rel(got["lse"], want["lse"]) < 1e-3


def test_forward_properties():
    """test_attention.cpp:164-247 on the device: causal mask, page-order invariance,
    bitwise replay, zero dO -> zero grads."""
    from paper_2602_02108_b200 import attention as A
    for dtype in ("fp32", "bf16"):
        c = qwen_slice_cfg() if dtype == "bf16" else small_cfg()
        case = attn_case(c, 4 * c.page_size, seed=61, dtype=np.float32)
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        cache = cache_for(c, dtype)
        dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", tdt)
        cache.append_chunk(0, dev(case["pk"]), dev(case["pv"]))
        q, kc, vc = dev(case["q"]), dev(case["kc"]), dev(case["vc"])
        m = c.chunk_size // c.page_size
        a = A.attn_forward(cache.cfg, q, cache, 0, [[0, 1, 2, 3]] * m, kc, vc)
        b = A.attn_forward(cache.cfg, q, cache, 0, [[2, 0, 3, 1]] * m, kc, vc)
        assert (a.out.float() - b.out.float()).abs().max().item() <= (1e-6 if dtype == "fp32" else 1e-2)
        r = A.attn_forward(cache.cfg, q, cache, 0, a.selected, kc, vc)
        assert torch.equal(a.out, r.out) and torch.equal(a.lse, r.lse)
        t_probe = 3
        k2, v2 = kc.clone(), vc.clone()
        k2[t_probe + 1:] += 7.5
        v2[t_probe + 1:] -= 2.5
        pert = A.attn_forward(cache.cfg, q, cache, 0, [[0, 1, 2, 3]] * m, k2, v2)
        assert torch.equal(pert.out[: t_probe + 1], a.out[: t_probe + 1])
        g = A.attn_backward(cache.cfg, torch.zeros_like(q), q, cache, 0, kc, vc, a)
        assert g.dq.abs().sum().item() == 0 and g.dk_cur.abs().sum().item() == 0 and g.dv_cur.abs().sum().item() == 0
        gp = cache.gather_grad_pages(0, [0, 1, 2, 3])
        assert gp.k.abs().sum().item() == 0 and gp.v.abs().sum().item() == 0
        cache.check_device_errors()


def test_sparse_degenerates_to_dense_bitwise():
    """k >= n selection runs the identical kernel path with identical lists as dense
    (test_chunk_trainer.cpp:166-185)."""
    from paper_2602_02108_b200 import attention as A
    c = qwen_slice_cfg()
    case = bf16_case(attn_case(c, 6 * 128, seed=71, dtype=np.float32))
    cache = cache_for(c, "bf16")
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16)
    cache.append_chunk(0, dev(case["pk"]), dev(case["pv"]))
    q = dev(case["q"])
    kc, vc = dev(case["kc"]), dev(case["vc"])
    dense = A.attn_forward(cache.cfg, q, cache, 0, [list(range(6))] * 4, kc, vc)
    vote = torch.rand(4, 6, device="cuda")
    sel = A.select_topk_rows(cache, vote, 64)
    assert sel.lists() == [list(range(6))] * 4
    sparse = A.attn_forward(cache.cfg, q, cache, 0, sel, kc, vc)
    assert torch.equal(dense.out, sparse.out) and torch.equal(dense.lse, sparse.lse)
