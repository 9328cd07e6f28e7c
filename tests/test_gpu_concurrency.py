"""Chunk-level concurrency the bench uses is bitwise invisible: consecutive chunks' forwards on two
streams, and the backward with deferred dQ joins (OOMB_ATTN_DEFER_DQ: chunk i-1's dK/dV runs
under chunk i's dQ, workspaces alternate) give the same outputs, gradients and gradient pages as
the plain sequential loop."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _layer(concurrent: bool, n_chunks=4, seed=7):
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200 import attention as A
    cfg = ModelConfig(n_layers=1, n_q_heads=28, n_kv_heads=4, head_dim=128, chunk_size=512, page_size=128,
                      retrieval_budget=3 * 128, attention_mode=["topk"])
    C, m = cfg.chunk_size, cfg.pages_per_chunk()
    cache = PagedCache(cfg, dtype="bf16", max_tokens=n_chunks * C)
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda h: [torch.randn(C, h, 128, device="cuda", generator=g).bfloat16() for _ in range(n_chunks)]
    qs, ks, vs, dos = r(28), r(4), r(4), r(28)
    comp = torch.cuda.current_stream()
    att = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs, sels = [], []
    for i in range(n_chunks):
        sel = A.select_pages_topk(cache, 0, qs[i], i * m) if i else A.Selection.from_lists(cache, [[]] * m)
        cache.append_chunk(0, ks[i], vs[i])
        st = comp
        if concurrent:
            st = att[i & 1]
            st.wait_stream(comp)
        outs.append(A.attn_forward(cfg, qs[i], cache, 0, sel, ks[i], vs[i], stream=st))
        sels.append(sel)
    for st in att:
        comp.wait_stream(st)
    grads = []
    for i in reversed(range(n_chunks)):
        gr = A.attn_backward(cfg, dos[i], qs[i], cache, 0, ks[i], vs[i], outs[i], defer_dq=concurrent)
        cache.accumulate_grad_pages(0, list(range(i * m, (i + 1) * m)), gr.dk_cur, gr.dv_cur)
        grads.append(gr)
    if concurrent:
        A.join_dq(cache)
    torch.cuda.synchronize()
    pages = cache.gather_grad_pages(0, list(range(n_chunks * m)))
    return ([(o.out.clone(), o.lse.clone()) for o in outs], [(x.dq, x.dk_cur, x.dv_cur) for x in grads],
            (pages.k.clone(), pages.v.clone()))


def test_concurrent_chunks_bitwise_equal_sequential():
    a_out, a_gr, a_pg = _layer(False)
    b_out, b_gr, b_pg = _layer(True)
    for (o1, l1), (o2, l2) in zip(a_out, b_out):
        assert torch.equal(o1, o2) and torch.equal(l1, l2)
    for x, y in zip(a_gr, b_gr):
        for u, w in zip(x, y):
            assert torch.equal(u, w)
    assert torch.equal(a_pg[0], b_pg[0]) and torch.equal(a_pg[1], b_pg[1])


def test_fp32_backward_replays_bitwise():
    """The fp32 parity path is deterministic too (SPEC determinism, SURVEY §8b threading): dQ is
    query-major and dK / dV key-major with one writer per element, summed in the reference's order,
    so two runs give the same bits for dq, dk_cur, dv_cur and the gradient pages."""
    import numpy as np
    from tests.test_gpu_parity import ATTN_CASES, attn_case, run_device
    mk, past, seed, sel = ATTN_CASES["small_sparse"]
    c = mk()
    case = attn_case(c, past, seed=seed, dtype=np.float32, selected=sel)
    a, _ = run_device(c, case, "fp32")
    b, _ = run_device(c, case, "fp32")
    for k in ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v"):
        assert np.array_equal(a[k], b[k]), k
