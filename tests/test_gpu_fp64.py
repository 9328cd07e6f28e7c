"""fp64 pools (OOMB_F64, the reference's Real = double) on the B200 against the reference's own f64
outputs and the f64 oracle.

* The golden fixtures attn_small_f64.npz were produced by the reference itself (oracle/_ref,
  PagedCache<double> / attn_forward / attn_backward at the reference test geometry,
  test_attention.cpp:19-31): every output of the device path — out, lse, dq, dk_cur, dv_cur,
  the scattered gradient pages — within 1e-12 relative L2, page tables bit-exact.
* The f64 oracle on larger geometries (Qwen / Llama slices, sparse, partial pages): 1e-10
  (the reference's own f64 bar, test_attention.cpp:249-298).
* Scoring and top-k in double: votes within 1e-12 of the oracle, ids bit-exact.
"""
import os

import numpy as np
import pytest
import torch

from oracle.oracle import Port, det_normal
from tests.golden.make_golden import attn_case, llama_slice_cfg, qwen_slice_cfg, run_attn, small_cfg
from tests.test_gpu_parity import cache_for, model_cfg, rel

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
F64_TOL = 1e-10


def D(x):
    return x.detach().cpu().numpy()


def run_f64(c, case):
    from paper_2602_02108_b200 import attention as A
    cache = cache_for(c, "fp64")
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to("cuda")
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
    assert saved.lse.dtype == grads.dq.dtype == gp.k.dtype == torch.float64
    return dict(out=D(saved.out), lse=D(saved.lse), dq=D(grads.dq), dk_cur=D(grads.dk_cur), dv_cur=D(grads.dv_cur),
                grad_k=D(gp.k), grad_v=D(gp.v), page_table=cache.page_table(0))


@pytest.mark.parametrize("name", ["dense", "sparse", "empty_first"])
def test_fp64_matches_reference_golden(name):
    g = np.load(os.path.join(G, "attn_small_f64.npz"))
    cfg = small_cfg()
    off, ids = g[f"{name}/sel_off"], g[f"{name}/sel_ids"]
    sel = [ids[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1)]
    case = attn_case(cfg, 5 * cfg.page_size - 3, seed=21 + 8, dtype=np.float64,
                     selected=None if name == "dense" else sel)
    got = run_f64(cfg, case)
    assert got["page_table"].tolist() == g[f"{name}/page_table"].tolist()
    for k in ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v"):
        assert rel(got[k], g[f"{name}/{k}"]) < 1e-12, (name, k, rel(got[k], g[f"{name}/{k}"]))


CASES = {
    "qwen_sparse": (qwen_slice_cfg, 8 * 128, 41, [[0, 3, 5], [1, 2], [7], [0, 4, 6, 7]]),
    "qwen_partial": (qwen_slice_cfg, 8 * 128 - 37, 44, [[0, 3, 7], [1, 7], [7], [0, 4, 6]]),
    "llama_sparse": (llama_slice_cfg, 6 * 256, 51, [[0, 3, 5], [1, 2, 4, 0]]),
}


@pytest.mark.parametrize("name", list(CASES))
def test_fp64_matches_oracle(name):
    mk, past, seed, sel = CASES[name]
    c = mk()
    case = attn_case(c, past, seed=seed, dtype=np.float64, selected=sel)
    got = run_f64(c, case)
    want = run_attn(Port(c, 8), c, case)
    assert got["page_table"].tolist() == want["page_table"].tolist()
    for k in ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v"):
        assert rel(got[k], want[k]) < F64_TOL, (name, k, rel(got[k], want[k]))


def test_fp64_scoring_and_topk():
    from paper_2602_02108_b200 import attention as A
    c = qwen_slice_cfg()
    n_pages, tokens = 24, c.chunk_size
    dirs = det_normal(71, (n_pages, c.n_kv_heads, c.head_dim), np.float64)
    pk = det_normal(72, (n_pages * c.page_size, c.n_kv_heads, c.head_dim), np.float64) + \
        np.repeat(dirs, c.page_size, axis=0)
    q = det_normal(73, (tokens, c.n_q_heads, c.head_dim), np.float64)
    cache = cache_for(c, "fp64")
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda")
    cache.append_chunk(0, dev(pk), dev(pk))
    sel = A.select_pages_topk(cache, 0, dev(q), n_pages)
    port = Port(c, 8)
    port.append(0, pk, pk)
    want = port.score_pages(q, port.mean_keys(0, n_pages))
    assert sel.vote.dtype == torch.float64
    assert rel(D(sel.vote), want) < 1e-12
    k = c.retrieval_budget // c.page_size
    assert sel.lists() == [Port.select_topk(want[i], k).tolist() for i in range(want.shape[0])]
    # the host select_topk compares in double, like the reference (ties to the lower id)
    assert A.select_topk([5.0, 5.0, 1.0], 1) == [0]
    assert A.select_topk([1.0 + 1e-12, 1.0, 1.0 + 2e-12], 2) == [0, 2]
