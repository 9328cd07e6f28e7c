"""oomb_attn_backward_readback (the dM_i read-back of a chunk's own pages folded into its backward call) gives
bit for bit what attn_backward followed by accumulate_grad_pages of the chunk's own pages gives
(chunk_trainer.hpp:575-587): on the tcgen05 path (head dim 128 / page 128 and head dim 64 / page 64,
where one 128-key block spans two pages) and on the SIMT parity paths (fp32, fp64)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = {"bf16_hd128_p128": ("bf16", 128, 128), "bf16_hd64_p64": ("bf16", 64, 64), "fp32_hd128_p128": ("fp32", 128, 128),
         "fp64_hd64_p64": ("fp64", 64, 64)}


def _layer(dtype, hd, P, fused, n_chunks=4, seed=5):
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200 import attention as A
    C = 4 * P
    cfg = ModelConfig(n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=hd, chunk_size=C, page_size=P,
                      retrieval_budget=2 * P, attention_mode=["topk"])
    m = cfg.pages_per_chunk()
    cache = PagedCache(cfg, dtype=dtype, max_tokens=n_chunks * C)
    g = torch.Generator(device="cuda").manual_seed(seed)
    el = {"bf16": torch.bfloat16, "fp32": torch.float32, "fp64": torch.float64}[dtype]
    r = lambda h: [torch.randn(C, h, hd, device="cuda", generator=g).to(el) for _ in range(n_chunks)]
    qs, ks, vs, dos = r(8), r(2), r(2), r(8)
    outs = []
    for i in range(n_chunks):
        sel = A.select_pages_topk(cache, 0, qs[i], i * m) if i else A.Selection.from_lists(cache, [[]] * m)
        cache.append_chunk(0, ks[i], vs[i])
        outs.append(A.attn_forward(cfg, qs[i], cache, 0, sel, ks[i], vs[i]))
    grads = []
    for i in reversed(range(n_chunks)):
        gr = A.attn_backward(cfg, dos[i], qs[i], cache, 0, ks[i], vs[i], outs[i],
                             own_first_page=i * m if fused else None)
        if not fused:
            cache.accumulate_grad_pages(0, list(range(i * m, (i + 1) * m)), gr.dk_cur, gr.dv_cur)
        grads.append([x.clone() for x in (gr.dq, gr.dk_cur, gr.dv_cur)])
    torch.cuda.synchronize()
    cache.check_device_errors()
    return grads


@pytest.mark.parametrize("name", sorted(CASES))
def test_readback_flag_bitwise(name):
    dtype, hd, P = CASES[name]
    a = _layer(dtype, hd, P, False)
    b = _layer(dtype, hd, P, True)
    for i, (x, y) in enumerate(zip(a, b)):
        for u, w, what in zip(x, y, ("dq", "dk_cur", "dv_cur")):
            assert torch.equal(u, w), (name, i, what)
    # the read-back really added something (later chunks selected earlier chunks' pages)
    assert any(not torch.equal(x[1], y[1]) for x, y in zip(a[1:], a[:-1]))


def test_readback_needs_whole_appended_pages():
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200 import attention as A
    from paper_2602_02108_b200.errors import ShapeError
    cfg = ModelConfig(n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=128, chunk_size=512, page_size=128,
                      retrieval_budget=256, attention_mode=["dense"])
    cache = PagedCache(cfg, dtype="bf16", max_tokens=2048)
    for c in (200, 256):
        q = torch.randn(c, 8, 128, device="cuda").bfloat16()
        k = torch.randn(c, 2, 128, device="cuda").bfloat16()
        sel = A.Selection.from_lists(cache, [[]] * ((c + 127) // 128))
        cache.append_chunk(0, k, k)
        o = A.attn_forward(cfg, q, cache, 0, sel, k, k)
        with pytest.raises(ShapeError):  # 200 keys: not whole pages; 256: pages 3, 4 are not appended
            A.attn_backward(cfg, q, q, cache, 0, k, k, o, own_first_page=0 if c == 200 else 3)
