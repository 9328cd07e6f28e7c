"""Fused projection epilogue: RoPE at absolute positions fused into the page
append, and rope / rope_backward on the device, against a numpy restatement of ops.hpp:192-230
(angles and trig in double, the rotation in fp32 with no contraction)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def rope_np(x: np.ndarray, pos_offset: int, base: float = 10000.0, sign: int = 1) -> np.ndarray:
    """ops.hpp:192-225 line by line (Real = float32)."""
    t, h, d = x.shape
    inv = np.array([np.power(np.float64(np.float32(base)), -2.0 * i / d) for i in range(d // 2)])
    y = np.empty_like(x, dtype=np.float32)
    for r in range(t):
        pos = float(sign) * float(pos_offset + r)
        ang = pos * inv
        c = np.cos(ang).astype(np.float32)
        s = np.sin(ang).astype(np.float32)
        x0 = x[r, :, 0::2].astype(np.float32)
        x1 = x[r, :, 1::2].astype(np.float32)
        y[r, :, 0::2] = (x0 * c) - (x1 * s)
        y[r, :, 1::2] = (x0 * s) + (x1 * c)
    return y


@pytest.mark.parametrize("pos", [0, 4096, 1 << 20])
def test_rope_matches_reference_restatement(pos):
    from paper_2602_02108_b200.attention import rope
    g = torch.Generator().manual_seed(pos + 1)
    x = torch.randn(64, 4, 128, generator=g)
    got = rope(x.cuda(), pos).cpu().numpy()
    want = rope_np(x.numpy(), pos)
    # identical but for a rare 1-ulp difference of the device's double cos/sin before the fp32 rounding
    assert np.mean(got == want) > 0.999
    assert np.allclose(got, want, rtol=2e-6, atol=2e-6)
    back = rope(torch.from_numpy(got).cuda(), pos, sign=-1).cpu().numpy()
    assert np.allclose(back, x.numpy(), rtol=1e-5, atol=1e-5)   # rope_backward inverts the rotation


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_fused_rope_append_equals_rope_then_append(dtype):
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200.attention import rope
    tdt = torch.float32 if dtype == "fp32" else torch.bfloat16
    cfg = ModelConfig(n_layers=1, n_q_heads=28, n_kv_heads=4, head_dim=128, chunk_size=512, page_size=128,
                      retrieval_budget=256)
    g = torch.Generator(device="cuda").manual_seed(5)
    chunks = [(torch.randn(512, 4, 128, device="cuda", generator=g).to(tdt),
               torch.randn(512, 4, 128, device="cuda", generator=g).to(tdt)) for _ in range(3)]
    fused = PagedCache(cfg, dtype=dtype, max_tokens=4096)
    split = PagedCache(cfg, dtype=dtype, max_tokens=4096)
    for i, (k, v) in enumerate(chunks):
        fused.append_chunk(0, k, v, rope_base=10000.0)
        split.append_chunk(0, rope(k, i * 512), v)
    ids = list(range(12))
    a, b = fused.gather_pages(0, ids), split.gather_pages(0, ids)
    assert torch.equal(a.k, b.k) and torch.equal(a.v, b.v)
    assert torch.equal(fused.page_mean_keys(0), split.page_mean_keys(0))


@pytest.mark.parametrize("pos", [4096, 1 << 20])
def test_reverse_epilogue_equals_readback_then_rope_backward(pos):
    """oomb_accumulate_grad_pages_rope == accumulate_grad_pages followed by rope(sign -1) on dK,
    bitwise (chunk_trainer.hpp:575-592 in one pass)."""
    from paper_2602_02108_b200 import ModelConfig, PagedCache
    from paper_2602_02108_b200.attention import rope
    cfg = ModelConfig(n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=128, chunk_size=256, page_size=128,
                      retrieval_budget=256)
    g = torch.Generator(device="cuda").manual_seed(5)
    cache = PagedCache(cfg, dtype="bf16", max_tokens=1024)
    kv = torch.randn(512, 2, 128, device="cuda", generator=g).bfloat16()
    cache.append_chunk(0, kv, kv)
    n = 512 // 128
    dk_pages = torch.randn(n * 128, 2, 128, device="cuda", generator=g)
    cache.scatter_add_grads(0, list(range(n)), dk_pages, 2 * dk_pages)  # grads of the "own" pages
    own = [2, 3]
    dk = torch.randn(256, 2, 128, device="cuda", generator=g)
    dv = torch.randn(256, 2, 128, device="cuda", generator=g)
    a_k, a_v = dk.clone(), dv.clone()
    cache.accumulate_grad_pages(0, own, a_k, a_v)
    a_k = rope(a_k, pos, 10000.0, sign=-1)
    b_k, b_v = dk.clone(), dv.clone()
    cache.accumulate_grad_pages_rope(0, own, b_k, b_v, pos, 10000.0)
    torch.cuda.synchronize()
    assert torch.equal(a_k, b_k) and torch.equal(a_v, b_v)
