"""Seeded randomized parity sweep: random geometries (page size, chunk, GQA group, head dim),
history lengths (incl. a partial last page and no history), and random selections (empty lists,
arbitrary order) through append -> attn_forward -> attn_backward, against the C oracle.
fp32 mode (SIMT kernels): 1e-5; bf16 on the tcgen05 shape (hd 128, P 128): 2e-2."""
import numpy as np
import pytest

from oracle.oracle import Cfg
from tests.test_gpu_parity import BF16_TOL, FP32_TOL, attn_case, bf16_case, rel, run_device, run_oracle

pytestmark = pytest.mark.gpu


def random_case(seed: int, tc: bool):
    rng = np.random.default_rng(1000 + seed)
    if tc:
        P, hd = 128, 128
        m = int(rng.integers(1, 5))
        hkv = int(rng.choice([1, 2, 4]))
        g = int(rng.integers(1, 8))
    else:
        P = int(rng.choice([4, 8, 16]))
        hd = int(rng.choice([8, 16, 32]))
        m = int(rng.integers(1, 5))
        hkv = int(rng.choice([1, 2]))
        g = int(rng.integers(1, 4))
    C = P * m
    full = int(rng.integers(0, 7))
    past = full * P - (int(rng.integers(0, P)) if full and rng.random() < 0.4 else 0)  # partial last page
    n_past = (past + P - 1) // P
    sel = []
    for _ in range(m):
        k = int(rng.integers(0, n_past + 1))
        ids = rng.permutation(n_past)[:k].tolist()
        if rng.random() < 0.5:
            ids.sort()
        sel.append(ids)
    c = Cfg(n_layers=1, n_q_heads=hkv * g, n_kv_heads=hkv, head_dim=hd, chunk_size=C, page_size=P,
            retrieval_budget=P, local_window=1)
    return c, past, sel


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_fp32(seed):
    c, past, sel = random_case(seed, tc=False)
    case = attn_case(c, past, seed=seed, dtype=np.float32, selected=sel)
    got, _ = run_device(c, case, "fp32")
    want = run_oracle(c, case)
    assert got["page_table"].tolist() == want["page_table"].tolist()
    for k in ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v"):
        assert rel(got[k], want[k]) < FP32_TOL, (c, past, sel, k, rel(got[k], want[k]))


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_bf16_tcgen05(seed):
    c, past, sel = random_case(seed, tc=True)
    case = bf16_case(attn_case(c, past, seed=seed, dtype=np.float32, selected=sel))
    got, _ = run_device(c, case, "bf16", "tcgen05")
    want = run_oracle(c, case)
    for k in ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v"):
        if np.linalg.norm(want[k]) == 0:  # e.g. no history: no gradient pages
            assert not np.any(got[k]), k
            continue
        assert rel(got[k], want[k]) < BF16_TOL, (c, past, sel, k, rel(got[k], want[k]))
