"""Error behaviour of the device path against the reference's error taxonomy.

The reference raises ShapeError for a page id outside the layer's pages (paged_kv.hpp
gather_pages / check range), for a selection with the wrong number of query-page lists
(attention.hpp:117-208, "selected.size() != m") and for a negative top-k budget
(attention.hpp:73). The backward, and the forward under residency enforcement, read the
selection on the host and raise at the call. The plain forward does not sync the selection to
the host: its kernels skip a bad id, raise a sticky flag, and `check_device_errors()` turns the
flag into the same ShapeError (and clears it). These tests pin that the skip leaves the rest of
the result intact and that each error class matches the reference's.
"""
import numpy as np
import pytest
import torch

from tests.golden.make_golden import attn_case, c1_cfg, qwen_slice_cfg
from tests.test_gpu_parity import T, cache_for

pytestmark = pytest.mark.gpu


def _forward(c, case, dtype, policy, selected, enforce=False):
    from paper_2602_02108_b200 import attention as A
    cache = cache_for(c, dtype)
    cache.set_kernel_policy(policy)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", tdt)
    cache.append_chunk(0, dev(case["pk"]), dev(case["pv"]))
    q, kc, vc, do = dev(case["q"]), dev(case["kc"]), dev(case["vc"]), dev(case["do"])
    cache.append_chunk(0, kc, vc)
    cache.set_residency_enforced(enforce)
    saved = A.attn_forward(cache.cfg, q, cache, 0, selected, kc, vc)
    torch.cuda.synchronize()
    return cache, saved, (q, kc, vc, do)


@pytest.mark.parametrize("dtype,policy,cfg", [("fp32", "simt", c1_cfg), ("bf16", "simt", c1_cfg),
                                              ("bf16", "tcgen05", qwen_slice_cfg)])
def test_bad_page_id_in_a_selection(dtype, policy, cfg):
    """Forward without enforcement: the kernel skips the id and flags it (no host sync on the
    hot path); with enforcement, and always in the backward (which reads the ids on the host to
    allocate gradient pages), the call itself raises ShapeError like the reference's gather."""
    from paper_2602_02108_b200 import ShapeError
    from paper_2602_02108_b200 import attention as A
    c = cfg()
    n_past = 6
    case = attn_case(c, n_past * c.page_size, seed=41, dtype=np.float32)
    m = c.chunk_size // c.page_size
    clean = [[0, 2, 5] for _ in range(m)]
    cache, s0, _ = _forward(c, case, dtype, policy, clean)
    cache.check_device_errors()
    n_total = cache.n_pages(0)  # past pages + the chunk's own pages
    # one id just past the layer's last page (still inside the pool's table) and one past the
    # table itself; two extra blocks keep every later block's warpgroup parity, so the surviving
    # pages are reduced in the same order and the result is bitwise that of the clean selection
    bad = [ids + [n_total + qp, 10 ** 6] for qp, ids in enumerate(clean)]
    cache2, s1, (q, kc, vc, do) = _forward(c, case, dtype, policy, bad)
    with pytest.raises(ShapeError):
        cache2.check_device_errors()
    cache2.check_device_errors()  # the flag is cleared once reported
    np.testing.assert_array_equal(T(s0.out), T(s1.out))
    np.testing.assert_array_equal(T(s0.lse), T(s1.lse))
    with pytest.raises(ShapeError, match="attn_backward"):
        A.attn_backward(cache2.cfg, do, q, cache2, 0, kc, vc, s1)
    with pytest.raises(ShapeError):
        _forward(c, case, dtype, policy, bad, enforce=True)
    cache2.check_device_errors()


def test_host_side_shape_errors():
    from paper_2602_02108_b200 import ShapeError
    from paper_2602_02108_b200 import attention as A
    c = c1_cfg()
    case = attn_case(c, 2 * c.page_size, seed=3, dtype=np.float32)
    cache = cache_for(c, "fp32")
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.float32)
    cache.append_chunk(0, dev(case["pk"]), dev(case["pv"]))
    q, kc, vc = dev(case["q"]), dev(case["kc"]), dev(case["vc"])
    m = c.chunk_size // c.page_size
    with pytest.raises(ShapeError):  # one list per query page (attention.hpp "selected.size() != m")
        A.attn_forward(cache.cfg, q, cache, 0, [[0]] * (m - 1), kc, vc)
    with pytest.raises(ShapeError):  # negative budget (attention.hpp:73)
        A.select_topk([1.0, 2.0], -1)
    with pytest.raises(ShapeError):  # layer out of range
        cache.gather_pages(5, [0])
    with pytest.raises(ShapeError):  # page out of range on the host-side gather
        cache.gather_pages(0, [7])
    cache.check_device_errors()
