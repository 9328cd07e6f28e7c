"""oomb_layer_step (the native layer loop) is the Python chunk loop, bitwise.

bench.Run.step runs the unsplit layer through chunk_loop.layer_step (one C call per phase); the
host loop (forward_pass + bwd_chunk, the call sequence AttentionChunkLoop follows) is the
reference for it here. Both run on the same bench inputs: every chunk's out / lse, the last
chunk's dq / dk_cur / dv_cur and the whole gradient pool must match bit for bit, for top-k (c3
shape, 16 chunks), dense (c2 shape, 8 chunks) and the c1 geometry (tcgen05 head dim 64 / page 64,
split-K).
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = {"c3_16chunks": ("c3", 16 * 4096), "c2_8chunks": ("c2", 8 * 4096), "c1": ("c1", None)}


@pytest.mark.parametrize("name", sorted(CASES))
def test_native_loop_bitwise(name):
    import bench
    cfg_name, tokens = CASES[name]
    cfg = dict(bench.CONFIGS[cfg_name])
    if tokens:
        cfg["T"] = tokens
    run = bench.Run(cfg, seed=1234, device=torch.device("cuda", 0))
    res = {}
    for native in (False, True):
        bench.NATIVE_LOOP = native
        run.step()
        torch.cuda.synchronize()
        run.cache.check_device_errors()
        n = run.cache.n_pages(0)
        gp = run.cache.gather_grad_pages(0, list(range(n)))
        res[native] = [run.o_all.clone(), run.lse_all.clone(), run.grads.dq.clone(), run.grads.dk_cur.clone(),
                       run.grads.dv_cur.clone(), gp.k.clone(), gp.v.clone()]
    bench.NATIVE_LOOP = True
    for a, b, what in zip(res[False], res[True], ("out", "lse", "dq", "dk_cur", "dv_cur", "grad_k", "grad_v")):
        assert torch.equal(a, b), (name, what)
