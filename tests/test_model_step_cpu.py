"""The whole-model chunked training step fixture (tests/golden/model_step.npz, made by the
reference's ChunkTrainer::train_step): its layout matches the device trainer's parameter order,
and, where the reference shim is built, re-running the reference reproduces it bitwise."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "model_step.npz")


def test_fixture_layout_matches_visit_order():
    from paper_2602_02108_b200.trainer import param_shapes
    from tests.golden.make_model_golden import model_cfg
    z = np.load(FIX)
    n = sum(int(np.prod(s)) for _, _, s in param_shapes(model_cfg()))
    assert z["params"].size == n
    for mode in ("dense", "topk", "local"):
        g = z[f"{mode}_grads_f32"]
        assert g.size == n and np.isfinite(g).all() and np.abs(g).max() > 0
        # f32 reference vs f64 reference: the fixture's own precision floor
        g64 = z[f"{mode}_grads_f64"]
        assert np.linalg.norm(g - g64) / np.linalg.norm(g64) < 1e-5
    # the reference's own chunked f64 step equals its exact non-chunked pass (test_chunk_trainer.cpp:54-90)
    assert np.linalg.norm(z["dense_grads_f64"] - z["full_grads_f64"]) / np.linalg.norm(z["full_grads_f64"]) < 1e-6
    cnt = z["topk_sel_counts"].reshape(5, 2, 4)  # chunks x layers x query pages
    assert (cnt[0] == 0).all() and (cnt[1] == 2).all() and (cnt[4] == 2).all()  # k = 16 / 8 = 2 pages


def test_fixture_reproduces_from_the_reference():
    from oracle.oracle import Ref, ref_init_params, ref_train_step
    from tests.golden.make_model_golden import model_cfg
    if not Ref.available():
        pytest.skip("reference shim not built (oracle/_ref)")
    z = np.load(FIX)
    assert np.array_equal(ref_init_params(model_cfg(), "dense", seed=7), z["params"])
    loss, g, cnt = ref_train_step(model_cfg("topk"), "topk", z["params"], z["tokens"])
    assert loss == float(z["topk_loss_f32"]) and np.array_equal(g, z["topk_grads_f32"])
    assert np.array_equal(cnt, z["topk_sel_counts"])
