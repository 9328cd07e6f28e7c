"""Golden fixture for the whole-model chunked training step, FROM THE
REFERENCE: chunktrain::ChunkTrainer<float/double>::train_step through oracle/_ref (the
unmodified reference headers compiled in place).

    make -f oracle/Makefile.ref && python tests/golden/make_model_golden.py

Writes model_step.npz: the configuration, init_params(seed) flattened in ModelParams::visit
order, a token window, and per attention mode (dense / topk / local) the f32 and f64 loss and
parameter gradients plus the selected-page counts, and full_forward_backward (oracle.hpp:89-276,
the exact non-chunked pass) in f64 as the ground truth of the dense step.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import (ref_full_forward_backward, ref_init_params, ref_train_step,  # noqa: E402
                           ref_train_step_offload)
from paper_2602_02108_b200.config import ModelConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
OFFLOAD_CAPACITY = 20  # device pages (both layers) of the offload variant


def model_cfg(mode: str = "dense") -> ModelConfig:
    """Small model at the reference's test scale: 2 layers, 4Q/2KV heads of 8, P 8, C 32."""
    return ModelConfig(n_layers=2, d_model=32, n_q_heads=4, n_kv_heads=2, head_dim=8, d_ff=64, vocab_size=48,
                       chunk_size=32, page_size=8, attention_mode=[mode], retrieval_budget=16, local_window=2,
                       rope_base=10000.0, seed=7)


def main():
    rng = np.random.default_rng(11)
    tokens = rng.integers(0, 48, size=150).astype(np.int32)  # 5 chunks, the last one partial
    params = ref_init_params(model_cfg(), "dense", seed=7, real_bytes=4)
    out = {"tokens": tokens, "params": params}
    for mode in ("dense", "topk", "local"):
        mc = model_cfg(mode)
        l32, g32, cnt = ref_train_step(mc, mode, params, tokens)
        l64, g64, _ = ref_train_step(mc, mode, params.astype(np.float64), tokens)
        out[f"{mode}_loss_f32"] = np.float64(l32)
        out[f"{mode}_grads_f32"] = g32
        out[f"{mode}_loss_f64"] = np.float64(l64)
        out[f"{mode}_grads_f64"] = g64.astype(np.float32)
        out[f"{mode}_sel_counts"] = cnt
        # the same step with the TieredEngine protocol at OFFLOAD_CAPACITY device pages: the
        # ScheduleLog's (kind, layer, page, chunk, phase, bytes) sequence and the (unchanged) gradients
        lo, go, ev, _ = ref_train_step_offload(mc, mode, params, tokens, OFFLOAD_CAPACITY)
        assert lo == l32 and np.array_equal(go, g32)
        out[f"{mode}_offload_events"] = ev
        print(mode, "loss f32", l32, "f64", l64, "grad rel (f32 vs f64)",
              float(np.linalg.norm(g32 - g64) / np.linalg.norm(g64)))
    # the exact non-chunked pass in f64: ground truth for the dense chunked step (acceptance criterion 1)
    lf, gf = ref_full_forward_backward(model_cfg("dense"), params.astype(np.float64), tokens)
    out["full_loss_f64"] = np.float64(lf)
    out["full_grads_f64"] = gf.astype(np.float32)
    print("full f64 loss", lf, "dense chunked f64 vs full f64 grad rel",
          float(np.linalg.norm(out["dense_grads_f64"] - gf) / np.linalg.norm(gf)))
    np.savez_compressed(os.path.join(OUT, "model_step.npz"), **out)


if __name__ == "__main__":
    main()
