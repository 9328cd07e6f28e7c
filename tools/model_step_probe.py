import numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2602_02108_b200.trainer import ChunkTrainer, flatten, unflatten
from tests.golden.make_model_golden import model_cfg
z = np.load("tests/golden/model_step.npz")
for mode in ("dense", "topk", "local"):
    cfg = model_cfg(mode)
    tr = ChunkTrainer(cfg, max_tokens=len(z["tokens"]) + cfg.chunk_size, dtype="fp32")
    p = unflatten(z["params"], cfg, tr.dev)
    m, g = tr.train_step(p, z["tokens"])
    gf = flatten(g, cfg).cpu().numpy()
    r32 = np.linalg.norm(gf - z[f"{mode}_grads_f32"]) / np.linalg.norm(z[f"{mode}_grads_f32"])
    r64 = np.linalg.norm(gf - z[f"{mode}_grads_f64"]) / np.linalg.norm(z[f"{mode}_grads_f64"])
    print(mode, "loss", m.loss, "ref f32", float(z[f"{mode}_loss_f32"]), "grad rel vs ref f32 %.2e vs ref f64 %.2e" % (r32, r64))
