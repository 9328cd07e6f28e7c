"""Bitwise comparison of a library variant against the in-tree build on one c3-shaped layer step
(usage on the box: python tools/variant_bitwise.py save <file> | compare <file>)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[3] if len(sys.argv) > 3 else "c3"])
if cfg["T"] > 32 * 4096:
    cfg["T"] = 32 * 4096
run = bench.Run(cfg, seed=77, device=torch.device("cuda", 0))
run.step()
torch.cuda.synchronize()
run.cache.check_device_errors()
n = run.cache.n_pages(0)
gp = run.cache.gather_grad_pages(0, list(range(n)))
res = {"out": run.o_all, "lse": run.lse_all, "dq": run.grads.dq, "dk": run.grads.dk_cur, "dv": run.grads.dv_cur,
       "gk": gp.k, "gv": gp.v}
if sys.argv[1] == "save":
    torch.save({k: v.cpu() for k, v in res.items()}, sys.argv[2])
    print("saved")
else:
    ref = torch.load(sys.argv[2])
    bad = [k for k in res if not torch.equal(res[k].cpu(), ref[k])]
    print("bitwise equal" if not bad else f"DIFFER: {bad}")
