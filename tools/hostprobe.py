import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import bench
cfg = bench.CONFIGS["c3"]
r = bench.Run(cfg, 0, torch.device("cuda:0"))
r.step(); torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); r.step(); th = time.perf_counter() - t0; e1.record(); torch.cuda.synchronize()
    print("host enqueue s", round(th, 3), "device s", round(e0.elapsed_time(e1) / 1e3, 3))
# per-phase host timing
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); r.step(); pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
