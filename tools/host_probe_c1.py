"""Is the c1 layer step host-bound? Host time to ISSUE each native phase (oomb_layer_step returns
before the GPU finishes) against the phase's GPU span (CUDA events), after warm-up."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2602_02108_b200.chunk_loop import layer_step

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"])
run = bench.Run(cfg, 0, torch.device("cuda:0"))
C = cfg["C"]
kv = (run.S, C, cfg["Hkv"], cfg["hd"])
args = (run.cache, 0, run.q_all, run.k_all.view(kv), run.v_all.view(kv), run.do_all, run.o_all, run.lse_all, run.grads)
comp = torch.cuda.current_stream()
for it in range(8):
    run.cache.reset()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    e[0].record(comp)
    t0 = time.perf_counter()
    layer_step(*args, mode=cfg["mode"], phase="forward")
    t1 = time.perf_counter()
    e[1].record(comp)
    t2 = time.perf_counter()
    layer_step(*args, mode=cfg["mode"], phase="backward")
    t3 = time.perf_counter()
    e[2].record(comp)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    if it >= 3:
        print(f"fwd issue {1e3*(t1-t0):.3f} ms gpu {e[0].elapsed_time(e[1]):.3f} | bwd issue {1e3*(t3-t2):.3f} ms "
              f"gpu {e[1].elapsed_time(e[2]):.3f} | wall {1e3*(t4-t0):.3f}")
