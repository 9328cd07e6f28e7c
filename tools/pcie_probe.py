"""Pinned host <-> device copy bandwidth on the box: H2D alone, D2H alone, both at once."""
import torch, time
d = torch.device("cuda:0")
n = 256 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
g1 = torch.empty(n, dtype=torch.uint8, device=d); g2 = torch.empty(n, dtype=torch.uint8, device=d)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=10):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): g1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h2.copy_(g2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return reps * n / dt / 1e9
run(True, True, 2)
print("H2D GB/s", round(run(True, False), 1), " D2H GB/s", round(run(False, True), 1), " both (each) GB/s", round(run(True, True), 1))
