"""Host topology of the GPU box and pinned-copy bandwidth with the process bound to each NUMA node."""
import os, subprocess, sys, time
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:1500])
nodes = sorted(int(d[4:]) for d in os.listdir("/sys/devices/system/node") if d.startswith("node") and d[4:].isdigit())
print("numa nodes", nodes, "cpus", os.cpu_count())
import torch
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
try:
    out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    bid = out.split("\n")[0].lower()
    bid = bid[4:] if bid.count(":") == 2 and len(bid.split(":")[0]) == 8 else bid
    for cand in (bid, bid.replace("00000000:", "0000:")):
        path = f"/sys/bus/pci/devices/{cand}/numa_node"
        if os.path.exists(path):
            print("gpu", cand, "numa_node", open(path).read().strip())
except Exception as e:
    print("bus id lookup failed", e)
for nd in nodes:
    cpus = open(f"/sys/devices/system/node/node{nd}/cpulist").read().strip()
    print("node", nd, "cpus", cpus)
n = 256 << 20
for nd in nodes:
    cpus = set()
    for part in open(f"/sys/devices/system/node/node{nd}/cpulist").read().strip().split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    h1.fill_(1); h2.fill_(1)
    g1 = torch.empty(n, dtype=torch.uint8, device="cuda"); g2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    def run(a, b, reps=8):
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(reps):
            if a:
                with torch.cuda.stream(s1): g1.copy_(h1, non_blocking=True)
            if b:
                with torch.cuda.stream(s2): h2.copy_(g2, non_blocking=True)
        torch.cuda.synchronize(); return reps * n / (time.perf_counter() - t) / 1e9
    run(True, True, 2)
    print(f"bound to node {nd}: H2D {run(True, False):.1f}  D2H {run(False, True):.1f}  both {run(True, True):.1f} GB/s")
    del h1, h2
