"""Offload regime at c3 with several physical slot slacks above the tier capacity (bench.offload_measure).
Usage: python tools/offload_slack_probe.py SLACK [SLACK...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

torch.cuda.set_device(0)
run = bench.Run(dict(bench.CONFIGS["c3"]), seed=1234, device=torch.device("cuda", 0))
run.step()
for sl in map(int, sys.argv[1:]):
    bench.OFFLOAD_SLACK = sl
    try:
        r = bench.offload_measure(run, 0.75, repeats=1)
        print(sl, json.dumps({k: v for k, v in r.items() if k != "note"}), flush=True)
    except Exception as e:  # noqa: BLE001
        print(sl, "error", repr(e), flush=True)
