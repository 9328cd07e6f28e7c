"""bench.py --impl reference (the reference arm) on CPU: it times the reference's own CPU path
(oracle/_ref, else the port) and needs no GPU, so its JSON contract and its torchrun behaviour
(rank 0 alone runs and prints; other ranks exit 0 without work) are checked here."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0", "--cpu-workers", "2"]


def _lines(out: str):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def test_reference_arm_line_on_cpu():
    r = subprocess.run([sys.executable, "bench.py", *ARGS], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s" and d["higher_is_better"]
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("reference", "port") and cb["cores"] == 2 and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("c1")


def test_reference_arm_under_torchrun_world2():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2", *ARGS],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)  # one line: rank 0's
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
