"""Per-kernel DRAM traffic and duration from ncu --set full reports -> JSON (bench.py's roofline.traffic).
Usage: python tools/ncu_traffic.py OUT.json "source description" name=rep.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

out, source, pairs = sys.argv[1], sys.argv[2], sys.argv[3:]
res = {"source": source}
for pr in pairs:
    name, rep = pr.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    get = lambda k: float(v[h.index(k)].replace(",", ""))
    unit = u[h.index("gpu__time_duration.sum")]
    dur = get("gpu__time_duration.sum") * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1.0)
    bunit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = get("dram__bytes_read.sum") * bunit.get(u[h.index("dram__bytes_read.sum")], 1)
    wr = get("dram__bytes_write.sum") * bunit.get(u[h.index("dram__bytes_write.sum")], 1)
    res[name] = {"dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "duration_us": dur,
                 "tensor_active_pct": get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
                 if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active" in h else None,
                 "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active")
                 if "smsp__issue_active.avg.pct_of_peak_sustained_active" in h else None,
                 "sm_active_pct": 100.0 * get("sm__cycles_active.avg") / get("sm__cycles_elapsed.avg")}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
