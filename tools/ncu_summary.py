"""Summarise an ncu report into profiles/: the details page as text and a
record in profiles/ncu_summary.json (read by bench.py for roofline.traffic).
    python tools/ncu_summary.py <rep> <key> <profiles/name.txt> "<description>"
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key, out_txt, desc = sys.argv[1:5]
repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--print-details", "all"],
                     capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
m = dict(zip(h, v))
u = dict(zip(h, units))


def num(k):
    x = float(m[k].replace(",", ""))
    unit = u.get(k, "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "ns": 1e-6,
             "usecond": 1e-3, "us": 1e-3, "msecond": 1, "ms": 1, "second": 1e3, "s": 1e3}[unit]
    return x * scale


stalls = {}
for k in h:
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(m[k])
        except ValueError:
            pass
top = dict(sorted(stalls.items(), key=lambda x: -x[1])[:6])
rec = {
    "kernel": m.get("Kernel Name"), "grid": m.get("Grid Size"), "block": m.get("Block Size"),
    "source": f"{out_txt} ({desc})",
    "duration_ms": num("gpu__time_duration.sum"),
    "dram_bytes_read": num("dram__bytes_read.sum"),
    "dram_bytes_write": num("dram__bytes_write.sum"),
    "l2_hit_rate_pct": float(m.get("lts__t_sector_hit_rate.pct", "nan")),
    "issue_active_pct": float(m.get("sm__inst_issued.avg.pct_of_peak_sustained_active", "nan")),
    "inst_executed": float(m.get("smsp__inst_executed.sum", "nan").replace(",", "")),
    "top_stalls": top,
}
rec["dram_bytes_per_launch"] = rec["dram_bytes_read"] + rec["dram_bytes_write"]
rec["dram_gbs"] = rec["dram_bytes_per_launch"] / (rec["duration_ms"] * 1e-3) / 1e9
try:
    peak = float(json.load(open(os.path.join(repo, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    peak = 6650.0
rec["dram_frac_of_peak"] = rec["dram_gbs"] / peak
with open(os.path.join(repo, out_txt), "w") as fh:
    fh.write(txt)
p = os.path.join(repo, "profiles", "ncu_summary.json")
d = json.load(open(p)) if os.path.exists(p) else {}
d[key] = rec
json.dump(d, open(p, "w"), indent=1)
print(key, json.dumps(rec)[:400])
