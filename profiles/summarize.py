"""Summarise a profile run (profiles/run_profile.sh TAG) into profiles/:
TAG_launches.md (per-kernel share of the step from the ncu launch list) and
TAG_ncu.md (key --set full metrics of the fused and merge kernels), and
update profiles/ncu_traffic.json (DRAM bytes per launch of the fused kernel,
read by bench.py as roofline.traffic).
  python profiles/summarize.py TAG WORKLOAD"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

TAG, WL = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "beam")
G = "gpurun_out"
P = os.path.dirname(os.path.abspath(__file__))

# ---- launch list
rows = [r for r in csv.reader(open(f"{G}/{TAG}_launches.csv")) if r and not r[0].startswith("==")]
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(list)
for r in rows[1:]:
    name = r[ik].split("(")[0].replace("void ", "")
    agg[name].append(float(r[iv].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
with open(f"{P}/{TAG}_launches.md", "w") as f:
    f.write(f"# {TAG}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
    f.write("Cold-cache, serialised per-launch times: compare SHARES, not absolutes.\n\n")
    f.write("| kernel | launches | mean us | share |\n|---|---|---|---|\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {100 * sum(v) / tot:.1f}% |\n")

# ---- full captures
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
out = {}
md = [f"# {TAG}: ncu --set full (workload {WL})\n"]
for part in ["fused", "merge"]:
    rep = f"{G}/{TAG}_{part}.ncu-rep"
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units, vals = rr[0], rr[1], rr[2]
    d = {}
    md.append(f"\n## {part}: {vals[h.index('Kernel Name')] if 'Kernel Name' in h else ''}\n\n"
              "| metric | value | unit |\n|---|---|---|\n")
    for m in want:
        if m in h:
            i = h.index(m)
            d[m] = (vals[i], units[i])
            md.append(f"| {m} | {vals[i]} | {units[i]} |\n")
    out[part] = d
open(f"{P}/{TAG}_ncu.md", "w").write("".join(md))

def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return float(v.replace(",", "")) * scale

if "fused" in out:
    f = out["fused"]
    tb = to_bytes(*f["dram__bytes_read.sum"]) + to_bytes(*f["dram__bytes_write.sum"])
    path = f"{P}/ncu_traffic.json"
    j = json.load(open(path)) if os.path.exists(path) else {}
    j[WL] = tb
    j[f"{WL}_source"] = f"profiles/{TAG}_ncu.md (ncu --set full, fused kernel, one launch)"
    json.dump(j, open(path, "w"), indent=1)
print(open(f"{P}/{TAG}_launches.md").read())
print("".join(md))
