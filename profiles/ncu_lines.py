"""Aggregate an ncu source page (--print-source sass,cuda --csv) by CUDA source
line: warp-stall samples and the dominant stall reasons. Usage:
  ncu -i X.ncu-rep --page source --csv --print-source sass,cuda > s.csv
  python profiles/ncu_lines.py s.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
agg = defaultdict(lambda: defaultdict(float))
src = {}
fname = "?"
hdr = None
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        line = (fname, r[0])
        src[line] = r[1]
    if line is None:
        continue
    for i, h in enumerate(hdr):
        if i < 4:
            continue
        if h in ("Warp Stall Sampling (All Samples)", "Instructions Executed") or (
                h.startswith("stall_") and "Not Issued" not in h):
            try:
                agg[line][h] += float(r[i] or 0)
            except ValueError:
                pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
itot = sum(v["Instructions Executed"] for v in agg.values())
print(f"total samples {tot:.0f}, warp-instructions {itot:.3g}")
if "--inst" in sys.argv:
    for ln, v in sorted(agg.items(), key=lambda kv: -kv[1]["Instructions Executed"])[:top]:
        i = v["Instructions Executed"]
        print(f"{i:11.0f} {100 * i / max(itot, 1):5.1f}% {ln[0]}:{ln[1]:<5} {src.get(ln, '')[:80]}")
    sys.exit(0)
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]:
    s = v["Warp Stall Sampling (All Samples)"]
    reasons = sorted(((k, x) for k, x in v.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:3]
    rs = " ".join(f"{k[6:]}={100 * x / max(s, 1):.0f}%" for k, x in reasons if x > 0)
    print(f"{s:7.0f} {100 * s / max(tot, 1):5.1f}% {ln[0]}:{ln[1]:<5} {src.get(ln, '')[:70]:<70} {rs}")
