"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
by CUDA source line: instructions executed, stall samples, top stall reasons.
usage: python tools/src_hot2.py file.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, hdr = None, None
agg = defaultdict(lambda: defaultdict(float))
text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].strip():
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    key = (fname, ln)
    text[key] = r[1].strip()[:80]
    for k, v in zip(hdr[4:], r[4:]):
        try:
            agg[key][k] += float(v)
        except ValueError:
            pass
ti = sum(a["Instructions Executed"] for a in agg.values())
ts = sum(a["Warp Stall Sampling (All Samples)"] for a in agg.values())
print(f"total warp instructions {ti:.4g}, stall samples {ts:.0f}")
tot = defaultdict(float)
for a in agg.values():
    for k, v in a.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            tot[k] += v
print("stall breakdown:", ", ".join(f"{k[6:]} {v / ts * 100:.1f}%" for k, v in
                                    sorted(tot.items(), key=lambda kv: -kv[1])[:9]))
for title, key in (("by stall samples", "Warp Stall Sampling (All Samples)"),
                   ("by instructions", "Instructions Executed")):
    print("---", title)
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        st = sorted(((n[6:], v) for n, v in a.items() if n.startswith("stall_") and
                     "Not Issued" not in n), key=lambda kv: -kv[1])[:2]
        s = a["Warp Stall Sampling (All Samples)"]
        print(f"{a['Instructions Executed'] / ti * 100:5.1f}%i {s / ts * 100:5.1f}%s "
              f"{k[0]}:{k[1]:<5} {text[k][:60]:60s} "
              + " ".join(f"{n}:{v / max(s, 1) * 100:.0f}%" for n, v in st))
