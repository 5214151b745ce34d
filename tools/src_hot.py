"""Aggregate an ncu 'cuda,sass' source-page CSV by source line: warp-instructions
executed and stall samples.  usage: src_hot.py file.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None; hdr = None
agg = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] == "Function Name" or hdr is None: continue
    if r[0] != "":
        ln = (fname, int(r[0]), r[1].strip()[:70])
        d = dict(zip(hdr[2:], r[2:]))
        def num(k):
            v = d.get(k, "0")
            try: return float(v)
            except: return 0.0
        agg[ln] = (num("Instructions Executed"), num("Warp Stall Sampling (All Samples)"))
tot_i = sum(v[0] for v in agg.values()); tot_s = sum(v[1] for v in agg.values())
print(f"total warp-instr {tot_i:.3e}  samples {tot_s:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]/tot_i*100:5.1f}%i {v[1]/tot_s*100:5.1f}%s  {k[0]}:{k[1]}  {k[2]}")
print("--- by stall samples")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[0]/tot_i*100:5.1f}%i {v[1]/tot_s*100:5.1f}%s  {k[0]}:{k[1]}  {k[2]}")
