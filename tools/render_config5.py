"""Render a tools/sweep_config5.py JSONL result as a markdown table.
usage: python tools/render_config5.py sweep.jsonl > table.md"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
print("| P | T | mesh (1/8 strip) | layout | kind | ts | ms/chain | DoF-updates/s | x untiled | frac | executor | smem/CTA | colours | legal |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    if "error" in r:
        print(f"| {r['p']} | {r['T']} | {r['mesh']} | {r.get('layout', 'none')} | {r['kind']} | {r['ts']} | "
              f"error: {r['error'][:60]} | | | | | | | |")
        continue
    leg = r.get("legality", {})
    ok = "yes" if leg == {"pairs": 0, "reductions": 0} else str(leg)
    print(f"| {r['p']} | {r['T']} | {r['mesh']} | {r.get('layout', 'none')} | {r['kind']} | {r['ts']} | "
          f"{r['ms_per_chain']:.2f} | {r['value']:.3g} | {r['tiled_over_untiled']:.2f} | {r['frac']:.3f} | "
          f"{r['executor']} | {r['smem']} | {r['colors']} | {ok} |")
