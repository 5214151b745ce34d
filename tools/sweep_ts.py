"""Seed-tile sweep of one BASELINE workload on one GPU (exploration tool).

usage: python tools/sweep_ts.py CONFIG [nx ny] --ts 8,12,16 [--steps 3]
Prints one JSON line per seed tile: device time per chain, DoF-updates/s,
executor/build, shared memory per CTA and peak HBM use.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1708_03183_b200 as lt
from paper_1708_03183_b200 import workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("dims", type=int, nargs="*")
ap.add_argument("--ts", default="16")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--chains", type=int, default=1)
ap.add_argument("--renumber", default=None)
a = ap.parse_args()
over = {"chains_per_step": a.chains}
if a.dims:
    over.update(nx=a.dims[0], ny=a.dims[1])
if a.renumber:
    over.update(renumber=a.renumber)
w = W.workload(a.config, **over)
t0 = time.perf_counter()
pb = W.build_problem(w)
print(json.dumps({"setup_s": round(time.perf_counter() - t0, 2), "cells": w.cells,
                  "hbm_gb": round(torch.cuda.memory_allocated() / 1e9, 2)}), flush=True)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()
for ts in (int(v) for v in a.ts.split(",")):
    try:
        t0 = time.perf_counter()
        s = lt.inspect_chain(pb.chain, ts, lt.ExecMode.SHARED)
        ti = time.perf_counter() - t0
        t0 = time.perf_counter()
        r = W.tiled_runner(pb, s, repeats=w.chains_per_step)
        g = r.graph(1)
        tp = time.perf_counter() - t0
        bench.timed(g.replay, 2, flush, stream)
        dt = bench.timed(g.replay, a.steps, flush, stream) / a.steps
        free, total = torch.cuda.mem_get_info()
        print(json.dumps({"ts": ts, "ms_per_step": round(dt * 1e3, 3),
                          "value": w.dofs * w.T * w.chains_per_step / dt,
                          "frac": W.roofline_bytes(pb.setup, w.heterogeneous) *
                          w.chains_per_step / dt / 6534.1e9,
                          "executor": r.executor, "wide": r.wide_build, "smem": r.smem_bytes,
                          "order": r.queue_order, "tiles": len(s.tiles),
                          "colors": len(s.color_order), "rounds": s.recolor_rounds,
                          "inspect_s": round(ti, 2), "plan_s": round(tp, 2),
                          "gpu_used_gb": round((total - free) / 1e9, 1)}), flush=True)
        del g, r, s
    except Exception as e:
        print(json.dumps({"ts": ts, "error": str(e)[:300]}), flush=True)
    torch.cuda.empty_cache()
