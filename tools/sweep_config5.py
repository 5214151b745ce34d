"""BASELINE config 5 on one B200: the degree x chain-length x seed-tile sweep.

Config 5 is P1-P4 x chain length 1/2/4 timesteps x seed tile 1K/4K/16K cells
at ~2e9 DoFs over 8 B200s (random per-cell materials U[1,2], seed 3, 20
timesteps per point).  One GPU of this run holds one rank's share: the first
of 8 horizontal strips of the suggested global meshes (P1
8192^2, P2 8192x4096, P3 4480^2, P4 3648^2), i.e. cells 0 .. C/8 -- whose
material draws are exactly the global draws of those cells.  Every point is
timed twice: at BASELINE's seed tile (1K/4K/16K cells: tiles far larger than a
CTA's shared memory, run by the global-memory tile executor) and at the seed
tile the shared-memory dataflow executor is tuned for.  The tuned tile is
chosen per (P, T) from a short sweep.  Each point checks legality
(lt_check_legality) and reports the tiled/untiled ratio.

usage: python tools/sweep_config5.py [--degrees 1,2,3,4] [--chains 1,2,4] [--out FILE]
"""
import argparse
import gc
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1708_03183_b200 as lt
from paper_1708_03183_b200 import workloads as W
from paper_1708_03183_b200.executor import UntiledRunner

GLOBAL = {1: (8192, 8192), 2: (8192, 4096), 3: (4480, 4480), 4: (3648, 3648)}
TUNE = {1: (24, 32, 48), 2: (12, 16, 24), 3: (8, 12, 16), 4: (6, 8, 12)}
# --layout block: every seed tile is one block of quads of the layout pass
# (dg.morton_renumber_device, "block:BXxBY" with 2*BX*BY = ts)
TUNE_BLOCK = {1: ((32, "4x4"), (48, "6x4"), (16, "4x2")), 2: ((32, "4x4"), (24, "4x3"), (16, "4x2")),
              3: ((24, "4x3"), (16, "4x2"), (8, "2x2")), 4: ((16, "4x2"), (12, "3x2"), (8, "2x2"))}
STATED_BLOCK = {1024: "32x16", 4096: "64x32", 16384: "128x64"}

ap = argparse.ArgumentParser()
ap.add_argument("--degrees", default="1,2,3,4")
ap.add_argument("--chains", default="1,2,4")
ap.add_argument("--stated", default="1024,4096,16384")
ap.add_argument("--timesteps", type=int, default=4, help="timesteps timed per point")
ap.add_argument("--out", default=None)
ap.add_argument("--layout", default="none", choices=["none", "block"])
a = ap.parse_args()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()
out = open(a.out, "a") if a.out else None


def emit(d):
    line = json.dumps(d)
    print(line, flush=True)
    if out:
        out.write(line + "\n")
        out.flush()


def time_runner(run, chains):
    bench.timed(run, 1, flush, stream)
    return bench.timed(run, chains, flush, stream) / chains


for p in (int(v) for v in a.degrees.split(",")):
    gx, gy = GLOBAL[p]
    for T in (int(v) for v in a.chains.split(",")):
        w = W.Workload(5, gx, gy // 8, p, T, ("uniform", 3), 1, 8.0, ts=TUNE[p][1],
                       ts_stated=None, job_chains=max(1, 20 // T), chains_per_step=1,
                       device_setup=True, text=f"config 5 share P{p} T={T}")
        t0 = time.perf_counter()
        pb = W.build_problem(w)
        setup_s = time.perf_counter() - t0
        chains = max(1, a.timesteps // T)
        ur = UntiledRunner(pb.chain, pb.bindings, pb.datasets, pb.registry)
        u_s = time_runner(ur, chains)
        del ur
        torch.cuda.empty_cache()
        upd = w.dofs * T
        base = {"p": p, "T": T, "mesh": f"{gx}x{gy // 8}", "cells": w.cells, "dofs": w.dofs,
                "untiled_ms_per_chain": round(u_s * 1e3, 3), "untiled_value": upd / u_s,
                "setup_s": round(setup_s, 1)}
        if a.layout == "block":
            points = [("tuned", ts, b) for ts, b in TUNE_BLOCK[p]] + \
                     [("stated", int(v), STATED_BLOCK[int(v)]) for v in a.stated.split(",")]
        else:
            points = [("tuned", ts, None) for ts in TUNE[p]] + \
                     [("stated", int(v), None) for v in a.stated.split(",")]
        for kind, ts, blk in points:
            if True:
                try:
                    if blk is not None:  # the layout is part of the problem: rebuild it
                        pb = None
                        gc.collect()  # problems hold reference cycles: free their tensors now
                        torch.cuda.empty_cache()
                        from dataclasses import replace
                        pb = W.build_problem(replace(w, renumber="block:" + blk))
                        base["layout"] = "block:" + blk
                    t0 = time.perf_counter()
                    s = lt.inspect_chain(pb.chain, ts, lt.ExecMode.SHARED)
                    insp = time.perf_counter() - t0
                    leg = lt.check_legality_gpu(s, pb.chain)
                    r = W.tiled_runner(pb, s, repeats=1)
                    g = r.graph(1)
                    dt = time_runner(g.replay, chains)
                    emit(dict(base, kind=kind, ts=ts, ms_per_chain=round(dt * 1e3, 3),
                              value=upd / dt, tiled_over_untiled=u_s / dt,
                              frac=W.roofline_bytes(pb.setup, True) / dt / 6534.1e9,
                              executor=r.executor, smem=r.smem_bytes, wide=r.wide_build,
                              colors=len(s.color_order), rounds=s.recolor_rounds,
                              inspect_s=round(insp, 2), legality=leg))
                    del g, r, s
                except Exception as e:
                    emit(dict(base, kind=kind, ts=ts, error=str(e).splitlines()[0][:200]))
                torch.cuda.empty_cache()
        pb = None
        torch.cuda.empty_cache()
