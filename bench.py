"""Benchmark: DoF-timestep updates/s of the tiled elastic-wave DG loop chain.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2|3|4]
    python bench.py --impl reference ...     # CPU reference arm (oracle port)

Workload (BASELINE.json configs[1], "config 2"): velocity-stress DG P1 on a
256x256 right-diagonal triangulation of [0,256]^2 (131,072 cells), rho=1,
lambda=2, mu=1, Gaussian pulse (sigma 8) + U[-1e-3,1e-3] noise (seed 1),
dt = 0.1/(sqrt(4)*3), one timestep per chain, 10 timesteps per job.
A bench *step* is that whole job: 10 chain executions (5 loops each) of the
fused tiled executor, captured in one CUDA graph, inputs resident in HBM.
L2 is flushed (256 MiB write) between timed steps because the working set
(~40 MB) fits the 126 MB L2.  Synthetic data (no datasets exist for this path).

Multi-GPU (torchrun): each rank runs its own replica of the job (weak
scaling, no data-path collective); time = max over ranks.

The JSON line carries ``roofline`` (compulsory bytes of the chain / device
time vs MEASURED_PEAKS hbm_gbs), ``cpu_baseline`` (the CPU oracle -- a
restatement of the reference's per-element executor -- on a bounded sample),
``e2e`` (the same job through the public API with host buffers: H2D of u,s
from pinned memory, 10 timesteps, D2H of u,s) and ``clocks``.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (nx, ny, p, steps_per_chain, chains_per_job, material, ts, renumber)
    2: dict(nx=256, ny=256, p=1, T=1, chains=10, material="homogeneous", ts=32,
            workload="elastic DG P1 256x256 (131072 cells), 1 timestep/chain, 10 timesteps"),
    3: dict(nx=2048, ny=2048, p=2, T=2, chains=1, material=("uniform", 2), ts=24,
            workload="elastic DG P2 2048x2048 (8.4M cells), 2 timesteps/chain, heterogeneous"),
}
METRIC = "DoF-timestep updates/s of tiled elastic-wave loop chain"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--ts", type=int, default=None)
    ap.add_argument("--renumber", default="none")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--chains", type=int, default=None,
                    help="override chain executions per step (exploration only)")
    ap.add_argument("--untiled", action="store_true", help="time the untiled GPU executor")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas instead of the partitioned mesh")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the partitioned (halo-exchange) path even at N=1")
    return ap.parse_args()


def dist_init(n):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl")
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm_sorted = sorted(sm)
        return {"sm_mhz": sm_sorted[len(sm) // 2], "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def cpu_oracle_sample(cfg, seconds_hint=True):
    """Time the CPU oracle (restatement of the reference executor) on a bounded
    sample: the same chain (degree, T) on a 64x64 mesh, one chain execution."""
    from oracle import looptile_oracle as O
    from paper_1708_03183_b200.chain import build_chain
    from paper_1708_03183_b200.dg import elastic_setup
    n = 64
    st = elastic_setup(n, n, cfg["p"], cfg["T"], material=cfg["material"],
                       sigma=8.0 * n / 256)
    chain = build_chain(tuple(st.spaces.values()), tuple(st.maps.values()), st.loops,
                        len(st.loops))
    ts = max(1, cfg["ts"] * n * n // (cfg["nx"] * cfg["ny"])) if cfg["nx"] > n else cfg["ts"]
    sched = O.inspect(chain, ts, "shared")
    kern = O.kernel_table(dg=(st.p, st.dt))
    data = {k: v.copy() for k, v in st.data.items()}
    t0 = time.perf_counter()
    O.execute_tiled(sched, chain, st.bindings, data, st.vpe, kern)
    dt = time.perf_counter() - t0
    return st.dofs * cfg["T"] / dt, dt, f"P{cfg['p']} {n}x{n} ({st.n_cells} cells), " \
        f"{cfg['T']} timestep chain, oracle execute_tiled (per-element numpy bodies, 1 core)"


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_oracle_sample(cfg)
    total_upd, total_t = 0.0, 0.0
    sample = ""
    for _ in range(args.steps):
        rate, dt, sample = cpu_oracle_sample(cfg)
        total_upd += rate * dt
        total_t += dt
    value = total_upd / total_t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "DoF-updates/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_t / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"] + " [CPU sample: " + sample + "]",
                       "parallelism": "cpu"},
            "cpu_baseline": {"value": value, "unit": "DoF-updates/s", "cores": 1,
                             "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "DoF-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_partitioned(args, cfg, rank, world, local):
    """Weak-scaled strip partition: rank r owns a 256 x 256-cell block of a
    256 x (256 N) mesh plus a 5T-strip extended halo; one NCCL halo exchange
    per chain (begin before the core tiles, end before the boundary tiles)."""
    import torch
    import paper_1708_03183_b200 as lt
    from paper_1708_03183_b200.dg import (compulsory_bytes, constant_datasets, elastic_problem,
                                          elastic_setup, local_elastic_setup)
    from paper_1708_03183_b200.distributed import HaloExchange, exchanged_from_chain
    from paper_1708_03183_b200.partition import partition_for_ranks
    T = cfg["T"]
    st = elastic_setup(cfg["nx"], cfg["ny"] * world, cfg["p"], T, material=cfg["material"],
                       renumbering=args.renumber)
    depth = 5 * T
    lm = partition_for_ranks(st.mesh, world, depth)[rank]
    loc = local_elastic_setup(st, lm)
    pb = elastic_problem(loc, depth=len(loc.loops))
    pb.install_params()
    t0 = time.perf_counter()
    sched = lt.inspect_chain(pb.chain, cfg["ts"], lt.ExecMode.SHARED)
    inspect_s = time.perf_counter() - t0
    const = constant_datasets(pb.chain, pb.bindings)
    exchanged = tuple(n for n in exchanged_from_chain(pb.chain, pb.bindings) if n not in const)
    ex = HaloExchange(lm, pb.datasets, exchanged)
    from paper_1708_03183_b200.executor import TiledRunner
    runner = TiledRunner(sched, pb.chain, pb.bindings, pb.datasets, pb.registry)
    launches = [0]

    def step():
        for _ in range(cfg["chains"]):
            launches[0] += runner.with_exchange(ex)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    barrier(world)
    stream = torch.cuda.current_stream()
    ev = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            ev.append((a, b))
        torch.cuda.synchronize()
        barrier(world)
    dev_s = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) * 1e-3, world)
    launches_per_step = launches[0] // max(args.warmup + args.steps, 1)
    # end to end: H2D of the rank's u,s (pinned), the step, D2H of u,s
    e2e_s = None
    if not args.no_e2e:
        host = {n: torch.empty(pb.datasets[n].values.numel(), dtype=torch.float64,
                               pin_memory=True) for n in ("u", "s")}
        for n in host:
            host[n].copy_(pb.datasets[n].values)
        h2d = sum(h.numel() * 8 for h in host.values())
        e2e_ev = []
        torch.cuda.synchronize()
        barrier(world)
        for _ in range(max(1, args.steps)):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for n in host:
                pb.datasets[n].values.copy_(host[n], non_blocking=True)
            step()
            for n in host:
                host[n].copy_(pb.datasets[n].values, non_blocking=True)
            b.record(stream)
            e2e_ev.append((a, b))
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(sum(a.elapsed_time(b) for a, b in e2e_ev) * 1e-3, world)
    owned = lm.sizes["cells"].owned_total
    owned_dofs = owned * 5 * (cfg["p"] + 1) * (cfg["p"] + 2) // 2
    total_dofs = owned_dofs
    if world > 1:
        import torch.distributed as dist
        tdofs = torch.tensor([owned_dofs], dtype=torch.float64, device="cuda")
        dist.all_reduce(tdofs)
        total_dofs = int(tdofs.item())
    updates = total_dofs * T * cfg["chains"] * args.steps
    value = updates / dev_s
    e2e = None
    if e2e_s is not None:
        e2e = {"value": total_dofs * T * cfg["chains"] * len(e2e_ev) / e2e_s,
               "unit": "DoF-updates/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d}
    totals = {n: loc.spaces[loc.space_of[n]].total for n in loc.vpe}
    b_chain = compulsory_bytes(pb.chain, pb.bindings, dict(loc.vpe), totals)
    peak, peak_kind = measured_peaks()
    achieved = b_chain * world * cfg["chains"] * args.steps / dev_s / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "DoF-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg["workload"] + f" per rank; strips of a {cfg['nx']}x"
                                   f"{cfg['ny'] * world} mesh, halo depth {depth}",
                       "p": cfg["p"], "cells_total": st.n_cells, "dofs_total": total_dofs,
                       "seed_tile": cfg["ts"], "mode": "shared", "colors_rank0":
                       len(sched.color_order), "inspect_s": round(inspect_s, 4),
                       "halo_exchange": "NCCL batch_isend_irecv once per chain" if world > 1
                       else "none (1 rank)",
                       "bytes_exchanged_per_chain_rank0": ex.bytes_exchanged //
                       max(ex.exchange_count, 1),
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"partitioned x{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world,
                         "unit": "GB/s", "frac": achieved / (peak * world), "traffic": None,
                         "peak_source": peak_kind,
                         "algorithmic_bytes_per_chain_rank0": b_chain},
            "cpu_baseline": None, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    cfg = dict(CONFIGS[args.config])
    if args.ts:
        cfg["ts"] = args.ts
    if args.chains:
        cfg["chains"] = args.chains
    import torch
    rank, world, local = (0, 1, 0)
    if args.impl == "reference":
        if int(os.environ.get("WORLD_SIZE", "1")) > 1 and int(os.environ.get("RANK", "0")) != 0:
            return
        run_reference(args, cfg, 0, 1)
        return
    rank, world, local = dist_init(args.gpus)
    torch.cuda.set_device(local)
    if (world > 1 and not args.replicas) or args.partitioned:
        return run_partitioned(args, cfg, rank, world, local)

    import paper_1708_03183_b200 as lt
    from paper_1708_03183_b200.dg import (compulsory_bytes, elastic_problem, elastic_setup)
    from paper_1708_03183_b200.executor import TiledRunner, UntiledRunner

    st = elastic_setup(cfg["nx"], cfg["ny"], cfg["p"], cfg["T"], material=cfg["material"],
                       renumbering=args.renumber)
    pb = elastic_problem(st)
    pb.install_params()
    t0 = time.perf_counter()
    sched = lt.inspect_chain(pb.chain, cfg["ts"], lt.ExecMode.SHARED)
    inspect_s = time.perf_counter() - t0
    if args.untiled:
        runner = UntiledRunner(pb.chain, pb.bindings, pb.datasets, pb.registry)
        graph = None
    else:
        runner = TiledRunner(sched, pb.chain, pb.bindings, pb.datasets, pb.registry,
                             repeats=cfg["chains"])
        graph = runner.graph(1)

    def step():
        if graph is not None:
            graph.replay()
        else:
            for _ in range(cfg["chains"]):
                runner()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    barrier(world)

    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        barrier(world)
    dev_s = sum(a.elapsed_time(b) for a, b in ev) * 1e-3
    dev_s = max_over_ranks(dev_s, world)

    dofs = st.dofs
    updates_per_step = dofs * cfg["T"] * cfg["chains"]
    value = updates_per_step * world * args.steps / dev_s
    ms_per_step = dev_s / args.steps * 1e3

    # roofline of the fused tile kernel (only kernel in the step)
    vpe = dict(st.vpe)
    totals = {n: st.spaces[st.space_of[n]].total for n in vpe}
    b_chain = compulsory_bytes(pb.chain, pb.bindings, vpe, totals)
    calls_per_step = 1 if graph is not None else cfg["chains"]
    launches_per_step = runner.launches_per_call * calls_per_step
    # the fused executor's step: one k_dataflow launch running all chains (plus,
    # for repeated chains, the k_pack_ro launch that feeds it, ~4 % of the
    # step); algorithmic bytes of the step over its device time
    achieved = b_chain * cfg["chains"] * args.steps / dev_s / 1e9
    peak, peak_kind = measured_peaks()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get(f"config{args.config}")

    # end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        host = {n: torch.empty(pb.datasets[n].values.numel(), dtype=torch.float64,
                               pin_memory=True) for n in ("u", "s")}
        for n in host:
            host[n].copy_(pb.datasets[n].values)
        h2d = sum(h.numel() * 8 for h in host.values())
        e2e_ev = []
        torch.cuda.synchronize()
        barrier(world)
        for i in range(max(1, args.steps)):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for n in host:
                pb.datasets[n].values.copy_(host[n], non_blocking=True)
            step()
            for n in host:
                host[n].copy_(pb.datasets[n].values, non_blocking=True)
            b.record(stream)
            e2e_ev.append((a, b))
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(sum(a.elapsed_time(b) for a, b in e2e_ev) * 1e-3, world)
        e2e = {"value": updates_per_step * world * len(e2e_ev) / e2e_s, "unit": "DoF-updates/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, dt, sample = cpu_oracle_sample(cfg)
        cpu = {"value": rate, "unit": "DoF-updates/s", "cores": 1, "kind": "port",
               "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "DoF-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "p": cfg["p"], "cells": st.n_cells,
                       "dofs": dofs, "timesteps_per_chain": cfg["T"],
                       "chains_per_step": cfg["chains"], "seed_tile": cfg["ts"],
                       "renumber": args.renumber, "mode": "shared",
                       "colors": len(sched.color_order), "rounds": sched.recolor_rounds,
                       "inspect_s": round(inspect_s, 4),
                       "executor": "untiled" if args.untiled else runner.executor,
                       "queue_order": None if args.untiled else runner.queue_order,
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_kind,
                         "algorithmic_bytes_per_chain": b_chain,
                         "unit_of_time": "bench step (k_dataflow + k_pack_ro launches)",
                         "traffic_of": "k_dataflow, ncu dram bytes per launch (profiles/traffic.json)",
                         "launches_per_step": launches_per_step},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
