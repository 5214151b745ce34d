"""Benchmark: DoF-timestep updates/s of the tiled elastic-wave DG loop chain.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2|3|4]
    python bench.py --impl reference ...     # the reference CPU path (looptile)

Workloads (``paper_1708_03183_b200/workloads.py``, BASELINE.json configs):

* default, config 4: DG P3 on the 8192x4096 right-diagonal mesh (67.1M
  cells, 3.36e9 DoFs), homogeneous, Gaussian pulse, two timesteps per chain
  -- the largest elastic-wave configuration and the one BASELINE strong-scales
  over 1/2/4/8 GPUs.  Generated on the GPU (no host pass over the mesh), cells
  numbered block by block (4x3 quads per seed tile) by the layout pass (``renumber``).
* config 3: DG P2 2048x2048, heterogeneous, two timesteps per chain
  (``--stated-ts`` also times BASELINE's seed tile 4096).
* config 2: DG P1 256x256, one timestep per chain, 10 chains per step.

A bench *step* executes ``chains_per_step`` chains of the fused tiled executor
(one persistent ``k_dataflow`` launch, captured in a CUDA graph) with the
inputs resident in HBM; L2 (126 MB) is flushed by a 256 MiB write between
steps.  Synthetic data (no datasets exist for this path).

Multi-GPU (torchrun, N > 1): the config-4 mesh is cut into N contiguous
horizontal strips (the reference partitioner's cell blocks) with extended
halos of depth = loops per chain; each rank generates only its strip, runs
core tiles, one NCCL halo exchange per chain, boundary tiles.  Strong
scaling (fixed global mesh); time = max over ranks.

The JSON line carries ``roofline`` (SURVEY 8(d) algorithmic bytes per launch
of the dominant kernel over its CUDA-event time vs MEASURED_PEAKS hbm_gbs),
``cpu_baseline`` (the reference's own executor on a bounded sample, host
cores of the GPU box), ``e2e`` (the same job through the public API with
host buffers: H2D of u, s from pinned memory, the step, D2H of u, s),
``omega`` (the GPU untiled executor on the same problem: the paper's
tiled/original speed-up on B200) and ``clocks``.
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

METRIC = "DoF-timestep updates/s of tiled elastic-wave loop chain"
DEFAULT_CONFIG = 4


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=(2, 3, 4))
    ap.add_argument("--ts", type=int, default=None, help="seed tile (default: tuned)")
    ap.add_argument("--stated-ts", action="store_true",
                    help="also time the configuration's stated seed tile (config 3: 4096)")
    ap.add_argument("--chains", type=int, default=None, help="chains per step")
    ap.add_argument("--renumber", default=None,
                    help="layout pass of the device generator: none, morton, block:BXxBY")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-omega", action="store_true")
    ap.add_argument("--untiled", action="store_true", help="time the untiled GPU executor")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas instead of the partitioned mesh")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the partitioned (halo-exchange) path even at N=1")
    return ap.parse_args(argv)


def dist_init():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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


def sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
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
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def recorded_traffic(config, ts):
    """ncu dram bytes per launch of k_dataflow for this workload (profiles/traffic.json)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as fh:
        d = json.load(fh)
    e = d.get(f"config{config}_ts{ts}")
    if isinstance(e, dict):
        return e.get("dram_bytes_per_launch"), e.get("source")
    return None, None


# ---- CPU baselines (reference looptile, bounded samples) --------------------------

CPU_SAMPLE = {2: 128, 3: 96, 4: 96}     # mesh edge of the cpu_baseline sample (~10-30 s)
REF_ARM_SAMPLE = {2: 48, 3: 40, 4: 40}  # per --impl reference step (~1-4 s)


def cpu_sample(w, n):
    """(rate, seconds, description, kind) of one chain on an n x n mesh."""
    from oracle import reference_runner
    ts = max(1, w.ts) if w.ts_stated is None else max(1, w.ts_stated * n * n // w.cells)
    r = reference_runner.sample_rate(w.p, w.T, n, w.material, ts, noise_seed=w.noise_seed)
    if r is not None:
        return r + ("reference",)
    from oracle import looptile_oracle as O
    from paper_1708_03183_b200.chain import build_chain
    from paper_1708_03183_b200.dg import elastic_setup
    st = elastic_setup(n, n, w.p, w.T, material=w.material, sigma=8.0 * n / 256)
    chain = build_chain(tuple(st.spaces.values()), tuple(st.maps.values()), st.loops,
                        len(st.loops))
    sched = O.inspect(chain, ts, "shared")
    data = {k: v.copy() for k, v in st.data.items()}
    t0 = time.perf_counter()
    O.execute_tiled(sched, chain, st.bindings, data, st.vpe, O.kernel_table(dg=(st.p, st.dt)))
    dt = time.perf_counter() - t0
    return (st.dofs * w.T / dt, dt, f"oracle port execute_tiled, DG P{w.p} {n}x{n}, one "
            f"{w.T}-timestep chain, 1 core", "port")


def run_reference(args, w):
    """--impl reference: the reference's own CPU executor, one bounded sample per step."""
    n = REF_ARM_SAMPLE[w.config]
    for _ in range(args.warmup):
        cpu_sample(w, 16)
    upd, tot, desc, kind = 0.0, 0.0, "", "port"
    for _ in range(args.steps):
        rate, dt, desc, kind = cpu_sample(w, n)
        upd += rate * dt
        tot += dt
    value = upd / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "DoF-updates/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if w.config == 4 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.text + f" [reference CPU sample per step: {desc}]",
                       "parallelism": "cpu, 1 core (GIL-bound Python executor)"},
            "cpu_baseline": {"value": value, "unit": "DoF-updates/s", "cores": 1, "kind": kind,
                             "sample": desc},
            "e2e": {"value": value, "unit": "DoF-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- GPU arm ---------------------------------------------------------------------

def timed(step, n, flush, stream):
    """CUDA-event time of n steps (L2 flushed before each), seconds."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(n)]
    for i in range(n):
        flush.zero_()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) * 1e-3


def run_single(args, w, rank, world, local):
    import torch
    import paper_1708_03183_b200 as lt
    from paper_1708_03183_b200 import workloads as W
    from paper_1708_03183_b200.executor import UntiledRunner
    t0 = time.perf_counter()
    pb = W.build_problem(w)
    setup_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    sched = lt.inspect_chain(pb.chain, w.ts, lt.ExecMode.SHARED)
    inspect_s = time.perf_counter() - t0
    chains = w.chains_per_step
    t0 = time.perf_counter()
    if args.untiled:
        runner = UntiledRunner(pb.chain, pb.bindings, pb.datasets, pb.registry)
        graph = None
    else:
        runner = W.tiled_runner(pb, sched, repeats=chains)
        graph = runner.graph(1)
    plan_s = time.perf_counter() - t0

    def step():
        if graph is not None:
            graph.replay()
        else:
            for _ in range(chains):
                runner()

    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    barrier(world)
    with ClockSampler(local) as clk:
        dev_s = timed(step, args.steps, flush, stream)
        barrier(world)
    dev_s = max_over_ranks(dev_s, world)
    updates_per_step = w.dofs * w.T * chains
    value = updates_per_step * world * args.steps / dev_s
    launches_per_step = runner.launches_per_call * (1 if graph is not None else chains)
    sched_stats = {"tiles": len(sched.tiles), "colors": len(sched.color_order),
                   "rounds": sched.recolor_rounds}
    executor = "untiled" if args.untiled else runner.executor
    build = None if args.untiled else ("wide (128 regs, <= 4 CTAs/SM)" if runner.wide_build
                                       else "narrow (80 regs, 6 CTAs/SM)")
    queue_order = None if args.untiled else runner.queue_order
    free_b, total_b = torch.cuda.mem_get_info()
    hbm_used_gb = round((total_b - free_b) / 1e9, 1)

    # roofline of the dominant kernel: k_dataflow is the step's only launch when
    # chains_per_step == 1 (with repeats > 1 the step adds k_pack_ro, ~4 %)
    b_chain = W.roofline_bytes(pb.setup, w.heterogeneous)
    peak, peak_src = measured_peaks()
    achieved = b_chain * chains * args.steps / dev_s / 1e9
    traffic, traffic_src = recorded_traffic(w.config, w.ts)

    stated = None
    if args.stated_ts and w.ts_stated and not args.untiled:
        s2 = lt.inspect_chain(pb.chain, w.ts_stated, lt.ExecMode.SHARED)
        r2 = W.tiled_runner(pb, s2, repeats=chains)
        g2 = r2.graph(1)
        timed(g2.replay, 1, flush, stream)
        s_s = timed(g2.replay, 2, flush, stream)
        stated = {"ts": w.ts_stated, "value": updates_per_step * 2 / s_s,
                  "ms_per_step": s_s / 2 * 1e3, "executor": r2.executor,
                  "colors": len(s2.color_order), "rounds": s2.recolor_rounds}
        del g2, r2

    e2e = None
    if not args.no_e2e:
        host = {n: torch.empty(pb.datasets[n].values.numel(), dtype=torch.float64,
                               pin_memory=True) for n in ("u", "s")}
        for n in host:
            host[n].copy_(pb.datasets[n].values)
        h2d = sum(h.numel() * 8 for h in host.values())
        torch.cuda.synchronize()
        barrier(world)

        def e2e_step():
            for n in host:
                pb.datasets[n].values.copy_(host[n], non_blocking=True)
            step()
            for n in host:
                host[n].copy_(pb.datasets[n].values, non_blocking=True)

        n_e2e = max(1, min(args.steps, 5))
        e2e_s = max_over_ranks(timed(e2e_step, n_e2e, flush, stream), world)
        e2e = {"value": updates_per_step * world * n_e2e / e2e_s, "unit": "DoF-updates/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d}
        del host

    # the paper's Omega on B200: the untiled GPU executor on the same problem
    # (run last, after the tiled plan is released: at 67M cells both do not fit)
    omega = None
    if not args.no_omega and not args.untiled and world == 1:
        graph = runner = sched = None  # releases the tiled plan (held by the schedule)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        try:
            ur = UntiledRunner(pb.chain, pb.bindings, pb.datasets, pb.registry)
            ustep = lambda: [ur() for _ in range(chains)]
            timed(ustep, 1, flush, stream)
            u_s = timed(ustep, 2, flush, stream)
            u_rate = updates_per_step * 2 / u_s
            omega = {"untiled_value": u_rate, "tiled_over_untiled": value / u_rate,
                     "untiled_launches_per_chain": ur.launches_per_call}
            del ur
        except Exception as e:  # memory: the untiled facet scratch at 67M cells
            omega = {"untiled_value": None, "error": str(e).splitlines()[0][:160]}
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, dt, sample, kind = cpu_sample(w, CPU_SAMPLE[w.config])
        cpu = {"value": rate, "unit": "DoF-updates/s", "cores": 1, "kind": kind,
               "sample": sample + f" ({dt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "DoF-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if w.config == 4 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.text, "p": w.p, "cells": w.cells, "dofs": w.dofs,
                       "timesteps_per_chain": w.T, "chains_per_step": chains,
                       "job_chains": w.job_chains, "seed_tile": w.ts,
                       "seed_tile_stated": w.ts_stated, "renumber": w.renumber or "none",
                       "mode": "shared",
                       **sched_stats, "setup_s": round(setup_s, 2),
                       "inspect_s": round(inspect_s, 3), "plan_s": round(plan_s, 2),
                       "executor": executor, "dataflow_build": build,
                       "queue_order": queue_order,
                       "l2": "flushed between steps (256 MiB write)",
                       "hbm_used_gb": hbm_used_gb,
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_dataflow" + ("" if chains == 1 else " + k_pack_ro"),
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_chain": b_chain,
                         "algorithmic_bytes_basis": "SURVEY 8(d): u,s read+written, if2c/ef2c, "
                         "cell+facet geometry, material if heterogeneous (workloads.roofline_bytes)",
                         "traffic_source": traffic_src,
                         "launches_per_step": launches_per_step},
            "cpu_baseline": cpu,
            "omega": omega,
            "stated_ts": stated,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main(argv=None):
    args = parse(argv)
    from paper_1708_03183_b200 import workloads as W
    over = {}
    if args.ts:
        over["ts"] = args.ts
    if args.chains:
        over["chains_per_step"] = args.chains
    if args.renumber:
        over["renumber"] = None if args.renumber == "none" else args.renumber
    w = W.workload(args.config, **over)
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        run_reference(args, w)
        return
    import torch
    rank, world, local = dist_init()
    torch.cuda.set_device(local)
    try:
        if (world > 1 and not args.replicas) or args.partitioned:
            from paper_1708_03183_b200 import strips
            strips.bench_partitioned(args, w, rank, world, local, sys.modules[__name__])
        else:
            run_single(args, w, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
