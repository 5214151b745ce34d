"""Rank-local strip partitions of the rectangular DG meshes (BASELINE config 4).

The reference partitioner (``pkg/src/looptile/partition.py:85-138``) splits the
cells into contiguous blocks (``np.array_split`` over the row-major cells:
horizontal bands of the structured mesh), grows ``depth`` halo strips through
shared vertices, and orders each rank's elements core | owned | exec |
non-exec by global id.  ``partition.partition_for_ranks`` restates it over
the whole mesh -- O(global) work and memory on every rank, which does not
reach the 67M-cell configuration.

Here each rank builds only its own strip: the same decomposition
(``partition.partition_with_owners``) runs on a *window* of quad rows around
the rank's band, wide enough (halo depth + 2 rows on each side) that every
element of the local mesh sees exactly the incidence it has in the global
mesh.  Global ids are restored in closed form (cells and vertices are
row-major; edges follow ``generate_rect_mesh``'s per-vertex order), so the
local mesh equals ``partition_for_ranks(global)[rank]`` -- sizes, global ids,
local maps and the local side of every exchange table
(tests/test_strips.py); the window does not hold the neighbours' local
numbering, so the neighbour column of the exchange tables is -1 (the halo
exchange only uses the local side).  The rank-local elastic problem is the
window's ``dg.elastic_setup`` (global pulse centre, random streams advanced
to the window's first cell) restricted like ``dg.local_elastic_setup``.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .mesh import CELLS, EDGES, VERTS, Mesh, generate_rect_mesh
from .partition import LocalMesh, partition_with_owners


def cell_blocks(n_cells: int, nranks: int) -> np.ndarray:
    """First cell of every rank's block, ``np.array_split`` semantics (+ end)."""
    sizes = np.full(nranks, n_cells // nranks, dtype=np.int64)
    sizes[: n_cells % nranks] += 1
    return np.concatenate([[0], np.cumsum(sizes)])


def edge_gid(a: np.ndarray, b: np.ndarray, nx: int, ny: int) -> np.ndarray:
    """Global id of the edge (a, b), a < b, of the nx x ny right-diagonal mesh:
    per vertex (i, j) in order, its right, up and diagonal edges (where they
    exist), the order ``mesh.generate_rect_mesh`` emits."""
    nvx = nx + 1
    i, j = a % nvx, a // nvx
    per_row = 3 * nx + 1
    base = np.where(j < ny, j * per_row + 3 * i, ny * per_row + i)
    slot = np.where(b - a == 1, 0, np.where(b - a == nvx, 1, 2))
    return np.where((j < ny) & (i < nx), base + slot, base)


@dataclass
class StripPartition:
    nx: int
    ny: int
    nranks: int
    depth: int
    rank: int
    rows: tuple           # window quad rows [j0, j1)
    window: Mesh          # window mesh (window-local ids, global coordinates)
    local_window: LocalMesh   # the rank's local mesh in window ids
    local: LocalMesh          # the same with global ids
    gid: dict                 # window id -> global id per space

    @property
    def cell_offset(self) -> int:
        return 2 * self.nx * self.rows[0]


def strip_partition(nx: int, ny: int, nranks: int, depth: int, rank: int) -> StripPartition:
    """``partition_for_ranks(generate_rect_mesh(nx, ny), nranks, depth)[rank]``
    built from a window of rows around the rank's strip."""
    C = 2 * nx * ny
    if not 0 <= rank < nranks or nranks > C:
        raise ValueError(f"rank {rank} of {nranks} for {C} cells")
    bounds = cell_blocks(C, nranks)
    lo_row = int(bounds[rank] // (2 * nx))
    hi_row = int((bounds[rank + 1] - 1) // (2 * nx)) + 1
    j0 = max(0, lo_row - depth - 2)
    j1 = min(ny, hi_row + depth + 2)
    # ranks whose cells meet the window: theirs and our exchange tables
    c0, c1 = 2 * nx * j0, 2 * nx * j1
    others = [q for q in range(nranks) if bounds[q] < c1 and bounds[q + 1] > c0]
    m = generate_rect_mesh(nx, j1 - j0)
    coords = m.vertex_coords.copy()
    coords[:, 1] += j0
    win = Mesh(m.num_vertices, m.num_cells, m.num_edges, m.cells_to_vertices,
               m.edges_to_vertices, coords)
    gcell = np.arange(win.num_cells, dtype=np.int64) + c0
    gvert = np.arange(win.num_vertices, dtype=np.int64) + (nx + 1) * j0
    pairs = win.edges_to_vertices.reshape(-1, 2) + (nx + 1) * j0
    gedge = edge_gid(pairs[:, 0], pairs[:, 1], nx, ny)
    owner = np.searchsorted(bounds, gcell, side="right") - 1
    lms = partition_with_owners(win, owner, nranks, depth, others, mirror=False)
    lw = lms[others.index(rank)]
    gid = {CELLS: gcell, VERTS: gvert, EDGES: gedge}
    g = LocalMesh(rank=rank, sizes=lw.sizes, cells_to_vertices=lw.cells_to_vertices,
                  edges_to_vertices=lw.edges_to_vertices, vertex_coords=lw.vertex_coords,
                  global_ids={sp: gid[sp][ids] for sp, ids in lw.global_ids.items()},
                  exchange_table=lw.exchange_table)
    return StripPartition(nx, ny, nranks, depth, rank, (j0, j1), win, lw, g, gid)


def strip_elastic_setup(sp: StripPartition, p: int, steps_per_chain: int, material,
                        noise_seed, sigma: float, dt: float):
    """The rank-local elastic problem of a strip (``dg.local_elastic_setup`` of
    the global problem, built from the window only).  ``dt`` is the global
    timestep (it depends on the largest wave speed over all cells)."""
    from .dg import elastic_setup, local_elastic_setup
    win = elastic_setup(sp.nx, sp.rows[1] - sp.rows[0], p, steps_per_chain, material=material,
                        noise_seed=noise_seed, sigma=sigma, dt=dt, mesh=sp.window,
                        centre=(sp.nx / 2.0, sp.ny / 2.0), cell_offset=sp.cell_offset)
    loc = local_elastic_setup(win, sp.local_window)
    loc.local_mesh = sp.local
    return loc


def global_dt(p: int, material, n_cells: int) -> float:
    """dt = 0.1 h / (c_p,max (2p+1)) over all cells (dg.elastic_setup's rule)."""
    if material == "homogeneous":
        cp = 2.0
    else:
        kind, seed = material
        rng = np.random.default_rng(seed)
        cp, left = 0.0, n_cells
        while left:
            n = min(left, 1 << 22)
            m = rng.uniform(1.0, 2.0, size=(n, 3))
            cp = max(cp, float(np.sqrt((m[:, 1] + 2 * m[:, 2]) / m[:, 0]).max()))
            left -= n
    return 0.1 * 1.0 / (cp * (2 * p + 1))


# ---- multi-GPU bench path (bench.py, torchrun N > 1) --------------------------------

def bench_partitioned(args, w, rank, world, local, bench):
    """Strong scaling of a BASELINE workload over ``world`` strips: each rank
    generates and inspects only its strip (mixed SHARED mode), then per chain:
    ``begin()`` (pack + grouped NCCL send/recv of the exchanged rows), core
    tiles, ``end()`` (wait + unpack), boundary tiles.  Time = max over ranks;
    value = DoF updates of the owned cells of all ranks / that time."""
    import json

    import torch

    from .dg import constant_datasets, elastic_problem
    from .distributed import HaloExchange, exchanged_from_chain
    from .executor import TiledRunner
    from .inspector import ExecMode, inspect_chain
    from .workloads import roofline_bytes

    depth = 5 * w.T                       # halo depth >= loops per chain (chain.py:227-229)
    t0 = time.perf_counter()
    sp = strip_partition(w.nx, w.ny, world, depth, rank)
    loc = strip_elastic_setup(sp, w.p, w.T, w.material, w.noise_seed, w.sigma,
                              global_dt(w.p, w.material, w.cells))
    pb = elastic_problem(loc, depth=len(loc.loops))
    pb.install_params()
    setup_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    ts = w.ts_strips or w.ts  # strips keep the generator's row-major numbering
    sched = inspect_chain(pb.chain, ts, ExecMode.SHARED)
    inspect_s = time.perf_counter() - t0
    const = constant_datasets(pb.chain, pb.bindings)
    exchanged = tuple(n for n in exchanged_from_chain(pb.chain, pb.bindings) if n not in const)
    ex = HaloExchange(sp.local, pb.datasets, exchanged)
    runner = TiledRunner(sched, pb.chain, pb.bindings, pb.datasets, pb.registry)
    chains = w.chains_per_step
    launches = [0]

    def step():
        for _ in range(chains):
            launches[0] += runner.with_exchange(ex)

    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    bench.barrier(world)
    launches[0] = 0
    with bench.ClockSampler(local) as clk:
        dev_s = bench.timed(step, args.steps, flush, stream)
        bench.barrier(world)
    dev_s = bench.max_over_ranks(dev_s, world)
    owned = sp.local.sizes[CELLS].owned_total
    nd5 = 5 * (w.p + 1) * (w.p + 2) // 2
    total_dofs = bench.sum_over_ranks(owned * nd5, world)
    updates = total_dofs * w.T * chains * args.steps
    value = updates / dev_s
    # roofline: 8(d) bytes of every rank's owned cells (local problem scaled)
    b_local = roofline_bytes(loc, w.heterogeneous) * owned / loc.spaces[CELLS].total
    b_all = bench.sum_over_ranks(b_local, world)
    peak, peak_src = bench.measured_peaks()
    achieved = b_all * chains * args.steps / dev_s / 1e9
    e2e = None
    if not args.no_e2e:
        host = {n: torch.empty(pb.datasets[n].values.numel(), dtype=torch.float64,
                               pin_memory=True) for n in ("u", "s")}
        for n in host:
            host[n].copy_(pb.datasets[n].values)
        h2d = sum(h.numel() * 8 for h in host.values())
        torch.cuda.synchronize()
        bench.barrier(world)

        def e2e_step():
            for n in host:
                pb.datasets[n].values.copy_(host[n], non_blocking=True)
            step()
            for n in host:
                host[n].copy_(pb.datasets[n].values, non_blocking=True)

        n_e2e = max(1, min(args.steps, 3))
        e2e_s = bench.max_over_ranks(bench.timed(e2e_step, n_e2e, flush, stream), world)
        e2e = {"value": total_dofs * w.T * chains * n_e2e / e2e_s, "unit": "DoF-updates/s",
               "h2d_bytes_per_step": int(bench.sum_over_ranks(h2d, world)),
               "d2h_bytes_per_step": int(bench.sum_over_ranks(h2d, world))}
    if rank == 0:
        print(json.dumps({
            "metric": bench.METRIC, "value": value, "unit": "DoF-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": w.text + f"; {world} contiguous strips, halo depth {depth}",
                       "p": w.p, "cells": w.cells, "dofs": w.dofs, "timesteps_per_chain": w.T,
                       "chains_per_step": chains, "seed_tile": ts, "renumber": "none",
                       "mode": "shared (mixed)",
                       "rank0_cells_local": loc.spaces[CELLS].total, "rank0_cells_owned": owned,
                       "colors_rank0": len(sched.color_order), "setup_s": round(setup_s, 1),
                       "inspect_s": round(inspect_s, 3),
                       "halo_exchange": "NCCL batch_isend_irecv once per chain"
                       if world > 1 else "none (1 rank)",
                       "bytes_exchanged_per_chain_rank0": ex.bytes_exchanged //
                       max(ex.exchange_count, 1),
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"partitioned x{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world,
                         "unit": "GB/s", "frac": achieved / (peak * world), "traffic": None,
                         "peak_source": peak_src + f" x {world} GPUs"},
            "cpu_baseline": None, "e2e": e2e,
            "gpu_launches": launches[0],
            "clocks": clk.summary(),
        }), flush=True)
