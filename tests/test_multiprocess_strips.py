"""The partitioned elastic chain on real processes (one rank per process).

* CPU, gloo, world 2 and 3: each rank builds only its strip
  (strips.strip_partition + strip_elastic_setup), poisons its halo rows and
  runs one HaloExchange (the product's begin()/end() protocol, grouped
  point-to-point); every halo row a neighbour owns must then hold the
  global problem's value (reference distsim.py:48-81 semantics).
* GPU (marked gpu), 2 processes on cuda:0, gloo with host staging: the full
  chain per rank -- begin(), core tiles (lt_execute), end(), boundary tiles
  -- for 3 chains with poisoned halos, gathered owned rows against the
  serial GPU untiled executor at 1e-12 (reference distsim.py:163-190
  gather semantics, tests/test_distsim.py:58-67).  Each process's kernels
  wait only on their own tiles; the exchange is host-synchronous.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

NX, NY, P, T = 6, 40, 1, 1


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def cpu_pack(values, k, rows, out):
    out.copy_(values.view(-1, k)[rows.long()].reshape(-1))


def cpu_unpack(values, k, rows, src):
    values.view(-1, k)[rows.long()] = src.view(-1, k)


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def _cpu_worker(rank, world, port, q, nx, ny, p, t):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from types import SimpleNamespace

        from paper_1708_03183_b200.dg import elastic_setup
        from paper_1708_03183_b200.distributed import HaloExchange
        from paper_1708_03183_b200.strips import global_dt, strip_elastic_setup, strip_partition
        depth = 5 * t
        mat = ("uniform", 2)
        sp = strip_partition(nx, ny, world, depth, rank)
        loc = strip_elastic_setup(sp, p, t, mat, 1, 4.0, global_dt(p, mat, 2 * nx * ny))
        glob = elastic_setup(nx, ny, p, t, material=mat, noise_seed=1, sigma=4.0)
        lm = sp.local
        gids = lm.global_ids["cells"]
        owned = lm.sizes["cells"].owned_total
        ds = {}
        for n in ("u", "s", "ru", "rs"):
            k = loc.vpe[n]
            v = torch.from_numpy(loc.data[n].copy())
            v.view(-1, k)[owned:] = 1e30
            ds[n] = SimpleNamespace(values=v, space=loc.spaces["cells"], values_per_element=k)
        ex = HaloExchange(lm, ds, ("u", "s", "ru", "rs"), pack=cpu_pack, unpack=cpu_unpack)
        ex.begin()
        ex.end()
        halo = set()
        for (space, nbr), table in lm.exchange_table.items():
            if space == "cells":
                halo.update(table[table[:, 0] >= owned, 0].tolist())
        rows = np.array(sorted(halo), dtype=np.int64)
        ok = len(rows) > 0
        for n in ("u", "s", "ru", "rs"):
            k = loc.vpe[n]
            want = glob.data[n].reshape(-1, k)[gids]
            got = ds[n].values.numpy().reshape(-1, k)
            ok &= np.array_equal(got[:owned], want[:owned]) and np.array_equal(got[rows],
                                                                                want[rows])
        q.put((rank, bool(ok), ex.bytes_exchanged))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strip_halo_exchange_over_gloo(world):
    for rank, ok, moved in _spawn(_cpu_worker, world, NX, NY, P, T):
        assert ok, f"rank {rank}: halo rows differ from the global problem"
        assert moved > 0


def _gpu_worker(rank, world, port, q, nx, ny, p, t, n_chains):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1708_03183_b200 as lt
        from paper_1708_03183_b200.dg import constant_datasets, elastic_problem
        from paper_1708_03183_b200.distributed import HaloExchange, exchanged_from_chain
        from paper_1708_03183_b200.executor import TiledRunner
        from paper_1708_03183_b200.strips import global_dt, strip_elastic_setup, strip_partition
        depth = 5 * t
        mat = ("uniform", 3)
        sp = strip_partition(nx, ny, world, depth, rank)
        loc = strip_elastic_setup(sp, p, t, mat, 1, 4.0, global_dt(p, mat, 2 * nx * ny))
        pb = elastic_problem(loc, depth=len(loc.loops))
        pb.install_params()
        owned = sp.local.sizes["cells"].owned_total
        for n in ("u", "s", "ru", "rs"):
            pb.datasets[n].values.view(-1, loc.vpe[n])[owned:] = 1e30
        sched = lt.inspect_chain(pb.chain, 12, lt.ExecMode.SHARED)
        const = constant_datasets(pb.chain, pb.bindings)
        exch = tuple(n for n in exchanged_from_chain(pb.chain, pb.bindings) if n not in const)
        ex = HaloExchange(sp.local, pb.datasets, exch)
        assert ex.staging
        runner = TiledRunner(sched, pb.chain, pb.bindings, pb.datasets, pb.registry)
        for _ in range(n_chains):
            runner.with_exchange(ex)
        torch.cuda.synchronize()
        gids = sp.local.global_ids["cells"][:owned]
        q.put((rank, gids, {n: pb.datasets[n].numpy().reshape(-1, loc.vpe[n])[:owned]
                            for n in ("u", "s")}, runner.executor))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_partitioned_chain_two_processes_matches_serial_untiled():
    from paper_1708_03183_b200.dg import elastic_problem, elastic_setup
    nx, ny, p, t, n_chains = 10, 36, 2, 2, 3
    glob = elastic_problem(elastic_setup(nx, ny, p, t, material=("uniform", 3), noise_seed=1,
                                         sigma=4.0))
    glob.run_untiled(n_chains=n_chains)
    ref = {n: glob.datasets[n].numpy().reshape(-1, glob.setup.vpe[n]) for n in ("u", "s")}
    seen = np.zeros(2 * nx * ny, dtype=bool)
    for rank, gids, vals, executor in _spawn(_gpu_worker, 2, nx, ny, p, t, n_chains):
        assert executor == "dataflow"
        seen[gids] = True
        for n in ("u", "s"):
            err = np.max(np.abs(vals[n] - ref[n][gids])) / np.max(np.abs(ref[n]))
            assert err <= 1e-12, (rank, n, err)
    assert seen.all()
