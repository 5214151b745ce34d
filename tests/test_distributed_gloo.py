"""Multi-process halo exchange host logic over gloo (CPU, world_size 2 and 3).

The product packs/unpacks with CUDA kernels (lt_halo_pack/unpack); on CPU the
test injects torch index ops so the exchange plan, grouped point-to-point
traffic and begin()/end() protocol are exercised without a GPU.
"""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1708_03183_b200 as lt
from paper_1708_03183_b200.distributed import HaloExchange
from paper_1708_03183_b200.partition import partition_for_ranks


def cpu_pack(values, k, rows, out):
    out.copy_(values.view(-1, k)[rows.long()].reshape(-1))


def cpu_unpack(values, k, rows, src):
    values.view(-1, k)[rows.long()] = src.view(-1, k)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, depth, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = lt.generate_rect_mesh(*dims)
        lm = partition_for_ranks(mesh, world, depth)[rank]
        rng = np.random.default_rng(7)
        glob = {"c": rng.random(mesh.num_cells * 3), "v": rng.random(mesh.num_vertices),
                "e": rng.random(mesh.num_edges * 2)}
        spaces = lm.spaces()
        ds = {}
        for name, space, k in (("c", "cells", 3), ("v", "verts", 1), ("e", "edges", 2)):
            gids = lm.global_ids[space]
            vals = torch.from_numpy(glob[name].reshape(-1, k)[gids].ravel().copy())
            owned = lm.sizes[space].owned_total
            vals[owned * k:] = -1.0  # poisoned halo
            ds[name] = SimpleNamespace(values=vals, space=spaces[space], values_per_element=k)
        ex = HaloExchange(lm, ds, ("c", "v", "e"), pack=cpu_pack, unpack=cpu_unpack)
        ex.begin()
        ex.end()
        ok = True
        for name, space, k in (("c", "cells", 3), ("v", "verts", 1), ("e", "edges", 2)):
            gids = lm.global_ids[space]
            want = glob[name].reshape(-1, k)[gids]
            got = ds[name].values.numpy().reshape(-1, k)
            # every halo row that some neighbour owns is now the owner's value
            halo = set()
            for (sp, nbr), table in lm.exchange_table.items():
                if sp == space:
                    halo.update(table[table[:, 0] >= lm.sizes[space].owned_total, 0].tolist())
            rows = np.array(sorted(halo), dtype=np.int64)
            owned = lm.sizes[space].owned_total
            ok &= np.array_equal(got[:owned], want[:owned])
            ok &= (len(rows) == 0) or np.array_equal(got[rows], want[rows])
        queue.put((rank, bool(ok), ex.exchange_count, ex.bytes_exchanged))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,depth", [(2, (8, 6), 2), (3, (9, 6), 3)])
def test_halo_exchange_over_gloo(world, dims, depth):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, depth, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, count, moved in results:
        assert ok, f"rank {rank}: halo rows differ from owner values"
        assert count == 1 and moved > 0
