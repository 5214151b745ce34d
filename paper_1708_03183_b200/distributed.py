"""Distributed-memory execution: halo exchange once per tiled chain.

Mirrors the reference ``distsim.py`` (``pkg/src/looptile/distsim.py:26-244``):
one exchange serves a whole chain execution -- ``begin()`` before the core
phase snapshots every owner's rows, ``end()`` between the core and boundary
phases commits them into the local exec/non-exec slots (Alg. 2 of the paper).
Core tiles therefore run against stale halos, exactly their contract.

Two transports behind the same ``begin()/end()/bytes_exchanged`` protocol:

* ``HaloEndpoint`` -- N virtual ranks in one process on one GPU (the
  reference's simulation, with device-side pack/unpack kernels); used by
  ``run_distributed`` and the single-GPU tests.
* ``HaloExchange`` -- one process per GPU over ``torch.distributed``: per
  neighbour, one contiguous send buffer packed by ``lt_halo_pack`` (all
  exchanged datasets of all spaces), grouped ``isend``/``irecv`` (NCCL over
  NVLink on B200s) posted in ``begin()`` so the transfer overlaps the core
  tiles, and ``lt_halo_unpack`` in ``end()``.

Exchanged datasets follow the reference rule (``distsim.py:152-160``): every
dataset a fused loop reads or increments.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .chain import AccessMode, LoopChain
from .errors import PartitionBugError


def _device_rows(rows: np.ndarray, device):
    import torch
    return torch.from_numpy(np.ascontiguousarray(rows, dtype=np.int32)).to(device)


def _gpu_pack(values, vpe, rows, out):
    from . import _lib
    _lib.halo_pack(values, vpe, rows, out)


def _gpu_unpack(values, vpe, rows, src):
    from . import _lib
    _lib.halo_unpack(values, vpe, rows, src)


class HaloEndpoint:
    """One virtual rank's side of the exchange (reference ``distsim.py:26-81``).

    ``begin()`` copies every neighbour-owned row this rank holds from the
    owner's device dataset into staging buffers; ``end()`` commits them.  The
    two calls strictly alternate.
    """

    def __init__(self, local_mesh, datasets: dict, exchanged: tuple[str, ...],
                 pack=_gpu_pack, unpack=_gpu_unpack):
        self.local_mesh = local_mesh
        self.rank = local_mesh.rank
        self.datasets = datasets
        self.exchanged = exchanged
        self.peers: dict[int, "HaloEndpoint"] = {}
        self.exchange_count = 0
        self.bytes_exchanged = 0
        self._staged = None
        self._pack, self._unpack = pack, unpack
        self._plan = None

    def link(self, endpoints: list["HaloEndpoint"]) -> None:
        self.peers = {e.rank: e for e in endpoints if e.rank != self.rank}

    def _build_plan(self):
        plan = []
        for (space, nbr), table in sorted(self.local_mesh.exchange_table.items()):
            owned_here = self.local_mesh.sizes[space].owned_total
            incoming = table[table[:, 0] >= owned_here]  # rows the neighbour owns
            if not len(incoming):
                continue
            for name in self.exchanged:
                ds = self.datasets[name]
                if ds.space.name != space:
                    continue
                dev = ds.values.device
                plan.append((name, nbr, ds.values_per_element,
                             _device_rows(incoming[:, 1], dev), _device_rows(incoming[:, 0], dev)))
        self._plan = plan

    def begin(self) -> None:
        import torch
        if self._staged is not None:
            raise PartitionBugError("begin() called twice without end()")
        if self._plan is None:
            self._build_plan()
        staged = []
        for name, nbr, k, src_rows, dst_rows in self._plan:
            src = self.peers[nbr].datasets[name].values
            buf = torch.empty(src_rows.numel() * k, dtype=src.dtype, device=src.device)
            self._pack(src, k, src_rows, buf)
            staged.append((name, k, dst_rows, buf))
        self._staged = staged

    def end(self) -> None:
        if self._staged is None:
            raise PartitionBugError("end() called without begin()")
        moved = 0
        for name, k, dst_rows, buf in self._staged:
            self._unpack(self.datasets[name].values, k, dst_rows, buf)
            moved += buf.numel() * buf.element_size()
        self._staged = None
        self.exchange_count += 1
        self.bytes_exchanged += moved


class _PreStaged:
    """Adapter for execute_schedule when staging happened chain-wide (``distsim.py:112-126``)."""

    def __init__(self, endpoint):
        self.endpoint = endpoint

    def begin(self) -> None:
        pass

    def end(self) -> None:
        self.endpoint.end()

    @property
    def bytes_exchanged(self) -> int:
        return self.endpoint.bytes_exchanged


def check_exchange_symmetry(endpoints) -> None:
    """Tables of each rank pair list identical global ids in identical order."""
    by_rank = {e.rank: e for e in endpoints}
    for e in endpoints:
        for (space, nbr), table in e.local_mesh.exchange_table.items():
            peer = by_rank[nbr]
            mirror = peer.local_mesh.exchange_table.get((space, e.rank))
            if mirror is None or len(mirror) != len(table):
                raise PartitionBugError(
                    f"asymmetric exchange table for {space} between ranks {e.rank} and {nbr}")
            here = e.local_mesh.global_ids[space][table[:, 0]]
            there = peer.local_mesh.global_ids[space][mirror[:, 0]]
            if not np.array_equal(here, there):
                raise PartitionBugError(
                    f"exchange tables for {space} pair different global ids "
                    f"between ranks {e.rank} and {nbr}")


def halo_exchange(endpoints) -> None:
    """One synchronous exchange: every owner's rows land in all halo copies."""
    check_exchange_symmetry(endpoints)
    for e in endpoints:
        e.begin()
    for e in endpoints:
        e.end()


def exchanged_dataset_names(problem_or_loops) -> tuple[str, ...]:
    """Datasets any fused loop reads or increments travel in the exchange."""
    loops = getattr(problem_or_loops, "loops", problem_or_loops)
    names = []
    for spec in loops:
        for access in spec.accesses:
            if access.mode in (AccessMode.READ, AccessMode.INC) and access.dataset not in names:
                names.append(access.dataset)
    return tuple(names)


def exchanged_from_chain(chain: LoopChain, bindings) -> tuple[str, ...]:
    names = []
    for loop, b in zip(chain.loops, bindings):
        for d, n in zip(loop.descriptors, b.args):
            if d.mode in (AccessMode.READ, AccessMode.INC) and n not in names:
                names.append(n)
    return tuple(names)


class HaloExchange:
    """Multi-process halo exchange over ``torch.distributed`` (one rank per GPU).

    Same protocol as :class:`HaloEndpoint`.  Per neighbour, the rows this rank
    owns and the neighbour holds are packed (all exchanged datasets, in
    table order) into one contiguous send buffer; rows the neighbour owns are
    received into one buffer and unpacked.  ``begin()`` posts the grouped
    point-to-point operations (NCCL over NVLink between B200s) so they
    overlap the core tiles; ``end()`` waits and unpacks.
    """

    def __init__(self, local_mesh, datasets: dict, exchanged: tuple[str, ...], group=None,
                 pack=_gpu_pack, unpack=_gpu_unpack, staging: bool | None = None):
        import torch
        import torch.distributed as dist
        self.local_mesh = local_mesh
        self.rank = local_mesh.rank
        self.datasets = datasets
        self.exchanged = exchanged
        self.group = group
        self.exchange_count = 0
        self.bytes_exchanged = 0
        self._pack, self._unpack = pack, unpack
        self._work = None
        self.neighbours = local_mesh.neighbors()
        some = next(iter(datasets.values())).values
        dev, dtype = some.device, some.dtype
        self._send, self._recv = {}, {}
        for nbr in self.neighbours:
            send_parts, recv_parts = [], []
            n_send = n_recv = 0
            for name in exchanged:
                ds = datasets[name]
                table = local_mesh.exchange_table.get((ds.space.name, nbr))
                if table is None:
                    continue
                owned_here = local_mesh.sizes[ds.space.name].owned_total
                mine = table[table[:, 0] < owned_here, 0]
                theirs = table[table[:, 0] >= owned_here, 0]
                k = ds.values_per_element
                if len(mine):
                    send_parts.append((name, k, _device_rows(mine, dev), n_send))
                    n_send += len(mine) * k
                if len(theirs):
                    recv_parts.append((name, k, _device_rows(theirs, dev), n_recv))
                    n_recv += len(theirs) * k
            self._send[nbr] = (send_parts, torch.empty(max(n_send, 1), dtype=dtype, device=dev),
                               n_send)
            self._recv[nbr] = (recv_parts, torch.empty(max(n_recv, 1), dtype=dtype, device=dev),
                               n_recv)
        # a transport without device buffers (gloo) moves the packed rows
        # through pinned host buffers: device pack -> host -> send, receive ->
        # host -> device unpack (NCCL sends the device buffers directly)
        if staging is None:
            staging = dev.type == "cuda" and dist.is_initialized() and \
                dist.get_backend(group) == "gloo"
        self.staging = bool(staging)
        self._host = {}
        if self.staging:
            for nbr in self.neighbours:
                self._host[nbr] = (
                    torch.empty(max(self._send[nbr][2], 1), dtype=dtype, pin_memory=True),
                    torch.empty(max(self._recv[nbr][2], 1), dtype=dtype, pin_memory=True))

    def begin(self) -> None:
        import torch.distributed as dist
        if self._work is not None:
            raise PartitionBugError("begin() called twice without end()")
        ops = []
        for nbr in self.neighbours:
            parts, buf, n = self._send[nbr]
            for name, k, rows, off in parts:
                self._pack(self.datasets[name].values, k, rows,
                           buf[off:off + rows.numel() * k])
            if n and self.staging:
                host = self._host[nbr][0]
                host[:n].copy_(buf[:n])      # synchronous: the packed rows are final
                ops.append(dist.P2POp(dist.isend, host[:n], nbr, group=self.group))
            elif n:
                ops.append(dist.P2POp(dist.isend, buf[:n], nbr, group=self.group))
        for nbr in self.neighbours:
            _, buf, n = self._recv[nbr]
            if n:
                dst = self._host[nbr][1][:n] if self.staging else buf[:n]
                ops.append(dist.P2POp(dist.irecv, dst, nbr, group=self.group))
        self._work = dist.batch_isend_irecv(ops) if ops else []

    def end(self) -> None:
        if self._work is None:
            raise PartitionBugError("end() called without begin()")
        for w in self._work:
            w.wait()
        moved = 0
        for nbr in self.neighbours:
            parts, buf, n = self._recv[nbr]
            if n and self.staging:
                buf[:n].copy_(self._host[nbr][1][:n])  # host buffer is reused next chain
            for name, k, rows, off in parts:
                self._unpack(self.datasets[name].values, k, rows,
                             buf[off:off + rows.numel() * k])
            moved += n * buf.element_size()
        self._work = None
        self.exchange_count += 1
        self.bytes_exchanged += moved


@dataclass
class VirtualRank:
    rank: int
    local_mesh: object
    chain: LoopChain
    datasets: dict
    bindings: tuple
    schedule: object
    endpoint: HaloEndpoint
    report: object = None


@dataclass
class DistributedResult:
    datasets: dict
    ranks: list
    reports: list = field(default_factory=list)

    @property
    def exchange_counts(self) -> list[int]:
        return [r.endpoint.exchange_count for r in self.ranks]


def gather(totals: dict, specs, ranks) -> dict:
    """Owned rows of every rank into global arrays (``distsim.py:163-190``).

    ``totals``: space -> global element count; ``specs``: (name, space, vpe).
    """
    out = {}
    for name, space, k in specs:
        n = totals[space]
        values = np.full(n * k, np.nan)
        seen = np.zeros(n, dtype=bool)
        for vr in ranks:
            owned = vr.local_mesh.sizes[space].owned_total
            gids = vr.local_mesh.global_ids[space][:owned]
            if np.any(seen[gids]):
                raise PartitionBugError(f"{space} ownership overlaps while gathering {name!r}")
            seen[gids] = True
            local = vr.datasets[name].numpy().reshape(-1, k)[:owned]
            values.reshape(-1, k)[gids] = local
        if not seen.all():
            raise PartitionBugError(f"{space} elements without owner while gathering {name!r}")
        out[name] = values
    return out


def run_distributed(mesh, problem, nranks: int, ts: int, depth: int, registry,
                    use_local_maps: bool = False, poison_halo: bool = False,
                    initial: dict | None = None, mode=None) -> DistributedResult:
    """Partition, inspect and execute on N virtual ranks sharing one GPU, then gather.

    Reference ``distsim.py:193-244``.  ``mode`` defaults to the reference's
    ExecMode.DISTRIBUTED; ExecMode.SHARED gives the mixed mode (colour
    classes per rank) the GPU executor wants.
    """
    from .executor import execute_schedule
    from .inspector import ExecMode, inspect_chain
    from .partition import partition_for_ranks
    from .problems import local_setup
    mode = mode or ExecMode.DISTRIBUTED
    local_meshes = partition_for_ranks(mesh, nranks, depth)
    exchanged = exchanged_dataset_names(problem)
    totals = {"cells": mesh.num_cells, "edges": mesh.num_edges, "verts": mesh.num_vertices}
    ranks, endpoints = [], []
    for lm in local_meshes:
        chain, datasets, bindings = local_setup(lm, problem, depth, global_totals=totals)
        if initial is not None:
            for name, ds in datasets.items():
                k = ds.values_per_element
                gids = lm.global_ids[ds.space.name]
                ds.values.copy_(ds.values.new_tensor(initial[name].reshape(-1, k)[gids].ravel()))
        if poison_halo:
            for ds in datasets.values():
                owned = lm.sizes[ds.space.name].owned_total
                ds.values[owned * ds.values_per_element:] = 1e30
        schedule = inspect_chain(chain, ts, mode)
        ep = HaloEndpoint(lm, datasets, exchanged)
        endpoints.append(ep)
        ranks.append(VirtualRank(lm.rank, lm, chain, datasets, bindings, schedule, ep))
    for e in endpoints:
        e.link(endpoints)
    check_exchange_symmetry(endpoints)
    for e in endpoints:
        e.begin()  # snapshot owners before anything runs
    reports = []
    for vr in ranks:
        vr.report = execute_schedule(vr.schedule, vr.chain, vr.bindings, vr.datasets, registry,
                                     exchange=_PreStaged(vr.endpoint),
                                     use_local_maps=use_local_maps)
        reports.append(vr.report)
    specs = [(d.name, d.space, d.values_per_element) for d in problem.datasets]
    return DistributedResult(gather(totals, specs, ranks), ranks, reports)
