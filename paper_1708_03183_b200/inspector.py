"""Run-time inspection on the GPU: build a legal sparse-tiling schedule.

Same entry point and result type as the reference (``inspector.py:433``:
``inspect_chain(chain, ts, mode) -> Schedule``).  The work runs in
``libltcuda.so`` (``lt_inspect``): seed partition, stable counting sort into
iteration lists, CSR inverse maps, projection and tiling kernels with a
device hash set for conflict pairs, and the recolouring loop, with greedy
colouring on the host.  The resulting tile membership, colours, round count
and local maps are bit-identical to the reference's (pinned by
``tests/golden``), so ``Schedule.serialize()`` reproduces the reference's
``schedule-v1`` bytes.

The ``Schedule`` keeps the device-resident schedule; ``tiles`` materialises
host ``Tile`` objects lazily (only tests, serialisation and tooling need
them).  A ``Schedule`` constructed from explicit tiles (e.g. a mutated or
reference-produced one) is uploaded with ``lt_schedule_import`` on first
execution.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from .chain import IterationSpace, LoopChain, MeshMap, Region

NO_TILE = -1


class ExecMode(enum.Enum):
    SEQUENTIAL = "sequential"
    SHARED = "shared"
    DISTRIBUTED = "distributed"

    @classmethod
    def parse(cls, token: str) -> "ExecMode":
        for mode in cls:
            if token == mode.value:
                return mode
        raise ValueError(f"unknown execution mode {token!r}")

    @property
    def code(self) -> int:
        return {"sequential": 0, "shared": 1, "distributed": 2}[self.value]


@dataclass(eq=False)
class Tile:
    """An atomically executed unit: one iteration list per loop, plus a color."""

    id: int
    region: Region
    color: int = -1
    iteration_lists: dict[int, np.ndarray] = field(default_factory=dict)
    local_maps: dict[tuple[int, str], np.ndarray] = field(default_factory=dict)

    def size(self, loop_index: int) -> int:
        lst = self.iteration_lists.get(loop_index)
        return 0 if lst is None else len(lst)


@dataclass
class TilingFunction:
    """Per-element tile assignment for one loop."""

    loop_index: int
    assignment: np.ndarray


@dataclass
class Projection:
    """Per-element record of the maximum-color tile that touched the element."""

    space: IterationSpace
    assignment: np.ndarray


@dataclass
class ConflictMatrix:
    """Symmetric, irreflexive relation over tile ids that grew adjacent."""

    pairs: set[tuple[int, int]] = field(default_factory=set)

    def add(self, a: int, b: int) -> None:
        if a != b:
            self.pairs.add((min(a, b), max(a, b)))

    def has_conflicts(self) -> bool:
        return bool(self.pairs)


@dataclass
class InspectionStats:
    partition_s: float = 0.0
    coloring_s: float = 0.0
    projection_tiling_s: float = 0.0
    local_maps_s: float = 0.0
    total_s: float = 0.0

    def dominant_phase(self) -> tuple[str, float]:
        phases = {
            "partition": self.partition_s,
            "coloring": self.coloring_s,
            "projection_tiling": self.projection_tiling_s,
            "local_maps": self.local_maps_s,
        }
        span = sum(phases.values()) or 1.0
        name = max(phases, key=phases.get)
        return name, phases[name] / span


class Schedule:
    """Inspector output: populated tiles plus the color execution order.

    Reference ``inspector.py:104-179``.  Either wraps a device schedule
    (``_handle``, from :func:`inspect_chain`) or holds explicit ``tiles``.
    """

    def __init__(self, mode: ExecMode, fingerprint: str, n_loops: int,
                 tiles=None, recolor_rounds: int = 1,
                 stats: InspectionStats | None = None, *, _handle=None, _chain=None):
        self.mode = mode
        self.fingerprint = fingerprint
        self.n_loops = n_loops
        self.recolor_rounds = recolor_rounds
        self.stats = stats or InspectionStats()
        self._handle = _handle
        self._chain = _chain
        self._tiles = tuple(tiles) if tiles is not None else None
        self._synced = None  # (colors, regions, list ids) the handle was built from
        if _handle is not None:
            info = _handle.info()
            self._n_tiles = info.n_tiles
            self._n_colors = info.n_colors
            colors, regions = _handle.tiles(info.n_tiles)
            self._colors, self._regions = colors, regions
        else:
            self._n_tiles = len(self._tiles)

    # -- lazy host view -------------------------------------------------------------
    @property
    def tiles(self) -> tuple[Tile, ...]:
        if self._tiles is None:
            self._tiles = self._materialize()
            self._synced = self._tile_state()
        return self._tiles

    def _materialize(self) -> tuple[Tile, ...]:
        h, chain = self._handle, self._chain
        tiles = [Tile(id=t, region=Region(int(self._regions[t])), color=int(self._colors[t]))
                 for t in range(self._n_tiles)]
        for j, loop in enumerate(chain.loops):
            off, el = h.lists(j, self._n_tiles, loop.space.total)
            el = el.astype(np.int64)
            for t in tiles:
                t.iteration_lists[j] = el[off[t.id]:off[t.id + 1]].copy()
            done = []
            for d in loop.descriptors:
                if d.is_direct or d.map.name in done:
                    continue
                done.append(d.map.name)
                mi = h.chain_desc.map_index[id(d.map)]
                flat = h.local_map(j, mi, loop.space.total * d.map.arity).astype(np.int64)
                a = d.map.arity
                for t in tiles:
                    t.local_maps[(j, d.map.name)] = flat[off[t.id] * a:off[t.id + 1] * a].copy()
        return tuple(tiles)

    def _tile_state(self):
        return tuple((t.id, int(t.region), t.color,
                      tuple(id(v) for v in t.iteration_lists.values())) for t in self._tiles)

    def device_handle(self, chain: LoopChain):
        """The device schedule, (re)uploading host tiles if they were edited."""
        from . import _lib
        if self._handle is not None and (self._tiles is None
                                         or self._tile_state() == self._synced):
            return self._handle
        tiles = self.tiles
        lists = []
        for j, loop in enumerate(chain.loops):
            n = loop.space.total
            sizes = np.array([t.size(j) for t in tiles], dtype=np.int64)
            off = np.zeros(len(tiles) + 1, dtype=np.int64)
            np.cumsum(sizes, out=off[1:])
            if off[-1] != n:
                from .errors import StaleScheduleError, ExecutionError
                raise ExecutionError(f"loop {j}: tiles cover {off[-1]} of {n} elements")
            el = (np.concatenate([t.iteration_lists.get(j, np.empty(0, np.int64))
                                  for t in tiles]) if tiles else np.empty(0, np.int64))
            lists.append((off, el))
        self._handle = _lib.import_schedule(
            chain, self.mode.code, [t.color for t in tiles], [int(t.region) for t in tiles],
            self.recolor_rounds, lists)
        self._chain = chain
        self._colors = np.array([t.color for t in tiles], dtype=np.int32)
        self._regions = np.array([int(t.region) for t in tiles], dtype=np.int32)
        self._synced = self._tile_state()
        return self._handle

    # -- reference API -----------------------------------------------------------------
    @property
    def color_order(self) -> list[int]:
        if self._tiles is None:
            return sorted({int(c) for c in self._colors})
        return sorted({t.color for t in self._tiles})

    @property
    def nonexec_tile(self) -> Tile:
        return self.tiles[-1]

    def executable_tiles(self) -> list[Tile]:
        return [t for t in self.tiles if t.region is not Region.NONEXEC]

    def tiles_in_region(self, region: Region) -> list[Tile]:
        return [t for t in self.tiles if t.region is region]

    def tile_colors(self) -> tuple[np.ndarray, np.ndarray]:
        """(colors, regions) per tile id without materialising the lists."""
        if self._tiles is None:
            return self._colors, self._regions
        return (np.array([t.color for t in self._tiles]),
                np.array([int(t.region) for t in self._tiles]))

    def tile_of(self, loop_index: int, n_elements: int) -> np.ndarray:
        out = np.full(n_elements, NO_TILE, dtype=np.int64)
        for t in self.tiles:
            lst = t.iteration_lists.get(loop_index)
            if lst is not None:
                out[lst] = t.id
        return out

    def serialize(self) -> bytes:
        """``schedule-v1`` text, byte-compatible with reference ``inspector.py:139-155``."""
        lines = [
            "schedule-v1",
            f"mode={self.mode.value}",
            f"fingerprint={self.fingerprint}",
            f"loops={self.n_loops}",
            f"rounds={self.recolor_rounds}",
            f"colors={','.join(map(str, self.color_order))}",
        ]
        for t in self.tiles:
            lines.append(f"tile id={t.id} region={t.region.name.lower()} color={t.color}")
            for j in sorted(t.iteration_lists):
                lines.append(f"  list {j}=" + ",".join(map(str, t.iteration_lists[j].tolist())))
            for (j, name) in sorted(t.local_maps):
                lines.append(f"  lmap {j} {name}=" +
                             ",".join(map(str, t.local_maps[(j, name)].tolist())))
        return ("\n".join(lines) + "\n").encode()

    @classmethod
    def deserialize(cls, data: bytes) -> "Schedule":
        """Parse ``schedule-v1`` bytes (the on-disk inspection cache format)."""
        lines = data.decode().split("\n")
        if not lines or lines[0] != "schedule-v1":
            raise ValueError("not a schedule-v1 document")
        head = dict(ln.split("=", 1) for ln in lines[1:6])
        tiles = []
        for ln in lines[6:]:
            if ln.startswith("tile "):
                kv = dict(x.split("=") for x in ln.split()[1:])
                tiles.append(Tile(int(kv["id"]), Region[kv["region"].upper()], int(kv["color"])))
            elif ln.startswith("  list "):
                key, _, vals = ln[7:].partition("=")
                tiles[-1].iteration_lists[int(key)] = np.array(
                    [int(v) for v in vals.split(",")] if vals else [], dtype=np.int64)
            elif ln.startswith("  lmap "):
                key, _, vals = ln[7:].partition("=")
                j, name = key.split(" ", 1)
                tiles[-1].local_maps[(int(j), name)] = np.array(
                    [int(v) for v in vals.split(",")] if vals else [], dtype=np.int64)
        return cls(ExecMode.parse(head["mode"]), head["fingerprint"], int(head["loops"]), tiles,
                   int(head["rounds"]))

    def summary(self) -> str:
        by_region = {r: len(self.tiles_in_region(r)) for r in Region}
        lines = [
            f"tiles: {len(self.tiles)} "
            f"(core {by_region[Region.CORE]}, boundary {by_region[Region.BOUNDARY]}, "
            f"non-exec {by_region[Region.NONEXEC]})",
            f"colors: {len(self.color_order)}",
            f"recolor rounds: {self.recolor_rounds}",
        ]
        for j in range(self.n_loops):
            sizes = [t.size(j) for t in self.executable_tiles()]
            lines.append(
                f"loop {j}: tile size min/mean/max = "
                f"{min(sizes)}/{sum(sizes) / len(sizes):.1f}/{max(sizes)}")
        s = self.stats
        lines.append(f"inspection wall time: {s.total_s * 1e3:.3f} ms")
        lines.append(
            "phases (ms): partition %.3f, coloring %.3f, projection+tiling %.3f, "
            "local maps %.3f" % (s.partition_s * 1e3, s.coloring_s * 1e3,
                                 s.projection_tiling_s * 1e3, s.local_maps_s * 1e3))
        name, share = s.dominant_phase()
        lines.append(f"dominant phase: {name} ({share:.1%})")
        return "\n".join(lines)


# -- inspection steps on the GPU, same signatures as reference inspector.py:185-418 --

def partition_seed(space: IterationSpace, ts: int) -> tuple[TilingFunction, list[Tile]]:
    """Chunk the seed space into tiles of ts iterations per region (``inspector.py:185-205``)."""
    from . import _lib
    if ts < 1:
        raise ValueError(f"tile size must be >= 1, got {ts}")
    assignment, m, k = _lib.partition_seed(space, ts)
    tiles = [Tile(id=i, region=Region.CORE) for i in range(m)]
    tiles += [Tile(id=m + j, region=Region.BOUNDARY) for j in range(k)]
    tiles.append(Tile(id=m + k, region=Region.NONEXEC))
    return TilingFunction(loop_index=0, assignment=assignment), tiles


def assign(sigma: TilingFunction, tiles: list[Tile]) -> None:
    """Per-tile ascending iteration lists by a stable GPU sort (``inspector.py:385-391``)."""
    from . import _lib
    off, el = _lib.assign(sigma.assignment, len(tiles))
    for t in tiles:
        t.iteration_lists[sigma.loop_index] = el[off[t.id]:off[t.id + 1]].copy()


def _seed_adjacency(tiles: list[Tile], seed_map: MeshMap | None) -> dict[int, set[int]]:
    """Tiles are adjacent iff their seed iterations share a target (``inspector.py:208-225``)."""
    from . import _lib
    adjacency: dict[int, set[int]] = {t.id: set() for t in tiles}
    if seed_map is None:
        return adjacency
    sigma0 = np.full(seed_map.source.total, NO_TILE, dtype=np.int64)
    for t in tiles:
        lst = t.iteration_lists.get(0)
        if lst is not None and len(lst):
            sigma0[lst] = t.id
    for a, b in _lib.seed_adjacency(seed_map, sigma0, len(tiles)):
        adjacency[a].add(b)
        adjacency[b].add(a)
    return adjacency


def color_tiles(tiles: list[Tile], seed_map: MeshMap | None,
                fake_connections: set[tuple[int, int]], mode: ExecMode,
                adjacency: dict[int, set[int]] | None = None) -> None:
    """Greedy first-fit colouring per region (SHARED) or colour = id (``inspector.py:228-263``)."""
    from . import _lib
    if mode is ExecMode.SHARED:
        if adjacency is None:
            adjacency = _seed_adjacency(tiles, seed_map)
        pos = {t.id: i for i, t in enumerate(tiles)}
        pairs = {(min(pos[a], pos[b]), max(pos[a], pos[b]))
                 for a, nbrs in adjacency.items() for b in nbrs if a in pos and b in pos}
        pairs |= {(min(pos[a], pos[b]), max(pos[a], pos[b])) for a, b in fake_connections}
        colors = _lib.color_tiles([int(t.region) for t in tiles], mode.code, sorted(pairs))
        for t, c in zip(tiles, colors.tolist()):
            t.color = c
    else:
        for t in tiles:
            t.color = t.id


def project(loop, sigma: TilingFunction, phi: dict, conflicts: ConflictMatrix,
            tiles: list[Tile], inverse_maps: dict | None = None) -> None:
    """Fold the loop's tiling into the per-space projections on the GPU
    (``inspector.py:266-316``); ``inverse_maps`` is accepted for signature parity
    (inverses are built on the device)."""
    from . import _lib
    colors = np.array([t.color for t in tiles], dtype=np.int64)
    arrays = {name: p.assignment for name, p in phi.items()}
    for a, b in _lib.project(loop, sigma.assignment, colors, arrays):
        conflicts.add(a, b)
    spaces = {loop.space.name: loop.space}
    for d in loop.descriptors:
        if d.map is not None:
            spaces[d.map.target.name] = d.map.target
    for name in spaces:
        if name in arrays and (name not in phi or arrays[name] is not phi[name].assignment):
            phi[name] = Projection(spaces[name], arrays[name])


def tile_loop(loop, phi: dict, tiles: list[Tile],
              conflicts: ConflictMatrix | None = None) -> TilingFunction:
    """Max-colour tiling of a loop from the projections (``inspector.py:319-382``)."""
    from . import _lib
    colors = np.array([t.color for t in tiles], dtype=np.int64)
    arrays = {name: p.assignment for name, p in phi.items()}
    assignment, pairs = _lib.tile_loop(loop, colors, arrays, conflicts is not None)
    if conflicts is not None:
        for a, b in pairs:
            conflicts.add(a, b)
    return TilingFunction(loop_index=loop.index, assignment=assignment)


def compute_local_maps(tiles: list[Tile], chain: LoopChain) -> None:
    """Map rows restricted to each tile's list, in list order (``inspector.py:397-418``)."""
    from . import _lib
    for t in tiles:
        t.local_maps.clear()
    empty = np.empty(0, dtype=np.int64)
    for j, loop in enumerate(chain.loops):
        done = []
        for d in loop.descriptors:
            if d.is_direct or d.map.name in done:
                continue
            done.append(d.map.name)
            lists = [t.iteration_lists.get(j, empty) for t in tiles]
            flat = _lib.gather_rows(d.map, np.concatenate(lists) if lists else empty)
            offset = 0
            for t, lst in zip(tiles, lists):
                span = len(lst) * d.map.arity
                t.local_maps[(j, d.map.name)] = flat[offset:offset + span].copy()
                offset += span


def find_seed_map(chain: LoopChain) -> MeshMap | None:
    """The map used for tile adjacency (reference ``inspector.py:421-430``)."""
    seed_space = chain.loops[0].space
    for d in chain.loops[0].descriptors:
        if not d.is_direct and d.map.source is seed_space:
            return d.map
    for m in chain.maps:
        if m.source is seed_space:
            return m
    return None


def check_legality_gpu(schedule: Schedule, chain: LoopChain) -> dict:
    """Legality of ``schedule`` for ``chain`` checked on the GPU at any size.

    Restates the reference's brute-force dependence oracle
    (``pkg/tests/legality.py:15-151``): returns ``{"pairs": n, "reductions": m}``,
    the number of distinct cross-loop dependence pairs whose later element runs
    in a different tile of a colour not above the earlier one's, and of
    reduction pairs split over distinct tiles of equal colour (0 and 0 for a
    legal schedule).  ``lt_check_legality`` in include/looptile_cuda.h.
    """
    from . import _lib
    from .errors import StaleScheduleError
    if schedule.fingerprint != chain.fingerprint:
        raise StaleScheduleError("schedule was inspected for a different chain")
    handle = schedule.device_handle(chain)
    return _lib.check_legality(handle, _lib.ChainDesc(chain, device=handle.ctx.device))


def inspect_chain(chain: LoopChain, ts: int, mode: ExecMode) -> Schedule:
    """Run the full inspection on the GPU and return a conflict-free schedule.

    Pure in (chain, ts, mode).  Raises ValueError for ts < 1,
    InspectionError for unreachable elements and ColoringLimitError when
    recolouring exceeds 10 * (number of tiles) rounds, like the reference.
    """
    from . import _lib
    if ts < 1:
        raise ValueError(f"tile size must be >= 1, got {ts}")
    handle = _lib.inspect(chain, ts, mode.code)
    info = handle.info()
    stats = InspectionStats(partition_s=info.partition_s, coloring_s=info.coloring_s,
                            projection_tiling_s=info.projection_tiling_s,
                            local_maps_s=info.local_maps_s, total_s=info.total_s)
    return Schedule(mode, chain.fingerprint, len(chain.loops), None, info.rounds, stats,
                    _handle=handle, _chain=chain)
