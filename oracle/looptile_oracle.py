"""CPU oracle for the sparse-tiling inspector/executor -- TEST INFRASTRUCTURE ONLY.

A plain numpy / Python restatement of the reference algorithm
(``/root/reference/pkg/src/looptile``), used as the checker for the CUDA
product path.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import it; the product package
never does.  It is pinned against fixtures generated from the real reference
(``tests/golden/make_golden.py``; ``tests/test_oracle.py``).

It consumes the host side of the product's chain objects (spaces, map
``values``, loops, descriptors) and plain numpy dataset arrays.

Restated functions, with the reference lines they follow:

* ``partition_seed``     inspector.py:185-205
* ``assign``             inspector.py:385-391
* ``seed_adjacency``     inspector.py:208-225 (+ find_seed_map :421-430)
* ``color_tiles``        inspector.py:228-263
* ``invert``             chain.py:118-135
* ``project``            inspector.py:266-316
* ``tile_loop``          inspector.py:319-382
* ``local_maps``         inspector.py:397-418
* ``inspect``            inspector.py:433-495
* ``serialize``          inspector.py:139-155
* ``execute_untiled``    executor.py:163-169 (+ _run_loop :128-160)
* ``execute_tiled``      executor.py:185-245 (+ _execute_tile :172-182)
* ``check_legality`` / ``footprint_conflicts``  tests/legality.py:43-151
* kernel bodies          problems.py:49-64; toy bodies (BASELINE config 1);
                         DG bodies in ``dg_oracle.py``.
"""

from __future__ import annotations

import math
from collections import defaultdict
from dataclasses import dataclass, field

import numpy as np

NO_TILE = -1
CORE, BOUNDARY, NONEXEC = 0, 1, 2
REGION_NAMES = {CORE: "core", BOUNDARY: "boundary", NONEXEC: "nonexec"}


class OracleInspectionError(RuntimeError):
    pass


class OracleColoringLimit(OracleInspectionError):
    pass


@dataclass
class OTile:
    id: int
    region: int
    color: int = -1
    lists: dict = field(default_factory=dict)
    lmaps: dict = field(default_factory=dict)


@dataclass
class OSchedule:
    mode: str
    fingerprint: str
    n_loops: int
    tiles: list
    rounds: int

    def serialize(self) -> bytes:
        colors = sorted({t.color for t in self.tiles})
        out = ["schedule-v1", f"mode={self.mode}", f"fingerprint={self.fingerprint}",
               f"loops={self.n_loops}", f"rounds={self.rounds}",
               "colors=" + ",".join(str(c) for c in colors)]
        for t in self.tiles:
            out.append(f"tile id={t.id} region={REGION_NAMES[t.region]} color={t.color}")
            for j in sorted(t.lists):
                out.append(f"  list {j}=" + ",".join(str(int(x)) for x in t.lists[j]))
            for key in sorted(t.lmaps):
                out.append(f"  lmap {key[0]} {key[1]}=" +
                           ",".join(str(int(x)) for x in t.lmaps[key]))
        return ("\n".join(out) + "\n").encode()

    def tile_of(self, j: int, n: int) -> np.ndarray:
        out = np.full(n, NO_TILE, dtype=np.int64)
        for t in self.tiles:
            if j in t.lists:
                out[t.lists[j]] = t.id
        return out


# ---- inspection -----------------------------------------------------------------------

def partition_seed(space, ts: int):
    if ts < 1:
        raise ValueError("tile size must be >= 1")
    m = -(-space.core_size // ts)
    k = -(-space.boundary_size // ts)
    regions = [CORE] * m + [BOUNDARY] * k + [NONEXEC]
    e = np.arange(space.total, dtype=np.int64)
    sigma = np.where(e < space.core_size, e // ts,
                     np.where(e < space.executable_size,
                              m + (e - space.core_size) // ts, m + k))
    return sigma.astype(np.int64), regions


def assign(sigma: np.ndarray, n_tiles: int) -> list[np.ndarray]:
    """Per-tile ascending element lists (counting sort; stable)."""
    order = np.argsort(sigma, kind="stable")
    cuts = np.searchsorted(sigma[order], np.arange(n_tiles + 1))
    return [order[cuts[t]:cuts[t + 1]].astype(np.int64) for t in range(n_tiles)]


def invert(values: np.ndarray, n_source: int, arity: int, n_target: int):
    """CSR inverse: offsets and source ids, each segment ascending by source."""
    src = np.repeat(np.arange(n_source, dtype=np.int64), arity)
    order = np.argsort(values, kind="stable")  # flat order is already source-major
    counts = np.bincount(values, minlength=n_target)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return offsets, src[order]


def find_seed_map(chain):
    seed = chain.loops[0].space
    for d in chain.loops[0].descriptors:
        if d.map is not None and d.map.source is seed:
            return d.map
    for m in chain.maps:
        if m.source is seed:
            return m
    return None


def seed_adjacency(sigma0: np.ndarray, seed_map, n_tiles: int) -> list[set]:
    adj = [set() for _ in range(n_tiles)]
    if seed_map is None:
        return adj
    rows = seed_map.values.reshape(-1, seed_map.arity)
    touch = defaultdict(set)
    for e in range(len(sigma0)):
        for g in rows[e].tolist():
            touch[g].add(int(sigma0[e]))
    for tiles in touch.values():
        for a in tiles:
            adj[a].update(tiles - {a})
    return adj


def color_tiles(regions, adjacency, fake, mode: str) -> list[int]:
    n = len(regions)
    colors = [-1] * n
    if mode != "shared":
        return list(range(n))
    adj = [set(s) for s in adjacency]
    for a, b in fake:
        adj[a].add(b)
        adj[b].add(a)
    floor = 0
    for region in (CORE, BOUNDARY):
        done = {}
        for t in range(n):
            if regions[t] != region:
                continue
            used = {done[x] for x in adj[t] if x in done}
            c = floor
            while c in used:
                c += 1
            done[t] = c
            colors[t] = c
        if done:
            floor = max(done.values()) + 1
    colors[n - 1] = floor
    return colors


def project(loop, sigma, phi, conflicts, colors, inverses):
    col = np.asarray(colors)
    for d in loop.descriptors:
        if d.map is None:
            name = loop.space.name
            old = phi.get(name)
            new = sigma.copy()
            if old is not None:
                hit = (old >= 0) & (new >= 0) & (old != new)
                hit &= col[np.where(old >= 0, old, 0)] == col[np.where(new >= 0, new, 0)]
                for e in np.flatnonzero(hit):
                    conflicts.add((min(old[e], new[e]), max(old[e], new[e])))
            phi[name] = new
            continue
        m = d.map
        if m.name not in inverses:
            inverses[m.name] = invert(m.values, m.source.total, m.arity, m.target.total)
        offsets, sources = inverses[m.name]
        old = phi.get(m.target.name)
        new = np.full(m.target.total, NO_TILE, dtype=np.int64)
        for e in range(m.target.total):
            first_of_color = {}
            best, best_c = NO_TILE, -1
            if old is not None and old[e] >= 0:
                best = int(old[e])
                best_c = int(col[best])
                first_of_color[best_c] = best
            for f in sources[offsets[e]:offsets[e + 1]]:
                t = int(sigma[f])
                c = int(col[t])
                first = first_of_color.setdefault(c, t)
                if first != t:
                    conflicts.add((min(first, t), max(first, t)))
                if c > best_c:
                    best, best_c = t, c
            new[e] = best
        phi[m.target.name] = new


def tile_loop(loop, phi, colors, conflicts, tne: int):
    col = np.asarray(colors)
    space = loop.space
    cands = []
    for d in loop.descriptors:
        if d.map is None:
            if space.name in phi:
                cands.append((phi[space.name], None, 1))
        elif d.map.target.name in phi:
            cands.append((phi[d.map.target.name], d.map.values, d.map.arity))
    if not cands:
        raise OracleInspectionError(f"loop {loop.index}: no projection covers any accessed space")
    held = np.full(space.total, NO_TILE, dtype=np.int64)
    held_c = np.full(space.total, -1, dtype=np.int64)
    for pa, vals, a in cands:
        for k in range(a):
            cand = pa[:space.total] if vals is None else pa[vals[k::a]]
            c = np.where(cand >= 0, col[np.where(cand >= 0, cand, 0)], -1)
            better = (cand >= 0) & (c > held_c)
            held = np.where(better, cand, held)
            held_c = np.where(better, c, held_c)
    ex = space.executable_size
    if np.any(held[:ex] < 0):
        raise OracleInspectionError(
            f"loop {loop.index}: element {int(np.flatnonzero(held[:ex] < 0)[0])} unreachable")
    for pa, vals, a in cands:
        for k in range(a):
            cand = (pa[:space.total] if vals is None else pa[vals[k::a]])[:ex]
            h = held[:ex]
            same = (cand >= 0) & (cand != h) & (col[np.where(cand >= 0, cand, 0)] == col[h])
            for e in np.flatnonzero(same):
                conflicts.add((min(h[e], cand[e]), max(h[e], cand[e])))
    held[ex:] = tne
    return held


def inspect(chain, ts: int, mode: str, fingerprint: str | None = None) -> OSchedule:
    """Alg. 1: seed, colour, project/tile per loop, recolour until conflict-free."""
    n = len(chain.loops)
    sigma0, regions = partition_seed(chain.loops[0].space, ts)
    n_tiles = len(regions)
    tne = n_tiles - 1
    lists = {0: assign(sigma0, n_tiles)}
    seed_map = find_seed_map(chain)
    adj = seed_adjacency(sigma0, seed_map, n_tiles) if mode == "shared" else [set()] * n_tiles
    inverses = {}
    fake = set()
    rounds = 0
    while True:
        rounds += 1
        if rounds > 10 * n_tiles:
            raise OracleColoringLimit("recoloring did not converge")
        colors = color_tiles(regions, adj, fake, mode)
        phi, conflicts = {}, set()
        sigma = sigma0
        for j in range(1, n):
            project(chain.loops[j - 1], sigma, phi, conflicts, colors, inverses)
            sigma = tile_loop(chain.loops[j], phi, colors, conflicts, tne)
            lists[j] = assign(sigma, n_tiles)
        if conflicts:
            fake |= conflicts
            continue
        break
    tiles = [OTile(t, regions[t], colors[t]) for t in range(n_tiles)]
    for j, per_tile in lists.items():
        for t in tiles:
            t.lists[j] = per_tile[t.id]
    for j, loop in enumerate(chain.loops):
        seen = []
        for d in loop.descriptors:
            if d.map is None or d.map.name in seen:
                continue
            seen.append(d.map.name)
            rows = d.map.values.reshape(-1, d.map.arity)
            for t in tiles:
                t.lmaps[(j, d.map.name)] = rows[t.lists[j]].ravel().astype(np.int64)
    return OSchedule(mode, fingerprint if fingerprint is not None else chain.fingerprint,
                     n, tiles, rounds)


# ---- kernel bodies (numpy views; INC/WRITE views mutable) --------------------------------

def _k_inc_each(x, targets):
    for v in targets:
        v += x


def _k_sum_read(out, targets):
    s = targets[0].copy()
    for v in targets[1:]:
        s = s + v
    out[:] = s


def _k_toy1(a, v):
    for x in v:
        x += a / 3.0


def _k_toy2(e, v):
    e[:] = 0.5 * (v[0] + v[1])


def _k_toy3(a, e):
    a += (e[0] + e[1] + e[2]) / 3.0


KERNELS = {
    "edge_inc": _k_inc_each, "cell_inc": _k_inc_each,
    "edge_read": _k_sum_read, "cell_read": _k_sum_read,
    "toy_k1": _k_toy1, "toy_k2": _k_toy2, "toy_k3": _k_toy3,
}


def kernel_table(dg: tuple[int, float] | None = None):
    """Scalar bodies, plus the DG bodies of degree p with timestep dt if given."""
    table = dict(KERNELS)
    if dg is not None:
        from oracle import dg_oracle
        table.update(dg_oracle.bodies(*dg))
    return table


def _run_loop(loop, binding, data, vpe, elements, kernels, local_rows=None):
    body = kernels[binding.kernel]
    plan = []
    for d, name in zip(loop.descriptors, binding.args):
        rows = None
        if d.map is not None:
            rows = local_rows[d.map.name] if local_rows is not None else d.map.values
        plan.append((d, data[name], vpe[name], rows))
    for pos, e in enumerate(elements):
        e = int(e)
        args = []
        for d, values, k, rows in plan:
            if d.map is None:
                args.append(values[e * k:(e + 1) * k])
            else:
                a = d.map.arity
                base = (pos if local_rows is not None else e) * a
                args.append([values[t * k:(t + 1) * k] for t in rows[base:base + a]])
        body(*args)


def execute_untiled(chain, bindings, data: dict, vpe: dict, kernels=None) -> None:
    kernels = kernels or kernel_table()
    for loop, binding in zip(chain.loops, bindings):
        _run_loop(loop, binding, data, vpe, range(loop.space.executable_size), kernels)


def execute_tiled(schedule: OSchedule, chain, bindings, data: dict, vpe: dict,
                  kernels=None, use_local_maps: bool = False, exchange_end=None) -> None:
    kernels = kernels or kernel_table()

    def run(region):
        for t in sorted((t for t in schedule.tiles if t.region == region),
                        key=lambda t: (t.color, schedule.tiles.index(t))):
            for j, (loop, binding) in enumerate(zip(chain.loops, bindings)):
                el = t.lists.get(j)
                if el is None or not len(el):
                    continue
                local = ({name: rows for (jj, name), rows in t.lmaps.items() if jj == j}
                         if use_local_maps else None)
                _run_loop(loop, binding, data, vpe, el, kernels, local)

    run(CORE)
    if exchange_end is not None:
        exchange_end()
    run(BOUNDARY)


# ---- legality (tests/legality.py:43-151) -------------------------------------------------

def _touches(loop, e, writes):
    out = []
    for d in loop.descriptors:
        is_write = d.mode.value != "r"
        if is_write != writes:
            continue
        if d.map is None:
            out.append((loop.space.name, e, True))
        else:
            for t in d.map.values[e * d.map.arity:(e + 1) * d.map.arity]:
                out.append((d.map.target.name, int(t), False))
    return out


def _by_target(loop, writes):
    table = defaultdict(list)
    for e in range(loop.space.executable_size):
        for sp, t, direct in _touches(loop, e, writes):
            table[(sp, t)].append((e, direct))
    return table


def dependence_pairs(chain):
    w = [_by_target(lp, True) for lp in chain.loops]
    r = [_by_target(lp, False) for lp in chain.loops]
    pairs = set()
    n = len(chain.loops)
    for x in range(n):
        for y in range(x + 1, n):
            for first, second in ((w[x], r[y]), (r[x], w[y]), (w[x], w[y])):
                for key, xs in first.items():
                    ys = second.get(key)
                    if not ys:
                        continue
                    for ex, dx in xs:
                        for ey, dy in ys:
                            if not (dx and dy):
                                pairs.add((x, ex, y, ey))
    red = set()
    for j, lp in enumerate(chain.loops):
        table = defaultdict(list)
        for e in range(lp.space.executable_size):
            for d in lp.descriptors:
                if d.map is None or d.mode.value != "i":
                    continue
                for t in d.map.values[e * d.map.arity:(e + 1) * d.map.arity]:
                    table[(d.map.target.name, int(t))].append(e)
        for es in table.values():
            for a in es:
                for b in es:
                    if a < b:
                        red.add((j, a, b))
    return sorted(pairs), sorted(red)


def check_legality(chain, tile_of: list[np.ndarray], colors: dict, tne: int) -> list[str]:
    """Violations of the ordering rules; ``tile_of[j]`` per-element tile of loop j."""
    pairs, red = dependence_pairs(chain)
    bad = []
    for x, ex, y, ey in pairs:
        tx, ty = int(tile_of[x][ex]), int(tile_of[y][ey])
        if NO_TILE in (tx, ty) or tne in (tx, ty):
            continue
        if colors[ty] < colors[tx] or (colors[ty] == colors[tx] and tx != ty):
            bad.append(f"L{x}[{ex}] -> L{y}[{ey}]: tiles {tx}/{ty}")
    for j, a, b in red:
        ta, tb = int(tile_of[j][a]), int(tile_of[j][b])
        if NO_TILE in (ta, tb) or tne in (ta, tb):
            continue
        if ta != tb and colors[ta] == colors[tb]:
            bad.append(f"reduction L{j}[{a}]~[{b}] split over equal colour")
    return bad


def footprint_conflicts(chain, lists_per_tile: dict, colors: dict, regions: dict) -> list:
    """Equal-coloured executed tiles sharing an indirect target one of them writes."""
    touched, written = {}, {}
    for t, lists in lists_per_tile.items():
        if regions[t] == NONEXEC:
            continue
        rd, wr = set(), set()
        for j, loop in enumerate(chain.loops):
            el = lists.get(j)
            if el is None:
                continue
            for d in loop.descriptors:
                if d.map is None:
                    continue
                rows = d.map.values.reshape(-1, d.map.arity)[el]
                (rd if d.mode.value == "r" else wr).update(
                    (d.map.target.name, int(v)) for v in rows.ravel())
        touched[t] = rd | wr
        written[t] = wr
    ids = sorted(touched)
    out = []
    for i, a in enumerate(ids):
        for b in ids[i + 1:]:
            if colors[a] == colors[b] and ((written[a] & touched[b]) or (written[b] & touched[a])):
                out.append((a, b))
    return out
