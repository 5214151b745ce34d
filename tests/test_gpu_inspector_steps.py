"""GPU inspector steps (partition_seed, assign, color_tiles, project, tile_loop,
compute_local_maps) with the known answers and properties of the reference's
unit tests (pkg/tests/test_inspector.py), restated."""

import numpy as np
import pytest

import paper_1708_03183_b200 as lt
from paper_1708_03183_b200.chain import AccessMode, Descriptor, IterationSpace, Loop, MeshMap
from paper_1708_03183_b200.inspector import (NO_TILE, ConflictMatrix, ExecMode, Projection,
                                             Tile, TilingFunction, _seed_adjacency, assign,
                                             color_tiles, compute_local_maps, find_seed_map,
                                             partition_seed, project, tile_loop)
from paper_1708_03183_b200.chain import Region
from cases import build_case

pytestmark = pytest.mark.gpu


def test_seed_chunks_and_regions():
    sigma, tiles = partition_seed(IterationSpace("s", 10), 4)
    assert [int(np.sum(sigma.assignment == t.id)) for t in tiles] == [4, 4, 2, 0]
    assert [t.region for t in tiles] == [Region.CORE] * 3 + [Region.NONEXEC]
    sigma, tiles = partition_seed(IterationSpace("s", 9, 4, 3), 3)
    assert [t.region for t in tiles] == [Region.CORE] * 3 + [Region.BOUNDARY] * 2 + [Region.NONEXEC]
    assert sigma.assignment[:9].tolist() == [e // 3 for e in range(9)]
    assert sigma.assignment[9:13].tolist() == [3 + (e - 9) // 3 for e in range(9, 13)]
    assert np.all(sigma.assignment[13:] == 5)
    with pytest.raises(ValueError):
        partition_seed(IterationSpace("s", 4), 0)


def seeded(space, ts):
    sigma, tiles = partition_seed(space, ts)
    assign(sigma, tiles)
    return sigma, tiles


def test_greedy_colouring_and_modes():
    edges, verts = IterationSpace("edges", 4), IterationSpace("verts", 4)
    e2v = MeshMap("e2v", edges, verts, 2, np.array([0, 1, 0, 2, 1, 2, 2, 3]))
    _, tiles = seeded(edges, 1)
    color_tiles(tiles, e2v, set(), ExecMode.SHARED)
    colors = [t.color for t in tiles[:-1]]
    assert colors[0] == colors[3] and len(set(colors)) == 3
    assert tiles[-1].color > max(colors)
    _, tiles = seeded(IterationSpace("s", 8, 8, 3), 4)
    color_tiles(tiles, None, set(), ExecMode.DISTRIBUTED)
    assert [t.color for t in tiles] == [0, 1, 2, 3, 4]
    _, tiles = seeded(edges, 1)
    color_tiles(tiles, None, set(), ExecMode.SHARED)
    assert tiles[0].color == tiles[3].color
    color_tiles(tiles, None, {(0, 3)}, ExecMode.SHARED)
    assert tiles[0].color != tiles[3].color


def seven_edges():
    edges, verts = IterationSpace("edges", 7), IterationSpace("verts", 8)
    e2v = MeshMap("e2v", edges, verts, 2, np.array([[0, i + 1] for i in range(7)]).ravel())
    tiles = [Tile(0, Region.CORE, color=0), Tile(1, Region.CORE, color=1),
             Tile(2, Region.NONEXEC, color=2)]
    sigma = TilingFunction(0, np.array([0, 0, 1, 1, 1, 1, 1]))
    return Loop(0, edges, (Descriptor(e2v, AccessMode.INC),), "k"), sigma, tiles


def test_projection_known_answers():
    loop, sigma, tiles = seven_edges()
    phi, c = {}, ConflictMatrix()
    project(loop, sigma, phi, c, tiles, {})
    assert phi["verts"].assignment[0] == 1 and not c.has_conflicts()
    before = phi["verts"].assignment.copy()
    project(Loop(1, loop.space, loop.descriptors, "k"), TilingFunction(1, np.zeros(7, np.int64)),
            phi, ConflictMatrix(), tiles, {})
    for v in range(8):
        if before[v] >= 0:
            assert tiles[int(phi["verts"].assignment[v])].color >= tiles[int(before[v])].color


@pytest.mark.parametrize("seed", range(12))
def test_projection_matches_bruteforce_max(seed):
    rng = np.random.default_rng(seed)
    edges, verts = IterationSpace("edges", 30), IterationSpace("verts", 12)
    e2v = MeshMap("e2v", edges, verts, 2, rng.integers(0, 12, size=60))
    tiles = [Tile(i, Region.CORE, color=int(c)) for i, c in enumerate(rng.integers(0, 4, 5))]
    tiles.append(Tile(5, Region.NONEXEC, color=10))
    sigma = TilingFunction(0, rng.integers(0, 5, size=30))
    phi = {}
    project(Loop(0, edges, (Descriptor(e2v, AccessMode.INC),), "k"), sigma, phi,
            ConflictMatrix(), tiles, {})
    got = phi["verts"].assignment
    for v in range(12):
        touch = [int(sigma.assignment[e]) for e in range(30) if v in e2v.row(e)]
        if not touch:
            assert got[v] == NO_TILE
        else:
            assert tiles[int(got[v])].color == max(tiles[t].color for t in touch)


def test_tiling_known_answers():
    cells, verts = IterationSpace("cells", 1), IterationSpace("verts", 3)
    c2v = MeshMap("c2v", cells, verts, 3, np.array([0, 1, 2]))
    tiles = [Tile(0, Region.CORE, color=0), Tile(1, Region.CORE, color=1),
             Tile(2, Region.NONEXEC, color=2)]
    phi = {"verts": Projection(verts, np.array([1, 0, 0]))}
    assert tile_loop(Loop(1, cells, (Descriptor(c2v, AccessMode.INC),), "k"), phi,
                     tiles).assignment[0] == 1
    with pytest.raises(lt.InspectionError):
        tile_loop(Loop(1, IterationSpace("x", 2), (Descriptor(None, AccessMode.READ),), "k"), {},
                  [Tile(0, Region.CORE, color=0)])
    cells2, verts2 = IterationSpace("cells", 2), IterationSpace("verts", 2)
    c2v2 = MeshMap("c2v", cells2, verts2, 3, np.array([0, 1, 0, 1, 0, 1]))
    t2 = [Tile(0, Region.CORE, color=0), Tile(1, Region.NONEXEC, color=1)]
    sig = tile_loop(Loop(1, cells2, (Descriptor(None, AccessMode.READ),
                                     Descriptor(c2v2, AccessMode.INC)), "k"),
                    {"verts": Projection(verts2, np.zeros(2, dtype=np.int64))}, t2)
    assert np.all(sig.assignment == 0)


def test_assign_known_answer_and_partition():
    tiles = [Tile(i, Region.CORE) for i in range(3)]
    assign(TilingFunction(2, np.array([2, 0, 1, 0, 2, 1, 0, 0, 2])), tiles)
    assert [t.iteration_lists[2].tolist() for t in tiles] == [[1, 3, 6, 7], [2, 5], [0, 4, 8]]
    rng = np.random.default_rng(3)
    tiles = [Tile(i, Region.CORE) for i in range(6)]
    assign(TilingFunction(0, rng.integers(0, 6, size=40)), tiles)
    cat = np.concatenate([t.iteration_lists[0] for t in tiles])
    assert sorted(cat.tolist()) == list(range(40))


@pytest.mark.parametrize("case", [("fig2", (8, 4), "none", 4, "shared"),
                                  ("eight", (8, 4), "rcm", 3, "shared"),
                                  ("toy", (8, 8), "none", 8, "sequential"),
                                  ("fig2", (4, 1), "rcm", 2, "shared")])
def test_steps_compose_to_inspect_chain(case):
    """Driving the GPU steps like inspect_chain (inspector.py:433-495) gives the
    same bytes as lt_inspect."""
    prob, dims, ren, ts, mode = case
    _, (chain, _, _, _) = build_case(prob, dims, ren)
    mode = ExecMode.parse(mode)
    sigma0, tiles = partition_seed(chain.loops[0].space, ts)
    assign(sigma0, tiles)
    seed_map = find_seed_map(chain)
    adj = _seed_adjacency(tiles, seed_map) if mode is ExecMode.SHARED else None
    fake, rounds = set(), 0
    tne = tiles[-1].id
    while True:
        rounds += 1
        color_tiles(tiles, seed_map, fake, mode, adjacency=adj)
        c, phi, sigma = ConflictMatrix(), {}, sigma0
        for j in range(1, len(chain.loops)):
            project(chain.loops[j - 1], sigma, phi, c, tiles, {})
            sigma = tile_loop(chain.loops[j], phi, tiles, c)
            sigma.assignment[chain.loops[j].space.executable_size:] = tne
            assign(sigma, tiles)
        if c.has_conflicts():
            fake |= c.pairs
            continue
        break
    compute_local_maps(tiles, chain)
    mine = lt.Schedule(mode, chain.fingerprint, len(chain.loops), tiles, rounds)
    assert mine.serialize() == lt.inspect_chain(chain, ts, mode).serialize()
