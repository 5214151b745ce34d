"""Host-side chain API: validation, fingerprints, mesh generator (CPU only)."""

import numpy as np
import pytest

import paper_1708_03183_b200 as lt
from paper_1708_03183_b200.chain import (AccessMode, Descriptor, IterationSpace, Loop,
                                         MeshMap, build_chain)


def test_mesh_counts_known_answers():
    # reference tests/test_mesh.py:11-21
    m = lt.generate_rect_mesh(1, 1)
    assert (m.num_cells, m.num_vertices, m.num_edges) == (2, 4, 5)
    m = lt.generate_rect_mesh(2, 1)
    assert (m.num_cells, m.num_vertices, m.num_edges) == (4, 6, 9)
    m = lt.generate_rect_mesh(32, 32)
    assert (m.num_cells, m.num_vertices, m.num_edges) == (2048, 1089, 3136)
    m.validate()


@pytest.mark.parametrize("nx,ny", [(1, 1), (3, 2), (7, 5), (16, 8)])
def test_euler_formula_and_validation(nx, ny):
    m = lt.generate_rect_mesh(nx, ny)
    m.validate()
    assert m.num_vertices - m.num_edges + m.num_cells == 1
    r = lt.rcm_renumber(m)
    r.validate()
    z = lt.morton_renumber(m)
    z.validate()


def test_rcm_reduces_bandwidth():
    from paper_1708_03183_b200.mesh import adjacency_bandwidth
    m = lt.generate_rect_mesh(16, 4)
    assert adjacency_bandwidth(lt.rcm_renumber(m)) <= adjacency_bandwidth(m)


def test_facets_partition_edges():
    m = lt.generate_rect_mesh(6, 5)
    ft = lt.facet_topology(m)
    assert ft.n_interior + ft.n_exterior == m.num_edges
    assert ft.n_exterior == 2 * (6 + 5)
    rows = ft.if2c.reshape(-1, 2)
    assert np.all(rows[:, 0] < rows[:, 1])


def _tiny():
    s = IterationSpace("s", 4)
    t = IterationSpace("t", 3)
    m = MeshMap("m", s, t, 2, np.array([0, 1, 1, 2, 2, 0, 0, 1]))
    return s, t, m


def test_build_chain_validation():
    s, t, m = _tiny()
    loop = Loop(0, s, (Descriptor(m, AccessMode.INC),), "edge_inc")
    with pytest.raises(lt.InvalidChainError):
        build_chain((s, t), (m,), (), 1)
    with pytest.raises(lt.InvalidChainError):
        build_chain((s, t), (m,), (loop,), 0)
    with pytest.raises(lt.InvalidChainError):
        build_chain((s, t), (m,), (Loop(1, s, loop.descriptors, "k"),), 1)
    with pytest.raises(lt.DepthExceededError):
        build_chain((s, t), (m,), (loop, Loop(1, s, loop.descriptors, "k")), 1,
                    distributed=True)
    other = MeshMap("m", s, t, 2, m.values)
    with pytest.raises(lt.InvalidChainError):
        build_chain((s, t), (m,), (Loop(0, s, (Descriptor(other, AccessMode.READ),), "k"),), 1)
    with pytest.raises(lt.InvalidChainError):
        MeshMap("bad", s, t, 2, np.array([0, 1, 2, 3, 0, 0, 0, 0]))


def test_rw_fingerprints_as_write():
    s, t, m = _tiny()
    a = build_chain((s, t), (m,), (Loop(0, s, (Descriptor(None, AccessMode.RW),), "k"),), 1)
    b = build_chain((s, t), (m,), (Loop(0, s, (Descriptor(None, AccessMode.WRITE),), "k"),), 1)
    c = build_chain((s, t), (m,), (Loop(0, s, (Descriptor(None, AccessMode.READ),), "k"),), 1)
    assert a.fingerprint == b.fingerprint != c.fingerprint
    assert AccessMode.parse("rw") is AccessMode.RW


def test_subchain_reindexes():
    s, t, m = _tiny()
    loops = tuple(Loop(i, s, (Descriptor(m, AccessMode.READ),), "k") for i in range(3))
    ch = build_chain((s, t), (m,), loops, 3)
    sub = ch.subchain(1, 3)
    assert [lp.index for lp in sub.loops] == [0, 1]
