"""Rank-local strip partitions (strips.py) equal the global partitioner.

``partition.partition_for_ranks`` is pinned to the reference's
``partition_for_ranks`` (tests/test_partition.py, golden fixtures); a strip
built from a window of rows must give the same local mesh -- sizes, global
ids, local connectivity, the local side of every exchange table -- and the
same rank-local elastic problem as ``dg.local_elastic_setup`` of the global
problem (bitwise, including advanced random streams for heterogeneous
materials and noise).
"""

import numpy as np
import pytest

from paper_1708_03183_b200.dg import elastic_setup, local_elastic_setup
from paper_1708_03183_b200.mesh import generate_rect_mesh
from paper_1708_03183_b200.partition import partition_for_ranks
from paper_1708_03183_b200.strips import edge_gid, global_dt, strip_elastic_setup, strip_partition


@pytest.mark.parametrize("nx,ny", [(1, 1), (3, 2), (7, 5)])
def test_edge_gid_closed_form(nx, ny):
    m = generate_rect_mesh(nx, ny)
    pairs = m.edges_to_vertices.reshape(-1, 2)
    assert np.array_equal(edge_gid(pairs[:, 0], pairs[:, 1], nx, ny), np.arange(m.num_edges))


CASES = [(6, 24, 3, 2), (5, 40, 4, 3), (8, 30, 2, 5), (4, 36, 3, 1), (9, 21, 3, 2),
         (6, 12, 4, 4), (3, 17, 5, 2), (7, 9, 8, 3)]


@pytest.mark.parametrize("nx,ny,nranks,depth", CASES)
def test_strip_partition_equals_global_partitioner(nx, ny, nranks, depth):
    ref = partition_for_ranks(generate_rect_mesh(nx, ny), nranks, depth)
    for r in range(nranks):
        sp = strip_partition(nx, ny, nranks, depth, r)
        a, b = sp.local, ref[r]
        assert a.sizes == b.sizes
        for space in b.global_ids:
            assert np.array_equal(a.global_ids[space], b.global_ids[space]), (r, space)
        assert np.array_equal(a.cells_to_vertices, b.cells_to_vertices)
        assert np.array_equal(a.edges_to_vertices, b.edges_to_vertices)
        assert np.array_equal(a.vertex_coords, b.vertex_coords)
        assert set(a.exchange_table) == set(b.exchange_table)
        for key, table in b.exchange_table.items():
            assert np.array_equal(a.exchange_table[key][:, 0], table[:, 0]), (r, key)


@pytest.mark.parametrize("material,noise,p,T", [("homogeneous", None, 3, 2),
                                                (("uniform", 2), 1, 2, 2),
                                                (("uniform", 5), 3, 1, 1)])
def test_strip_elastic_setup_equals_restricted_global(material, noise, p, T):
    nx, ny, nranks = 6, 30, 3
    depth = 5 * T
    g = elastic_setup(nx, ny, p, T, material=material, noise_seed=noise, sigma=4.0)
    assert global_dt(p, material, g.n_cells) == g.dt
    lms = partition_for_ranks(g.mesh, nranks, depth)
    for r in range(nranks):
        want = local_elastic_setup(g, lms[r])
        got = strip_elastic_setup(strip_partition(nx, ny, nranks, depth, r), p, T, material,
                                  noise, 4.0, g.dt)
        assert got.dt == want.dt
        for name, sp in want.spaces.items():
            assert (got.spaces[name].core_size, got.spaces[name].boundary_size,
                    got.spaces[name].nonexec_size) == (sp.core_size, sp.boundary_size,
                                                       sp.nonexec_size), name
        for name, m in want.maps.items():
            assert np.array_equal(got.maps[name].values, m.values), (r, name)
        for name, v in want.data.items():
            if name in ("u", "s"):
                np.testing.assert_allclose(got.data[name], v, rtol=0, atol=1e-15)
            else:
                assert np.array_equal(got.data[name], v), (r, name)
