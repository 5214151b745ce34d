"""The GPU-side problem generator (configs 3-4) equals the host generator.

``dg.elastic_setup_device`` builds the mesh, facets, geometry, material and
initial state with torch ops (run here on the CPU device); it must reproduce
``dg.elastic_setup`` (host numpy, whose mesh numbering is pinned to the
reference generator through the chain fingerprints in tests/golden): maps
and geometry exactly, the chain fingerprint byte for byte (device maps hash
their int64 bytes in chunks), the Gaussian projection to rounding.
"""

import numpy as np
import pytest
import torch

from paper_1708_03183_b200.chain import build_chain
from paper_1708_03183_b200.dg import elastic_setup, elastic_setup_device


@pytest.mark.parametrize("nx,ny,p,T,material,noise", [
    (1, 1, 1, 1, "homogeneous", 1),
    (3, 2, 2, 2, ("uniform", 2), 1),
    (7, 5, 3, 2, "homogeneous", None),
    (16, 9, 1, 1, ("uniform", 3), 4),
    (12, 12, 4, 1, "homogeneous", 1),
])
def test_device_setup_equals_host_setup(nx, ny, p, T, material, noise):
    h = elastic_setup(nx, ny, p, T, material=material, noise_seed=noise, sigma=3.0)
    d = elastic_setup_device(nx, ny, p, T, material=material, noise_seed=noise, sigma=3.0,
                             device="cpu")
    assert d.n_cells == h.n_cells and d.dt == h.dt
    for name, m in h.maps.items():
        dm = d.maps[name]
        assert dm.on_device_only
        assert np.array_equal(dm.host_values(), m.values), name
    for name, sp in h.spaces.items():
        assert (d.spaces[name].core_size, d.spaces[name].boundary_size,
                d.spaces[name].nonexec_size) == (sp.core_size, sp.boundary_size,
                                                 sp.nonexec_size)
    for name in ("cgeo", "mat", "figeo", "fegeo", "ru", "rs"):
        got = d.data[name].numpy()
        assert np.array_equal(got, h.data[name]), name
    for name in ("u", "s"):
        np.testing.assert_allclose(d.data[name].numpy(), h.data[name], rtol=0, atol=1e-14)
    ch = build_chain(tuple(h.spaces.values()), tuple(h.maps.values()), h.loops, len(h.loops))
    cd = build_chain(tuple(d.spaces.values()), tuple(d.maps.values()), d.loops, len(d.loops))
    assert ch.fingerprint == cd.fingerprint


def test_device_map_validation():
    from paper_1708_03183_b200.chain import IterationSpace, MeshMap
    from paper_1708_03183_b200.errors import InvalidChainError
    a, b = IterationSpace("a", 4), IterationSpace("b", 3)
    m = MeshMap("m", a, b, 2, torch.tensor([0, 1, 2, 0, 1, 1, 2, 2]))
    assert m.row(2).tolist() == [1, 1] and m.row(3).tolist() == [2, 2]
    with pytest.raises(InvalidChainError):
        MeshMap("m", a, b, 2, torch.tensor([0, 1, 2, 0, 1, 1, 2, 3]))
    with pytest.raises(InvalidChainError):
        MeshMap("m", a, b, 2, torch.tensor([0, 1, 2]))


@pytest.mark.parametrize("nx,ny,p,T,material,noise,scheme", [
    (6, 4, 1, 1, "homogeneous", 1, "morton"),
    (8, 8, 2, 2, ("uniform", 2), 1, "morton"),
    (5, 3, 3, 1, ("uniform", 7), None, "morton"),
    (8, 6, 2, 1, ("uniform", 4), 3, "block:4x3"),
    (7, 5, 1, 2, "homogeneous", 1, "block:4x2"),
])
def test_morton_renumbering_is_a_consistent_permutation(nx, ny, p, T, material, noise, scheme):
    """The layout pass (north star item 3) permutes cells and facets and changes
    nothing else: per-cell inputs follow their cells, every facet still joins
    the same two cells through the same faces, and the oracle's untiled chain
    on the renumbered problem gives the row-major result, permuted (1e-12:
    facet contributions reach a cell in a different order)."""
    from oracle import looptile_oracle as O
    from paper_1708_03183_b200.dg import morton_renumber_device, rect_mesh_device
    a = elastic_setup_device(nx, ny, p, T, material=material, noise_seed=noise, sigma=2.0,
                             device="cpu")
    b = elastic_setup_device(nx, ny, p, T, material=material, noise_seed=noise, sigma=2.0,
                             device="cpu", renumber=scheme)
    block = None if scheme == "morton" else tuple(int(v) for v in scheme[6:].split("x"))
    old_of_new = morton_renumber_device(rect_mesh_device(nx, ny, "cpu"), nx, ny,
                                        block=block)["old_of_new"]
    old_of_new = old_of_new.numpy()
    assert sorted(old_of_new.tolist()) == list(range(2 * nx * ny))
    if block is not None:  # the first 2*bx*by cells are the bx x by block of quads at the origin
        bx, by = block
        quads = sorted(set(int(c) // 2 for c in old_of_new[:2 * bx * by]))
        assert {(q % nx, q // nx) for q in quads} == {(i, j) for i in range(bx) for j in range(by)}
    # Morton: 16 consecutive cells = 4 x 2 quads
    elif nx >= 4 and ny >= 2:
        quads = sorted(set(int(c) // 2 for c in old_of_new[:16]))
        assert {(q % nx, q // nx) for q in quads} == {(i, j) for i in range(4) for j in range(2)}
    for name in ("cgeo", "mat", "u", "s"):
        v = a.vpe[name]
        np.testing.assert_array_equal(b.data[name].numpy().reshape(-1, v),
                                      a.data[name].numpy().reshape(-1, v)[old_of_new], name)
    # facets: same set of (cell pair, face pair) in the generator's numbering
    def facets(st, to_old):
        f = st.maps["if2c"].host_values().reshape(-1, 2)
        g = st.data["figeo"].numpy().reshape(-1, 5)
        out = set()
        for (ca, cb), row in zip(f, g):
            ka, kb = (int(to_old[ca]), int(row[3])), (int(to_old[cb]), int(row[4]))
            out.add((min(ka, kb), max(ka, kb)))
        return out
    ident = np.arange(2 * nx * ny)
    assert facets(a, ident) == facets(b, old_of_new)
    fb = b.maps["if2c"].host_values().reshape(-1, 2)
    assert (fb[:, 0] < fb[:, 1]).all() and (np.diff(fb[:, 0]) >= 0).all()
    res = []
    from paper_1708_03183_b200.chain import MeshMap
    from paper_1708_03183_b200.dg import chain_loops
    for st in (a, b):
        maps = {k: MeshMap(k, m.source, m.target, m.arity, m.host_values())
                for k, m in st.maps.items()}           # host copies for the oracle
        loops, _ = chain_loops(p, T, st.spaces, maps)
        chain = build_chain(tuple(st.spaces.values()), tuple(maps.values()), loops, len(loops))
        data = {k: np.array(v.numpy() if hasattr(v, "numpy") else v, dtype=np.float64)
                for k, v in st.data.items()}
        O.execute_untiled(chain, st.bindings, data, st.vpe, O.kernel_table(dg=(p, st.dt)))
        res.append(data)
    for name in ("u", "s", "ru", "rs"):
        v = a.vpe[name]
        ra = res[0][name].reshape(-1, v)[old_of_new]
        rb = res[1][name].reshape(-1, v)
        assert np.max(np.abs(ra - rb)) <= 1e-12 * max(np.max(np.abs(ra)), 1e-300), name
