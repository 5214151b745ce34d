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
