"""The C-ABI library builds, loads and exports every declared symbol (CPU only)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_npz, has_gpu

import paper_1708_03183_b200 as lt
from paper_1708_03183_b200 import _lib


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "looptile_cuda.h")).read()
    return sorted(set(re.findall(r"\b(lt_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing a ctypes signature"


def test_abi_version_and_kernel_table():
    lib = _lib.load()
    assert lib.lt_abi_version() == 2
    names = _lib.kernel_names()
    for k in ("edge_inc", "cell_inc", "edge_read", "cell_read", "toy_k1", "toy_k2", "toy_k3"):
        assert k in names
    for p in (1, 2, 3, 4):
        for k in ("vol", "iflux", "eflux", "minv", "axpy"):
            assert f"dg_{k}_p{p}" in names
    kid, nargs = _lib.kernel_lookup("edge_inc")
    assert (kid, nargs) == (0, 2)
    with pytest.raises(lt.ExecutionError):
        _lib.kernel_lookup("no_such_kernel")


def test_error_codes_map_to_reference_exceptions():
    assert _lib._ERRORS[-1] is lt.InvalidChainError
    assert _lib._ERRORS[-4] is lt.ColoringLimitError
    assert _lib._ERRORS[-6] is lt.StaleScheduleError
    assert issubclass(lt.ColoringLimitError, lt.InspectionError)
    assert issubclass(lt.StaleScheduleError, lt.ExecutionError)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    mesh = lt.generate_rect_mesh(2, 2)
    from cases import setup
    chain, _, _, _ = setup(mesh, "fig2")
    with pytest.raises(lt.ExecutionError):
        lt.inspect_chain(chain, 4, lt.ExecMode.SHARED)


def test_native_rcm_matches_reference_orders():
    ref = golden_npz("rcm.npz")
    for key, order in ref.items():
        nx, ny = (int(v) for v in key.split("x"))
        mesh = lt.generate_rect_mesh(nx, ny)
        np.testing.assert_array_equal(lt.mesh.rcm_ordering(mesh), order, err_msg=key)


def test_rcm_rejects_disconnected_graph():
    with pytest.raises(ValueError):
        _lib.rcm_order(np.array([0, 0, 0]), np.array([], dtype=np.int64))


def test_registry_rejects_python_bodies():
    reg = lt.KernelRegistry()
    with pytest.raises(lt.ExecutionError):
        reg.register("k", lambda x: None, 1)
    reg.register("edge_inc", lt.native_kernel("edge_inc"), 2)
    with pytest.raises(lt.ExecutionError):
        reg.register("edge_inc", lt.native_kernel("edge_inc"), 2)
    with pytest.raises(lt.ExecutionError):
        reg.get("missing")
