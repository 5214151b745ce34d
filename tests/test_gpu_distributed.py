"""Distributed execution (virtual ranks on one B200) vs reference run_distributed."""

import numpy as np
import pytest

from conftest import golden_npz

import paper_1708_03183_b200 as lt
from paper_1708_03183_b200.distributed import run_distributed

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("exec_mode")]


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("mode", ["distributed", "shared"])
@pytest.mark.parametrize("use_local", [False, True])
def test_gpu_run_distributed_matches_reference(nranks, mode, use_local):
    ref = golden_npz("distributed.npz")
    mesh = lt.rcm_renumber(lt.generate_rect_mesh(8, 4))
    res = run_distributed(mesh, lt.FIG2, nranks, 4, depth=3, registry=lt.default_registry(),
                          poison_halo=True, use_local_maps=use_local,
                          mode=lt.ExecMode.parse(mode))
    for n, v in res.datasets.items():
        np.testing.assert_array_equal(v, ref[f"fig2_8x4_rcm/n{nranks}/gathered/{n}"], err_msg=n)
    assert res.exchange_counts == [1] * nranks


@pytest.mark.parametrize("nranks,depth", [(2, 8), (3, 8)])
def test_gpu_eight_loop_distributed_equals_serial(nranks, depth):
    mesh = lt.rcm_renumber(lt.generate_rect_mesh(16, 8))
    chain, ds, b = lt.global_setup(mesh, lt.EIGHT_LOOP, depth)
    lt.execute_untiled(chain, b, ds, lt.default_registry())
    res = run_distributed(mesh, lt.EIGHT_LOOP, nranks, 8, depth=depth,
                          registry=lt.default_registry(), poison_halo=True,
                          mode=lt.ExecMode.SHARED)
    for n, v in res.datasets.items():
        np.testing.assert_array_equal(v, ds[n].numpy(), err_msg=n)
