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


@pytest.mark.parametrize("p,steps,nranks", [(1, 1, 2), (1, 2, 3), (2, 1, 4)])
def test_gpu_elastic_distributed_equals_serial(p, steps, nranks):
    from paper_1708_03183_b200.dg import elastic_problem, elastic_setup, run_elastic_distributed
    st = elastic_setup(24, 20, p, steps, material=("uniform", 3), sigma=4.0)
    serial = elastic_problem(elastic_setup(24, 20, p, steps, material=("uniform", 3), sigma=4.0))
    serial.run_untiled(n_chains=2)
    got, ranks = run_elastic_distributed(st, nranks, depth=5 * steps, ts=16, n_chains=2,
                                         poison_halo=True)
    for n in ("u", "s"):
        ref = serial.datasets[n].numpy()
        assert np.all(np.isfinite(got[n])), n
        err = np.max(np.abs(got[n] - ref)) / np.max(np.abs(ref))
        assert err <= 1e-12, (n, err)
    assert all(r[3].exchange_count == 2 for r in ranks)
