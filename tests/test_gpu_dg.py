"""Elastic-wave DG on the B200 vs the reference-executor goldens (float64)."""

import numpy as np
import pytest

from conftest import golden_npz, golden_schedules, parse_case
from cases import dg_setup

import paper_1708_03183_b200 as lt
from paper_1708_03183_b200.dg import ElasticProblem, elastic_problem

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("exec_mode")]
DG_CASES = sorted(c for c in golden_schedules()["schedules"] if c.startswith("dg"))
MODES = {"sequential": lt.ExecMode.SEQUENTIAL, "shared": lt.ExecMode.SHARED}
RTOL = 1e-12  # north_star: float64 fields within 1e-12 relative (normwise per field)


def rel_err(got, ref):
    return np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)


def problem(tag) -> ElasticProblem:
    st, _ = dg_setup(tag)
    return elastic_problem(st)


@pytest.mark.parametrize("tag", sorted({c.rsplit("_", 2)[0] for c in DG_CASES}))
def test_gpu_dg_untiled_vs_reference(tag):
    pb = problem(tag)
    pb.run_untiled()
    ref = golden_npz("values.npz")
    for n in ("u", "s", "ru", "rs"):
        assert rel_err(pb.datasets[n].numpy(), ref[f"{tag}/untiled/{n}"]) <= RTOL, n


@pytest.mark.parametrize("case", DG_CASES)
@pytest.mark.parametrize("use_local", [False, True])
def test_gpu_dg_tiled_vs_reference(case, use_local):
    tag = case.rsplit("_", 2)[0]
    _, _, _, ts, mode = parse_case(case)
    pb = problem(tag)
    s = lt.inspect_chain(pb.chain, ts, MODES[mode])
    pb.run_tiled(s, use_local_maps=use_local)
    ref = golden_npz("values.npz")
    for n in ("u", "s", "ru", "rs"):
        assert rel_err(pb.datasets[n].numpy(), ref[f"{case}/tiled/{n}"]) <= RTOL, n


@pytest.mark.parametrize("p,steps", [(1, 1), (2, 2), (3, 1), (4, 1)])
def test_gpu_dg_tiled_equals_untiled_at_scale(p, steps):
    from paper_1708_03183_b200.dg import elastic_setup
    st = elastic_setup(48, 40, p, steps, material=("uniform", 3), sigma=6.0)
    a = elastic_problem(st)
    a.run_untiled(n_chains=2)
    for ts, mode in ((32, lt.ExecMode.SHARED), (128 // (p * steps), lt.ExecMode.SHARED)):
        st2 = elastic_setup(48, 40, p, steps, material=("uniform", 3), sigma=6.0)
        b = elastic_problem(st2)
        b.run_tiled(lt.inspect_chain(b.chain, ts, mode), n_chains=2)
        for n in ("u", "s"):
            assert rel_err(b.datasets[n].numpy(), a.datasets[n].numpy()) <= RTOL, (ts, n)


def test_gpu_dg_p4_matches_oracle():
    from oracle import looptile_oracle as O
    st, chain = dg_setup("dg4s1_4x4_none")
    data = {n: v.copy() for n, v in st.data.items()}
    O.execute_untiled(chain, st.bindings, data, st.vpe, O.kernel_table(dg=(4, st.dt)))
    pb = elastic_problem(dg_setup("dg4s1_4x4_none")[0])
    pb.run_tiled(lt.inspect_chain(pb.chain, 8, lt.ExecMode.SHARED))
    for n in ("u", "s", "ru", "rs"):
        assert rel_err(pb.datasets[n].numpy(), data[n]) <= RTOL, n


@pytest.mark.parametrize("repeats", [1, 3])
def test_gpu_dg_repeat_equals_sequential_calls(repeats):
    from paper_1708_03183_b200.dg import elastic_setup
    from paper_1708_03183_b200.executor import TiledRunner
    st = elastic_setup(40, 30, 1, 1, sigma=5.0)
    a = elastic_problem(st)
    a.install_params()
    s = lt.inspect_chain(a.chain, 24, lt.ExecMode.SHARED)
    for _ in range(repeats):
        lt.execute_schedule(s, a.chain, a.bindings, a.datasets, a.registry, use_local_maps=True)
    b = elastic_problem(elastic_setup(40, 30, 1, 1, sigma=5.0))
    s2 = lt.inspect_chain(b.chain, 24, lt.ExecMode.SHARED)
    TiledRunner(s2, b.chain, b.bindings, b.datasets, b.registry, repeats=repeats)()
    for n in ("u", "s", "ru", "rs"):
        np.testing.assert_array_equal(b.datasets[n].numpy(), a.datasets[n].numpy(), err_msg=n)


@pytest.mark.parametrize("p,steps", [(1, 1), (2, 2)])
def test_gpu_dg_repeat_repacks_constants_each_call(p, steps):
    """Repeated execution packs the read-only rows (geometry, material) into the
    tile programs once per call: a change of a read-only dataset between calls
    must be seen by the next call."""
    from paper_1708_03183_b200.dg import elastic_setup
    from paper_1708_03183_b200.executor import TiledRunner
    mk = lambda: elastic_problem(elastic_setup(36, 28, p, steps, material=("uniform", 5),
                                               sigma=5.0))
    a, b = mk(), mk()
    a.install_params()
    sa = lt.inspect_chain(a.chain, 24, lt.ExecMode.SHARED)
    sb = lt.inspect_chain(b.chain, 24, lt.ExecMode.SHARED)
    runner = TiledRunner(sb, b.chain, b.bindings, b.datasets, b.registry, repeats=2)
    runner()
    for _ in range(2):
        lt.execute_schedule(sa, a.chain, a.bindings, a.datasets, a.registry, use_local_maps=True)
    for pb in (a, b):  # change the material between calls (rho -> 1.5 rho)
        pb.datasets["mat"].values.view(-1, pb.datasets["mat"].values_per_element)[:, 0] *= 1.5
    for _ in range(2):
        lt.execute_schedule(sa, a.chain, a.bindings, a.datasets, a.registry, use_local_maps=True)
    runner()
    for n in ("u", "s", "ru", "rs"):
        np.testing.assert_array_equal(b.datasets[n].numpy(), a.datasets[n].numpy(), err_msg=n)


@pytest.mark.parametrize("order", ["wave", "colour"])
def test_gpu_dg_queue_orders_equal_sequential_calls(order, monkeypatch):
    """The dataflow queue order (wavefront or colour-major) never changes
    results: repeated execution is bitwise equal to sequential calls."""
    from paper_1708_03183_b200.dg import elastic_setup
    from paper_1708_03183_b200.executor import TiledRunner
    monkeypatch.setenv("LT_ORDER", order)
    mk = lambda: elastic_problem(elastic_setup(44, 36, 2, 2, material=("uniform", 7), sigma=5.0))
    a, b = mk(), mk()
    a.install_params()
    sa = lt.inspect_chain(a.chain, 16, lt.ExecMode.SHARED)
    for _ in range(4):
        lt.execute_schedule(sa, a.chain, a.bindings, a.datasets, a.registry, use_local_maps=True)
    sb = lt.inspect_chain(b.chain, 16, lt.ExecMode.SHARED)
    r = TiledRunner(sb, b.chain, b.bindings, b.datasets, b.registry, repeats=2)
    if r.executor == "dataflow":
        assert r.queue_order == ("wavefront" if order == "wave" else "colour-major")
    r()
    r()
    for n in ("u", "s", "ru", "rs"):
        np.testing.assert_array_equal(b.datasets[n].numpy(), a.datasets[n].numpy(), err_msg=n)


def test_gpu_dg_wide_register_build_matches_untiled(exec_mode):
    """P2 two-step tiles large enough that shared memory allows <= 4 CTAs per
    SM run the 128-register dataflow build; results equal the untiled path."""
    from paper_1708_03183_b200.dg import elastic_setup
    from paper_1708_03183_b200.executor import TiledRunner
    mk = lambda: elastic_problem(elastic_setup(64, 48, 2, 2, material=("uniform", 9), sigma=6.0))
    a, b = mk(), mk()
    a.run_untiled(n_chains=3)
    s = lt.inspect_chain(b.chain, 32, lt.ExecMode.SHARED)
    b.install_params()
    r = TiledRunner(s, b.chain, b.bindings, b.datasets, b.registry, repeats=3)
    if exec_mode.startswith("dataflow"):
        assert r.executor == "dataflow", r.executor
        assert r.wide_build, r.smem_bytes
    else:
        assert r.executor == exec_mode, r.executor
    r()
    for n in ("u", "s"):
        assert rel_err(b.datasets[n].numpy(), a.datasets[n].numpy()) <= RTOL, n
