"""GPU executor parity vs the reference values (bitwise) and the oracle (B200)."""

import numpy as np
import pytest

from conftest import golden_npz, parse_case
from cases import build_case

import paper_1708_03183_b200 as lt
from oracle import looptile_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("exec_mode")]
MODES = {"sequential": lt.ExecMode.SEQUENTIAL, "shared": lt.ExecMode.SHARED}


def device_run(prob, dims, ren, ts=None, mode=None, use_local=False, schedule=None):
    mesh, (chain, data, vpe, bind) = build_case(prob, dims, ren)
    ds = {n: lt.Dataset(n, chain.space_named(_space_of(chain, bind, n)), vpe[n], v)
          for n, v in data.items()}
    reg = lt.default_registry()
    if ts is None:
        lt.execute_untiled(chain, bind, ds, reg)
        s = None
    else:
        s = schedule or lt.inspect_chain(chain, ts, MODES[mode])
        lt.execute_schedule(s, chain, bind, ds, reg, use_local_maps=use_local)
    return {n: d.numpy() for n, d in ds.items()}, chain, s


def _space_of(chain, bind, name):
    for loop, b in zip(chain.loops, bind):
        for d, n in zip(loop.descriptors, b.args):
            if n == name:
                return (loop.space if d.is_direct else d.map.target).name
    raise KeyError(name)


@pytest.mark.parametrize("tag", ["fig2_16x8_rcm", "fig2_8x4_none", "eight_16x8_rcm",
                                 "eight_8x4_rcm", "toy_32x32_none", "toy_32x32_rcm",
                                 "toy_8x8_none"])
def test_gpu_untiled_bitwise_vs_reference(tag):
    prob, d, ren = tag.split("_")
    dims = tuple(int(v) for v in d.split("x"))
    got, _, _ = device_run(prob, dims, ren)
    ref = golden_npz("values.npz")
    for n, v in got.items():
        np.testing.assert_array_equal(v, ref[f"{tag}/untiled/{n}"], err_msg=n)


@pytest.mark.parametrize("case", ["toy_32x32_none_ts64_shared", "toy_32x32_rcm_ts64_shared",
                                  "toy_32x32_none_ts64_sequential", "toy_8x8_rcm_ts8_shared",
                                  "toy_8x8_none_ts16_sequential"])
@pytest.mark.parametrize("use_local", [False, True])
def test_gpu_tiled_bitwise_vs_reference_execute_schedule(case, use_local):
    prob, dims, ren, ts, mode = parse_case(case)
    got, _, _ = device_run(prob, dims, ren, ts, mode, use_local)
    ref = golden_npz("values.npz")
    for n, v in got.items():
        np.testing.assert_array_equal(v, ref[f"{case}/tiled/{n}"], err_msg=n)


@pytest.mark.parametrize("dims", [(1, 1), (2, 1), (4, 2), (8, 4), (16, 8)])
@pytest.mark.parametrize("ts", [1, 4, 16, 64])
@pytest.mark.parametrize("mode", ["sequential", "shared"])
def test_gpu_fig2_acceptance_sweep(dims, ts, mode):
    # reference acceptance criterion 1: tiled == untiled bitwise (integer data)
    got, _, _ = device_run("fig2", dims, "rcm", ts, mode)
    ref = golden_npz("values.npz")
    tag = f"fig2_{dims[0]}x{dims[1]}_rcm"
    for n, v in got.items():
        np.testing.assert_array_equal(v, ref[f"{tag}/untiled/{n}"], err_msg=n)


def test_gpu_toy_tiled_within_1e12_of_untiled_at_scale():
    for ren in ("none", "rcm"):
        unt, _, _ = device_run("toy", (128, 96), ren)
        for ts, mode in ((32, "shared"), (64, "shared"), (64, "sequential")):
            til, _, _ = device_run("toy", (128, 96), ren, ts, mode)
            for n in unt:
                err = np.max(np.abs(til[n] - unt[n])) / max(np.max(np.abs(unt[n])), 1e-300)
                assert err <= 1e-12, (ren, ts, n, err)


def test_gpu_executes_oracle_schedule_like_reference():
    # executor independent of the GPU inspector: run the oracle's schedule
    mesh, (chain, data, vpe, bind) = build_case("toy", (16, 16), "rcm")
    os_ = O.inspect(chain, 16, "shared")
    tiles = [lt.Tile(t.id, lt.Region(t.region), t.color, dict(t.lists), {}) for t in os_.tiles]
    sched = lt.Schedule(lt.ExecMode.SHARED, chain.fingerprint, len(chain.loops), tiles,
                        os_.rounds)
    ref = {n: v.copy() for n, v in data.items()}
    O.execute_tiled(os_, chain, bind, ref, vpe)
    ds = {n: lt.Dataset(n, chain.space_named(_space_of(chain, bind, n)), vpe[n], v)
          for n, v in data.items()}
    lt.execute_schedule(sched, chain, bind, ds, lt.default_registry())
    for n in ref:
        np.testing.assert_array_equal(ds[n].numpy(), ref[n], err_msg=n)


def test_gpu_stale_schedule_and_binding_errors():
    mesh, (chain, data, vpe, bind) = build_case("fig2", (4, 2), "none")
    _, (other, _, _, _) = build_case("fig2", (4, 2), "rcm")
    s = lt.inspect_chain(other, 4, lt.ExecMode.SHARED)
    ds = {n: lt.Dataset(n, chain.space_named(_space_of(chain, bind, n)), vpe[n], v)
          for n, v in data.items()}
    reg = lt.default_registry()
    with pytest.raises(lt.StaleScheduleError):
        lt.execute_schedule(s, chain, bind, ds, reg)
    with pytest.raises(lt.ExecutionError):
        lt.execute_untiled(chain, bind[:-1], ds, reg)
    empty = lt.KernelRegistry()
    with pytest.raises(lt.ExecutionError):
        lt.execute_untiled(chain, bind, ds, empty)


def test_gpu_nonexec_tile_never_runs():
    # a space with non-exec elements: their values must stay untouched
    cells = lt.IterationSpace("cells", 6, 2, 3)
    verts = lt.IterationSpace("verts", 5)
    rng = np.random.default_rng(5)
    c2v = lt.MeshMap("c2v", cells, verts, 3, rng.integers(0, 5, size=33))
    loops = (lt.Loop(0, cells, (lt.Descriptor(None, lt.AccessMode.READ),
                                lt.Descriptor(c2v, lt.AccessMode.INC)), "cell_inc"),
             lt.Loop(1, cells, (lt.Descriptor(None, lt.AccessMode.WRITE),
                                lt.Descriptor(c2v, lt.AccessMode.READ)), "cell_read"))
    chain = lt.build_chain((cells, verts), (c2v,), loops, 2)
    bind = (lt.KernelBinding("cell_inc", ("w", "acc")), lt.KernelBinding("cell_read", ("out", "acc")))
    data = {"w": np.arange(11, dtype=float) + 1, "acc": np.zeros(5), "out": np.full(11, -7.0)}
    vpe = {"w": 1, "acc": 1, "out": 1}
    ds = {"w": lt.Dataset("w", cells, 1, data["w"]), "acc": lt.Dataset("acc", verts, 1, data["acc"]),
          "out": lt.Dataset("out", cells, 1, data["out"])}
    for mode in ("sequential", "shared"):
        s = lt.inspect_chain(chain, 3, MODES[mode])
        osch = O.inspect(chain, 3, mode)
        assert s.serialize() == osch.serialize()
        d2 = {n: d.copy() for n, d in ds.items()}
        lt.execute_schedule(s, chain, bind, d2, lt.default_registry())
        ref = {n: v.copy() for n, v in data.items()}
        O.execute_tiled(osch, chain, bind, ref, vpe)
        for n in ref:
            np.testing.assert_array_equal(d2[n].numpy(), ref[n], err_msg=(mode, n))
        # elements whose inputs depend on non-exec data fall into T_ne and keep values
        tne = s.tiles[-1]
        assert np.all(d2["out"].numpy()[tne.iteration_lists[1]] == -7.0)


@pytest.mark.parametrize("ts", [2, 4, 8])
def test_gpu_executes_illegal_reference_schedule_correctly(ts):
    """The reference inspector emits, for FIG2's sub-chain [edge_inc, cell_inc],
    schedules whose last-loop reductions split across equal-coloured tiles
    (violations of its own legality oracle).  The executor orders such tiles
    (write-conflict sub-colours in id order) and matches the sequential result."""
    mesh, (chain, data, vpe, bind) = build_case("fig2", (16, 8), "rcm")
    sub = chain.subchain(0, 2)
    sched = lt.inspect_chain(sub, ts, lt.ExecMode.SHARED)
    ds = {n: lt.Dataset(n, chain.space_named(_space_of(chain, bind, n)), vpe[n], v)
          for n, v in data.items()}
    lt.execute_schedule(sched, sub, bind[:2], ds, lt.default_registry())
    ref = {n: v.copy() for n, v in data.items()}
    O.execute_untiled(sub, bind[:2], ref, vpe)
    for n in ref:
        np.testing.assert_array_equal(ds[n].numpy(), ref[n], err_msg=n)
