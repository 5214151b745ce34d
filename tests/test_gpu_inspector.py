"""GPU inspector parity: byte-identical schedules vs the reference (B200)."""

import numpy as np
import pytest

from conftest import golden_npz, golden_schedule_text, golden_schedules, parse_case
from cases import build_case

import paper_1708_03183_b200 as lt
from oracle import looptile_oracle as O

pytestmark = pytest.mark.gpu
ALL = sorted(c for c in golden_schedules()["schedules"])
MODES = {"sequential": lt.ExecMode.SEQUENTIAL, "shared": lt.ExecMode.SHARED}


@pytest.mark.parametrize("case", ALL)
def test_gpu_schedule_bytes_match_reference(case):
    prob, dims, ren, ts, mode = parse_case(case)
    _, (chain, _, _, _) = build_case(prob, dims, ren)
    s = lt.inspect_chain(chain, ts, MODES[mode])
    got = s.serialize()
    want = golden_schedule_text(case)
    assert got == want
    assert s.recolor_rounds == golden_schedules()["meta"][case]["rounds"]


def test_gpu_invert_map_round_trips():
    inv = golden_npz("invert.npz")
    for i in range(100):
        n_src, n_tgt, arity = (int(v) for v in inv[f"{i}/shape"])
        m = lt.MeshMap("m", lt.IterationSpace("s", n_src), lt.IterationSpace("t", n_tgt),
                       arity, inv[f"{i}/values"])
        im = lt.invert_map(m)
        np.testing.assert_array_equal(im.offsets, inv[f"{i}/inv_offsets"])
        np.testing.assert_array_equal(im.values, inv[f"{i}/inv_values"])


@pytest.mark.parametrize("ts,mode", [(1, "shared"), (4, "shared"), (7, "sequential"),
                                     (16, "shared")])
def test_gpu_schedule_is_legal(ts, mode):
    _, (chain, _, _, _) = build_case("eight", (8, 4), "none")
    s = lt.inspect_chain(chain, ts, MODES[mode])
    tile_of = [s.tile_of(j, lp.space.total) for j, lp in enumerate(chain.loops)]
    colors = {t.id: t.color for t in s.tiles}
    regions = {t.id: int(t.region) for t in s.tiles}
    assert O.check_legality(chain, tile_of, colors, s.tiles[-1].id) == []
    lists = {t.id: t.iteration_lists for t in s.tiles}
    assert O.footprint_conflicts(chain, lists, colors, regions) == []


def test_gpu_inspection_matches_oracle_at_scale():
    # beyond the reference fixtures: 64x64 toy chain, RCM, shared
    _, (chain, _, _, _) = build_case("toy", (64, 64), "rcm")
    for ts in (32, 256):
        g = lt.inspect_chain(chain, ts, lt.ExecMode.SHARED)
        o = O.inspect(chain, ts, "shared")
        assert g.serialize() == o.serialize()


def test_gpu_partition_invariant_and_regions():
    # reference tests/test_inspector.py:313-321 and acceptance criterion 6
    _, (chain, _, _, _) = build_case("fig2", (8, 4), "none")
    s = lt.inspect_chain(chain, 6, lt.ExecMode.SHARED)
    for j, loop in enumerate(chain.loops):
        cat = np.concatenate([t.iteration_lists[j] for t in s.tiles])
        assert sorted(cat.tolist()) == list(range(loop.space.total))
    core = [t.color for t in s.tiles if t.region is lt.Region.CORE]
    assert s.nonexec_tile.color > max(core)


def test_gpu_inspection_errors():
    with pytest.raises(ValueError):
        _, (chain, _, _, _) = build_case("fig2", (2, 2), "none")
        lt.inspect_chain(chain, 0, lt.ExecMode.SHARED)
    # a loop whose spaces no earlier loop touched cannot be tiled
    s = lt.IterationSpace("s", 4)
    t = lt.IterationSpace("t", 4)
    loops = (lt.Loop(0, s, (lt.Descriptor(None, lt.AccessMode.READ),), "k"),
             lt.Loop(1, t, (lt.Descriptor(None, lt.AccessMode.READ),), "k"))
    chain = lt.build_chain((s, t), (), loops, 2)
    with pytest.raises(lt.InspectionError):
        lt.inspect_chain(chain, 2, lt.ExecMode.SHARED)


def test_gpu_determinism():
    _, (chain, _, _, _) = build_case("fig2", (8, 4), "none")
    a = lt.inspect_chain(chain, 4, lt.ExecMode.SHARED).serialize()
    b = lt.inspect_chain(chain, 4, lt.ExecMode.SHARED).serialize()
    assert a == b


def _oracle_violations(chain, s):
    tile_of = [s.tile_of(j, lp.space.total) for j, lp in enumerate(chain.loops)]
    colors = {t.id: t.color for t in s.tiles}
    bad = O.check_legality(chain, tile_of, colors, s.tiles[-1].id)
    red = sum(1 for b in bad if b.startswith("reduction"))
    return {"pairs": len(bad) - red, "reductions": red}


@pytest.mark.parametrize("case,dims,ren,ts,mode,sub", [
    ("eight", (8, 4), "none", 4, "shared", None),
    ("eight", (8, 4), "none", 7, "sequential", None),
    ("toy", (8, 8), "rcm", 8, "shared", None),
    ("fig2", (16, 8), "rcm", 16, "shared", None),
    ("fig2", (16, 8), "rcm", 4, "shared", 2),   # reference emits an illegal schedule here
    ("fig2", (16, 8), "rcm", 2, "shared", 2),
    ("dg2s2", (6, 6), "none", 12, "shared", None),
])
def test_gpu_legality_checker_matches_oracle(case, dims, ren, ts, mode, sub):
    """lt_check_legality == the oracle's restatement of pkg/tests/legality.py
    (violation counts), including the reference's own illegal FIG2 sub-chain
    schedules, and every tile edit that breaks legality is seen."""
    _, (chain, _, _, _) = build_case(case, dims, ren)
    if sub:
        chain = chain.subchain(0, sub)
    s = lt.inspect_chain(chain, ts, MODES[mode])
    want = _oracle_violations(chain, s)
    assert lt.check_legality_gpu(s, chain) == want
    if sub:
        assert want["reductions"] > 0 or want["pairs"] > 0 or ts == 2
    # break it: give every tile the same colour (all cross-tile dependences violate)
    for t in s.tiles:
        t.color = 0
    want = _oracle_violations(chain, s)
    assert want["pairs"] + want["reductions"] > 0
    assert lt.check_legality_gpu(s, chain) == want
