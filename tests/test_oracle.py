"""Pin the CPU oracle to fixtures produced by the real reference (CPU only)."""

import numpy as np
import pytest

from conftest import golden_npz, golden_schedule_text, golden_schedules, parse_case
from cases import build_case
from oracle import looptile_oracle as O

ALL = sorted(golden_schedules()["schedules"])
FAST = [c for c in ALL if not c.startswith("dg_")]


@pytest.mark.parametrize("case", FAST)
def test_oracle_schedule_matches_reference_bytes(case):
    prob, dims, ren, ts, mode = parse_case(case)
    _, (chain, _, _, _) = build_case(prob, dims, ren)
    s = O.inspect(chain, ts, mode)
    assert s.serialize() == golden_schedule_text(case)


def test_fingerprints_match_reference(golden):
    for tag, fp in golden["fingerprints"].items():
        prob, rest = tag.split("_", 1)
        if prob == "dg":
            continue
        d, ren = rest.split("_")
        dims = tuple(int(v) for v in d.split("x"))
        _, (chain, _, _, _) = build_case(prob, dims, ren)
        assert chain.fingerprint == fp, tag


@pytest.mark.parametrize("tag", ["fig2_16x8_rcm", "fig2_8x4_none", "eight_16x8_rcm",
                                 "toy_32x32_none", "toy_32x32_rcm", "toy_8x8_rcm"])
def test_oracle_untiled_matches_reference(tag):
    prob, d, ren = tag.split("_")
    dims = tuple(int(v) for v in d.split("x"))
    _, (chain, data, vpe, bind) = build_case(prob, dims, ren)
    O.execute_untiled(chain, bind, data, vpe)
    ref = golden_npz("values.npz")
    for n, v in data.items():
        np.testing.assert_array_equal(v, ref[f"{tag}/untiled/{n}"], err_msg=n)


@pytest.mark.parametrize("case", ["toy_32x32_none_ts64_shared", "toy_32x32_rcm_ts64_shared",
                                  "toy_32x32_rcm_ts64_sequential", "toy_8x8_none_ts8_shared"])
def test_oracle_tiled_matches_reference_bitwise(case):
    prob, dims, ren, ts, mode = parse_case(case)
    _, (chain, data, vpe, bind) = build_case(prob, dims, ren)
    s = O.inspect(chain, ts, mode)
    O.execute_tiled(s, chain, bind, data, vpe)
    ref = golden_npz("values.npz")
    for n, v in data.items():
        np.testing.assert_array_equal(v, ref[f"{case}/tiled/{n}"], err_msg=n)


def test_oracle_invert_round_trips():
    inv = golden_npz("invert.npz")
    for i in range(100):
        n_src, n_tgt, arity = inv[f"{i}/shape"]
        off, src = O.invert(inv[f"{i}/values"], int(n_src), int(arity), int(n_tgt))
        np.testing.assert_array_equal(off, inv[f"{i}/inv_offsets"])
        np.testing.assert_array_equal(src, inv[f"{i}/inv_values"])


def test_oracle_legality_and_footprint_on_toy_shared():
    _, (chain, _, _, _) = build_case("toy", (8, 8), "none")
    s = O.inspect(chain, 8, "shared")
    tile_of = [s.tile_of(j, lp.space.total) for j, lp in enumerate(chain.loops)]
    colors = {t.id: t.color for t in s.tiles}
    regions = {t.id: t.region for t in s.tiles}
    assert O.check_legality(chain, tile_of, colors, s.tiles[-1].id) == []
    assert O.footprint_conflicts(chain, {t.id: t.lists for t in s.tiles}, colors, regions) == []


def test_oracle_detects_illegal_schedule():
    _, (chain, _, _, _) = build_case("fig2", (4, 2), "rcm")
    s = O.inspect(chain, 4, "shared")
    colors = {t.id: 0 for t in s.tiles}  # collapse all colours: must violate
    tile_of = [s.tile_of(j, lp.space.total) for j, lp in enumerate(chain.loops)]
    assert O.check_legality(chain, tile_of, colors, s.tiles[-1].id)


def test_known_answer_assign():
    # reference tests/test_inspector.py:249-256
    lists = O.assign(np.array([2, 0, 1, 0, 2, 1, 0, 0, 2]), 3)
    assert [x.tolist() for x in lists] == [[1, 3, 6, 7], [2, 5], [0, 4, 8]]


def test_known_answer_seed_chunks():
    # reference tests/test_inspector.py:21-26 and :39-49
    from paper_1708_03183_b200.chain import IterationSpace
    sigma, regions = O.partition_seed(IterationSpace("s", 10), 4)
    assert [int(np.sum(sigma == t)) for t in range(len(regions))] == [4, 4, 2, 0]
    sigma, regions = O.partition_seed(IterationSpace("s", 9, 4, 3), 3)
    assert regions == [0] * 3 + [1] * 2 + [2]
    assert sigma[:9].tolist() == [e // 3 for e in range(9)]
    assert sigma[9:13].tolist() == [3 + (e - 9) // 3 for e in range(9, 13)]
    assert np.all(sigma[13:] == 5)
