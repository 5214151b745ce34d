"""Config parsing, schedule-v1 round trips and VTK export (CPU only)."""

import os

import numpy as np
import pytest

from conftest import ROOT, golden_schedule_text, golden_schedules

import paper_1708_03183_b200 as lt
from paper_1708_03183_b200.config import ConfigError, parse_config, parse_fusion
from paper_1708_03183_b200.inspector import ExecMode, Schedule
from paper_1708_03183_b200.vtk import export_vtk, parse_vtk
from cases import build_case


def test_parse_shipped_configs():
    cfg = parse_config(os.path.join(ROOT, "configs", "fig2.ini"))
    assert (cfg.nx, cfg.ny, cfg.renumber, cfg.mode, cfg.tile_size) == (16, 8, "rcm",
                                                                       ExecMode.SHARED, 16)
    assert [(s.start, s.stop, s.tile_size) for s in cfg.fusion] == [(0, 3, 16)]
    cfg = parse_config(os.path.join(ROOT, "configs", "eight_loop.ini"))
    assert [(s.start, s.stop, s.tile_size) for s in cfg.fusion] == [(0, 4, 16), (4, 6, 8),
                                                                  (6, 8, 16)]


def test_fusion_grammar_errors():
    with pytest.raises(ConfigError):
        parse_fusion("1-2:4", 4, 4, 4, ExecMode.SHARED)        # gap at 0
    with pytest.raises(ConfigError):
        parse_fusion("0-5:4", 4, 4, 4, ExecMode.SHARED)        # out of bounds
    with pytest.raises(ConfigError):
        parse_fusion("0-1:0", 4, 4, 4, ExecMode.SHARED)        # tile size
    with pytest.raises(lt.DepthExceededError):
        parse_fusion("0-3:4", 4, 4, 2, ExecMode.DISTRIBUTED)   # 4 loops > depth 2
    assert parse_fusion("0-1,2-3:8", 4, 4, 4, ExecMode.SHARED)[1].tile_size == 8


def test_explicit_chain_config(tmp_path):
    p = tmp_path / "x.ini"
    p.write_text("[mesh]\nnx = 4\nny = 2\nrenumber = none\n[chain]\ndepth = 2\n"
                 "[loops]\n0 = edges edge_inc r@-:w, i@e2v:acc\n1 = edges edge_read w@-:o, r@e2v:acc\n"
                 "[datasets]\nw = edges 1 ramp\nacc = verts 1 zeros\no = edges 1 zeros\n"
                 "[run]\nmode = shared\ntile_size = 3\n")
    cfg = parse_config(str(p))
    assert len(cfg.problem.loops) == 2 and cfg.problem.loops[0].accesses[1].map == "e2v"
    bad = tmp_path / "bad.ini"
    bad.write_text("[mesh]\nnx = 4\nny = 2\n[chain]\npreset = nope\n")
    with pytest.raises(ConfigError):
        parse_config(str(bad))


@pytest.mark.parametrize("case", ["fig2_16x8_rcm_ts16_shared", "toy_8x8_none_ts8_shared",
                                  "eight_8x4_rcm_ts3_sequential"])
def test_schedule_v1_round_trip(case):
    text = golden_schedule_text(case)
    sched = Schedule.deserialize(text)
    assert sched.serialize() == text
    assert sched.recolor_rounds == golden_schedules()["meta"][case]["rounds"]


def test_vtk_round_trip(tmp_path):
    mesh, (chain, _, _, _) = build_case("fig2", (16, 8), "rcm")
    sched = Schedule.deserialize(golden_schedule_text("fig2_16x8_rcm_ts16_shared"))
    path = str(tmp_path / "tiles.vtk")
    export_vtk(sched, chain, mesh, path)
    v = parse_vtk(path)
    assert v["cells"].shape == (mesh.num_cells, 3)
    np.testing.assert_array_equal(v["cells"].ravel(), mesh.cells_to_vertices)
    np.testing.assert_array_equal(v["cell_data"]["tile_id"], sched.tile_of(1, mesh.num_cells))
    colors = {t.id: t.color for t in sched.tiles}
    assert all(colors[t] == c for t, c in zip(v["cell_data"]["tile_id"],
                                              v["cell_data"]["color"]))
