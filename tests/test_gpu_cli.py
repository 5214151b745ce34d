"""CLI driver on the GPU: verify, distributed fusion schemes, schedule cache, exit codes."""

import os

import pytest

from conftest import ROOT

from paper_1708_03183_b200 import cli
from paper_1708_03183_b200.config import parse_config

pytestmark = pytest.mark.gpu
CFG = os.path.join(ROOT, "configs")


def test_verify_fig2_and_toy_exit_zero(tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    assert cli.main(["verify", os.path.join(CFG, "fig2.ini")]) == 0
    assert cli.main(["verify", os.path.join(CFG, "toy.ini")]) == 0
    assert cli.main(["run", os.path.join(CFG, "fig2.ini")]) == 0
    assert os.path.exists("out/fig2_summary.txt") and os.path.exists("out/fig2_tiles.vtk")
    # the dumps of verify reproduce the reference's shipped value dumps format
    assert cli.main(["inspect-only", os.path.join(CFG, "fig2.ini")]) == 0


def test_verify_distributed_fusion_scheme():
    assert cli.main(["verify", os.path.join(CFG, "eight_loop.ini")]) == 0


def test_sweep_rows_all_pass(capsys):
    cfg = parse_config(os.path.join(CFG, "fig2.ini"))
    from paper_1708_03183_b200.inspector import ExecMode
    rows = cli.sweep_config(cfg, [4, 16], [ExecMode.SEQUENTIAL, ExecMode.SHARED],
                            ["0-2", "0-1,2"])
    assert len(rows) == 8 and all(r["verify"] == "pass" for r in rows)


def test_schedule_cache_persists_across_runs(tmp_path):
    cfg = parse_config(os.path.join(CFG, "fig2.ini"))
    cfg.cache_dir = str(tmp_path / "cache")
    c1 = cli.ScheduleCache(cfg.cache_dir)
    r1 = cli.run_config(cfg, c1)
    assert c1.misses == 1 and os.listdir(cfg.cache_dir)
    c2 = cli.ScheduleCache(cfg.cache_dir)
    r2 = cli.run_config(cfg, c2)
    assert c2.loads == 1 and c2.misses == 0
    for n in r1.values:
        assert (r1.values[n] == r2.values[n]).all()


def test_mutated_schedule_fails_verification():
    cfg = parse_config(os.path.join(CFG, "toy.ini"))
    cache = cli.ScheduleCache()
    cli.run_config(cfg, cache)
    sched = next(iter(cache._store.values()))
    for t in sched.tiles:        # collapse every colour: concurrent tiles now race
        t.color = 0
    cache.hits = 0
    with pytest.raises(Exception):
        cli.verify_config(cfg, cache)


def test_exit_codes(tmp_path):
    bad = tmp_path / "bad.ini"
    bad.write_text("[mesh]\nnx = 4\n")
    assert cli.main(["run", str(bad)]) == 2
    deep = tmp_path / "deep.ini"
    deep.write_text("[mesh]\nnx = 4\nny = 2\n[chain]\npreset = eight_loop\ndepth = 2\n"
                    "[run]\nmode = distributed\nfusion = 0-7:4\n")
    assert cli.main(["run", str(deep)]) == 4
