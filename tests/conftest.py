import base64
import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


_CACHE = {}


def golden_schedules() -> dict:
    if "sched" not in _CACHE:
        with gzip.open(os.path.join(GOLDEN, "schedules.json.gz"), "rt") as fh:
            _CACHE["sched"] = json.load(fh)
    return _CACHE["sched"]


def golden_schedule_text(name: str) -> bytes:
    return gzip.decompress(base64.b64decode(golden_schedules()["schedules"][name]))


def golden_npz(name: str):
    if name not in _CACHE:
        _CACHE[name] = dict(np.load(os.path.join(GOLDEN, name)))
    return _CACHE[name]


def parse_case(name: str):
    """'fig2_16x8_rcm_ts16_shared' -> ('fig2', (16, 8), 'rcm', 16, 'shared')."""
    parts = name.split("_")
    prob = parts[0]
    nx, ny = (int(v) for v in parts[1].split("x"))
    return prob, (nx, ny), parts[2], int(parts[3][2:]), parts[4]


@pytest.fixture(scope="session")
def golden():
    return golden_schedules()


@pytest.fixture(params=["dataflow", "dataflow-wave", "staged", "global"])
def exec_mode(request, monkeypatch):
    """Run a GPU executor test with shared-memory staging (dataflow queue in
    colour-major and in wavefront order, per-colour launches) and with the
    global path."""
    mode = request.param
    if mode == "dataflow-wave":
        monkeypatch.setenv("LT_ORDER", "wave")
        mode = "dataflow"
    monkeypatch.setenv("LT_EXEC", mode)
    return request.param
