"""Per-tile record chunks of the dataflow executor (DG facet loops).

A tile's record scratch starts behind its own program and rows, so tiles
smaller than the largest get longer chunks (fewer records + ordered-apply
phases).  Contributions still reach every target row in the reference's
(element, k) order, so the result is bitwise that of uniform chunks, and both
are within 1e-12 of the untiled executor (reference ``execute_untiled``,
executor.py:163-169).
"""

import numpy as np
import pytest

import paper_1708_03183_b200 as lt
from paper_1708_03183_b200.dg import elastic_problem, elastic_setup
from paper_1708_03183_b200.executor import TiledRunner

pytestmark = pytest.mark.gpu
RTOL = 1e-12


def rel_err(got, ref):
    return np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)


@pytest.mark.parametrize("p,ts", [(1, 32), (2, 16), (3, 12), (4, 8)])
def test_per_tile_chunks_equal_uniform_chunks_and_untiled(p, ts, monkeypatch):
    monkeypatch.setenv("LT_EXEC", "dataflow")
    mk = lambda: elastic_problem(elastic_setup(48, 40, p, 2, material=("uniform", 5), sigma=6.0))
    ref = mk()
    ref.run_untiled(n_chains=2)
    out = {}
    for uniform in (True, False):
        if uniform:
            monkeypatch.setenv("LT_UNIFORM_CHUNKS", "1")
        else:
            monkeypatch.delenv("LT_UNIFORM_CHUNKS", raising=False)
        b = mk()
        b.install_params()
        s = lt.inspect_chain(b.chain, ts, lt.ExecMode.SHARED)
        r = TiledRunner(s, b.chain, b.bindings, b.datasets, b.registry, use_local_maps=True,
                        repeats=2)
        assert r.executor == "dataflow", r.executor
        r()
        out[uniform] = {n: b.datasets[n].numpy().copy() for n in ("u", "s", "ru", "rs")}
        for n in ("u", "s"):
            assert rel_err(out[uniform][n], ref.datasets[n].numpy()) <= RTOL, (uniform, n)
    for n in ("u", "s", "ru", "rs"):
        np.testing.assert_array_equal(out[True][n], out[False][n], err_msg=n)


@pytest.mark.parametrize("p,T,ts", [(1, 1, 32), (3, 2, 16)])
def test_dataflow_results_do_not_depend_on_scheduling(p, T, ts, monkeypatch):
    """Race check without a sanitizer (compute-sanitizer is closed on this GPU
    pool): the persistent dataflow executor must produce bitwise the same
    fields whatever the queue order (colour-major / wavefront), the number of
    resident CTAs per SM (shared-memory padding: 6-4, 2 and 1 per SM) and the
    chunking, over several repeats in one launch.  A missing dependency, a
    stale L1 line or an early release shows up as a differing bit in at least
    one of these schedules."""
    monkeypatch.setenv("LT_EXEC", "dataflow")
    mk = lambda: elastic_problem(elastic_setup(96, 64, p, T, material=("uniform", 11),
                                               sigma=9.0))
    ref = mk()
    ref.run_untiled(n_chains=4)
    results = []
    for order, pad, uniform in (("colour", "0", False), ("wave", "0", False),
                                ("wave", "60", False), ("colour", "150", True),
                                ("wave", "150", False), ("colour", "0", True)):
        monkeypatch.setenv("LT_ORDER", order)
        monkeypatch.setenv("LT_SMEM_PAD_KB", pad)
        if uniform:
            monkeypatch.setenv("LT_UNIFORM_CHUNKS", "1")
        else:
            monkeypatch.delenv("LT_UNIFORM_CHUNKS", raising=False)
        b = mk()
        b.install_params()
        s = lt.inspect_chain(b.chain, ts, lt.ExecMode.SHARED)
        r = TiledRunner(s, b.chain, b.bindings, b.datasets, b.registry, use_local_maps=True,
                        repeats=4)
        assert r.executor == "dataflow", r.executor
        r()
        results.append({n: b.datasets[n].numpy().copy() for n in ("u", "s", "ru", "rs")})
        for n in ("u", "s"):
            assert rel_err(results[-1][n], ref.datasets[n].numpy()) <= RTOL, (order, pad, n)
    for k, res in enumerate(results[1:], 1):
        for n in ("u", "s", "ru", "rs"):
            np.testing.assert_array_equal(res[n], results[0][n], err_msg=f"run {k} {n}")
