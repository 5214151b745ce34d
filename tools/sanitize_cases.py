"""Small executor cases for compute-sanitizer (memcheck / racecheck / synccheck).

usage: compute-sanitizer --tool racecheck python tools/sanitize_cases.py
Runs the dataflow tile executor (and the staged/global/untiled ones) on:
toy 32x32 (BASELINE config 1), FIG2 16x8 RCM, DG P1 one-step chains repeated
in one persistent launch, DG P2 two-step chains in wavefront queue order, a DG P3
two-step chain (per-tile record chunks),
and a 2-virtual-rank partitioned DG chain (core-only + boundary-only calls).
Each result is checked (bitwise or 1e-12) so the run also proves the
instrumented kernels computed the right thing.  Exit code 0 = all checks ok.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import paper_1708_03183_b200 as lt
from cases import build_case
from oracle import looptile_oracle as O
from paper_1708_03183_b200.dg import elastic_problem, elastic_setup, run_elastic_distributed
from paper_1708_03183_b200.executor import TiledRunner


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def toy_and_fig2(exec_mode):
    os.environ["LT_EXEC"] = exec_mode
    for prob, dims, ts in (("toy", (32, 32), 64), ("fig2", (16, 8), 16)):
        mesh, (chain, data, vpe, bind) = build_case(prob, dims, "rcm")
        sched = lt.inspect_chain(chain, ts, lt.ExecMode.SHARED)
        spaces = {}
        for lp, b in zip(chain.loops, bind):
            for d, n in zip(lp.descriptors, b.args):
                spaces[n] = d.map.target if d.map is not None else lp.space
        ds = {n: lt.Dataset(n, spaces[n], vpe[n], v) for n, v in data.items()}
        lt.execute_schedule(sched, chain, bind, ds, lt.default_registry())
        osched = O.inspect(chain, ts, "shared")
        ref = {n: v.copy() for n, v in data.items()}
        O.execute_tiled(osched, chain, bind, ref, vpe)
        for n in ref:
            assert np.array_equal(ds[n].numpy(), ref[n]), (exec_mode, prob, n)
    os.environ.pop("LT_EXEC")


def dg(p, steps, repeats, order):
    os.environ["LT_ORDER"] = order
    mk = lambda: elastic_problem(elastic_setup(24, 20, p, steps, material=("uniform", 4),
                                               sigma=4.0))
    a, b = mk(), mk()
    a.run_untiled(n_chains=repeats)
    s = lt.inspect_chain(b.chain, 12, lt.ExecMode.SHARED)
    b.install_params()
    r = TiledRunner(s, b.chain, b.bindings, b.datasets, b.registry, repeats=repeats)
    assert r.executor == "dataflow"
    r()
    for n in ("u", "s"):
        assert rel(b.datasets[n].numpy(), a.datasets[n].numpy()) <= 1e-12, (p, n)
    os.environ.pop("LT_ORDER")


def distributed():
    st = elastic_setup(16, 12, 1, 1, sigma=3.0)
    got, _ = run_elastic_distributed(st, 2, 5, 12, n_chains=2, poison_halo=True)
    ser = elastic_problem(elastic_setup(16, 12, 1, 1, sigma=3.0))
    ser.run_untiled(n_chains=2)
    for n in ("u", "s"):
        assert rel(got[n], ser.datasets[n].numpy()) <= 1e-12, n


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for mode in ("dataflow", "staged", "global"):
        toy_and_fig2(mode)
    dg(1, 1, 3, "colour")
    dg(2, 2, 2, "wave")
    dg(3, 2, 1, "colour")  # per-tile record chunks, grouped inverse-mass/update items
    distributed()
    torch.cuda.synchronize()
    print("sanitize cases ok")
