"""Time the REAL reference CPU executor on a bounded sample -- TEST/BENCH INFRASTRUCTURE.

The reference (``looptile``, pure Python/numpy) is its own CPU path, so the
CPU baseline is that package's ``inspect_chain`` + ``execute_schedule``
(src/inspector.py:433-495, src/executor.py:185-245) with the oracle's numpy
elastic-wave bodies registered in its ``KernelRegistry`` (the reference has
no elastic-wave solver; oracle/dg_oracle.py).  ``__graft_entry__.build()``
copies the unmodified package from /root/reference/pkg/src/looptile into
``oracle/_ref/looptile`` (git-ignored, not gpurun-ignored) so it travels to
the GPU box, like a compiled reference would; nothing here is on the product
path.  Only ``bench.py``'s ``cpu_baseline`` leg and ``--impl reference`` arm
import this module.
"""

from __future__ import annotations

import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
_CANDIDATES = (os.path.join(HERE, "_ref"), "/root/reference/pkg/src")


def load_reference():
    """Import the reference ``looptile`` package (oracle/_ref first); None if absent."""
    for path in _CANDIDATES:
        if os.path.isdir(os.path.join(path, "looptile")):
            if path not in sys.path:
                sys.path.insert(0, path)
            sys.dont_write_bytecode = True
            import looptile
            return looptile
    return None


def sample_rate(p: int, T: int, n: int, material, ts: int, noise_seed=1, sigma=None,
                untiled: bool = False):
    """One chain (T timesteps) of the elastic DG chain on an n x n mesh through
    the reference executor.  Returns (DoF-updates/s, seconds, description)."""
    L = load_reference()
    if L is None:
        return None
    from oracle import dg_oracle
    prob = dg_oracle.build_problem_reference(L, (n, n), p, steps=T, seed=noise_seed,
                                             material=material,
                                             sigma=8.0 * n / 256 if sigma is None else sigma)
    dofs = prob.setup.dofs
    if untiled:
        t0 = time.perf_counter()
        L.execute_untiled(prob.chain, prob.bindings, prob.datasets, prob.registry)
        dt = time.perf_counter() - t0
        what = "execute_untiled"
    else:
        sched = L.inspect_chain(prob.chain, ts, L.ExecMode.SHARED)
        t0 = time.perf_counter()
        L.execute_schedule(sched, prob.chain, prob.bindings, prob.datasets, prob.registry)
        dt = time.perf_counter() - t0
        what = f"inspect_chain(ts={ts}, SHARED) + execute_schedule (timed)"
    desc = (f"reference looptile {what}, DG P{p} {n}x{n} ({prob.setup.n_cells} cells), "
            f"one {T}-timestep chain, numpy bodies, 1 core (GIL-bound)")
    return dofs * T / dt, dt, desc
