"""Full-size golden for BASELINE config 2, produced by the REAL reference.

Run in the build container (the reference is not present on GPU boxes):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_full.py

BASELINE configs[1]: elastic DG P1 on the 256x256 right-diagonal mesh of
[0,256]^2 (131,072 cells), rho=1, lambda=2, mu=1, Gaussian pulse sigma 8 at
the centre + U[-1e-3,1e-3] noise (seed 1), dt = 0.1/(sqrt(4)*3), one timestep
per chain, 10 timesteps.  The chain is declared on the reference API
(``looptile``, imported read-only from /root/reference/pkg/src) with the
oracle's numpy DG bodies registered in the reference ``KernelRegistry``
(oracle/dg_oracle.py); the reference's own ``execute_untiled``
(src/executor.py:163-169) is called 10 times -- "untiled sequential
execution", the semantic oracle BASELINE names.

The reference inspector is also run on that chain at the bench's seed tile
(ts=32, SHARED; src/inspector.py:433-495) and the SHA-256 of its
``serialize()`` text is recorded, so the GPU inspector is checked byte-exact
at the benchmarked size.

Written to ``config2_full.npz`` (kept small for git):
* ``u_rows``/``s_rows``/``ru_rows``/``rs_rows``: the final values of every
  16th cell (8,192 of 131,072 cells), ``rows`` their cell ids;
* ``norms``: per-field max-abs and 2-norm of the FULL arrays (u, s, ru, rs);
* ``init_sha``: SHA-256 of the initial u||s bytes (pins the setup);
* ``sched_sha``/``sched_meta``: reference schedule hash, tiles, colours, rounds.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True

import looptile as L  # noqa: E402
from looptile.inspector import ExecMode  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import dg_oracle  # noqa: E402

DIMS, P, STEPS, TS, STRIDE = (256, 256), 1, 10, 32, 16


def main():
    t0 = time.time()
    prob = dg_oracle.build_problem_reference(L, DIMS, P, steps=1, seed=1, sigma=8.0)
    ds = prob.datasets
    init_sha = hashlib.sha256(ds["u"].values.tobytes() + ds["s"].values.tobytes()).hexdigest()
    assert abs(prob.setup.dt - 0.1 / (np.sqrt(4.0) * 3)) < 1e-15
    print(f"setup {time.time() - t0:.1f}s, dt {prob.setup.dt!r}", flush=True)
    t0 = time.time()
    sched = L.inspect_chain(prob.chain, TS, ExecMode.SHARED)
    text = sched.serialize()
    sched_sha = hashlib.sha256(text).hexdigest()
    meta = np.array([len(sched.tiles), len(sched.color_order), sched.recolor_rounds])
    print(f"reference inspect {time.time() - t0:.1f}s: tiles/colours/rounds {meta}", flush=True)
    for step in range(STEPS):
        t0 = time.time()
        L.execute_untiled(prob.chain, prob.bindings, ds, prob.registry)
        print(f"step {step}: {time.time() - t0:.1f}s", flush=True)
    rows = np.arange(0, prob.setup.n_cells, STRIDE)
    out = {"rows": rows, "init_sha": np.array(init_sha), "sched_sha": np.array(sched_sha),
           "sched_meta": meta, "dims": np.array(DIMS), "p": np.array(P),
           "steps": np.array(STEPS), "ts": np.array(TS)}
    norms = []
    for n in ("u", "s", "ru", "rs"):
        v = ds[n].values.reshape(prob.setup.n_cells, -1)
        out[f"{n}_rows"] = v[rows].copy()
        norms.append([np.abs(v).max(), np.linalg.norm(v)])
    out["norms"] = np.array(norms)
    np.savez_compressed(os.path.join(HERE, "config2_full.npz"), **out)
    print("written", out["norms"])


if __name__ == "__main__":
    main()
