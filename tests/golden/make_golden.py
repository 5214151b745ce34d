"""Generate golden fixtures from the REAL reference implementation.

Run in the build container (the reference is not present on GPU boxes):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports ``looptile`` read-only from /root/reference/pkg/src and writes small
fixtures next to this script:

* ``schedules.json.gz`` -- ``Schedule.serialize()`` text of the reference
  inspector for FIG2 / EIGHT_LOOP / toy (BASELINE config 1) / DG-shaped chains
  over meshes x tile sizes x modes x renumberings, plus chain fingerprints.
* ``values.npz``        -- dataset values after ``execute_untiled`` and
  ``execute_schedule`` (FIG2, EIGHT_LOOP, toy, DG-shaped), and the shipped
  ``pkg/out/fig2_report.txt.{tiled,untiled}`` dumps, checked here to reproduce.
* ``invert.npz``        -- ``invert_map`` of 100 random maps (seed 2024, the
  reference's own property test, tests/test_acceptance.py:174-186).
* ``rcm.npz``           -- reference RCM vertex orders.
* ``distributed.npz``   -- ``partition_for_ranks`` regions/global ids/exchange
  tables and ``run_distributed`` gathered values (FIG2, 2 and 4 ranks).

The toy chain needs a ``c2e`` map the reference lacks;
it is built here independently of the product code (dict lookup of sorted
vertex pairs, side order (v0,v1),(v1,v2),(v0,v2)).  RW is declared WRITE on
the reference side (inspection ignores modes).
"""

from __future__ import annotations

import base64
import gzip
import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True

import looptile as L  # noqa: E402
from looptile.chain import AccessMode, Descriptor, Loop, MeshMap, build_chain  # noqa: E402
from looptile.executor import Dataset, KernelBinding  # noqa: E402
from looptile.inspector import ExecMode  # noqa: E402
from legality import check_legality, footprint_conflicts  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import dg_oracle  # noqa: E402  (numpy DG bodies + setup, test infra)

MODES = {"sequential": ExecMode.SEQUENTIAL, "shared": ExecMode.SHARED}


def c2e_rows(mesh) -> np.ndarray:
    pairs = mesh.edges_to_vertices.reshape(-1, 2).tolist()
    index = {tuple(sorted(p)): i for i, p in enumerate(pairs)}
    rows = []
    for a, b, c in mesh.cells_to_vertices.reshape(-1, 3).tolist():
        for s in ((a, b), (b, c), (a, c)):
            rows.append(index[tuple(sorted(s))])
    return np.array(rows, dtype=np.int64)


def toy_registry():
    reg = L.KernelRegistry()

    def k1(a, v):
        for x in v:
            x += a / 3.0

    def k2(e, v):
        e[:] = 0.5 * (v[0] + v[1])

    def k3(a, e):
        a += (e[0] + e[1] + e[2]) / 3.0

    reg.register("toy_k1", k1, 2)
    reg.register("toy_k2", k2, 2)
    reg.register("toy_k3", k3, 2)
    return reg


def toy_setup(mesh):
    sp = L.mesh_spaces(mesh) if hasattr(L, "mesh_spaces") else None
    from looptile.mesh import mesh_maps, mesh_spaces
    sp = mesh_spaces(mesh)
    mp = mesh_maps(mesh, sp)
    mp["c2e"] = MeshMap("c2e", sp["cells"], sp["edges"], 3, c2e_rows(mesh))
    R, W, I = AccessMode.READ, AccessMode.WRITE, AccessMode.INC
    loops, binds = [], []
    for it in range(2):
        for space, kern, descs, args in (
                ("cells", "toy_k1", ((None, R), ("c2v", I)), ("a", "v")),
                ("edges", "toy_k2", ((None, W), ("e2v", R)), ("e", "v")),
                ("cells", "toy_k3", ((None, W), ("c2e", R)), ("a", "e"))):
            loops.append(Loop(len(loops), sp[space],
                              tuple(Descriptor(None if m is None else mp[m], md)
                                    for m, md in descs), kern))
            binds.append(KernelBinding(kern, args))
    chain = build_chain(tuple(sp.values()), tuple(mp.values()), loops, depth=6)
    ds = {"a": Dataset("a", sp["cells"], 1, np.random.default_rng(0).random(mesh.num_cells)),
          "v": Dataset("v", sp["verts"], 1, np.zeros(mesh.num_vertices)),
          "e": Dataset("e", sp["edges"], 1, np.zeros(mesh.num_edges))}
    return chain, ds, tuple(binds)


def main():
    schedules, fingerprints, meta = {}, {}, {}
    values = {}
    reg = L.default_registry()

    def record(name, chain, ts, mode, check=True):
        s = L.inspect_chain(chain, ts, MODES[mode])
        if check:
            assert check_legality(chain, s) == [], name
            assert footprint_conflicts(chain, s) == [], name
        text = s.serialize()
        schedules[name] = base64.b64encode(gzip.compress(text, 9)).decode()
        meta[name] = {"sha256": hashlib.sha256(text).hexdigest(), "rounds": s.recolor_rounds,
                      "tiles": len(s.tiles), "colors": len(s.color_order)}
        return s

    # FIG2: the acceptance sweep (tests/test_acceptance.py:44-63) + unrenumbered meshes
    for dims in [(1, 1), (2, 1), (4, 2), (8, 4), (16, 8)]:
        for ren in ("rcm", "none"):
            mesh = L.generate_rect_mesh(*dims)
            if ren == "rcm":
                mesh = L.rcm_renumber(mesh)
            chain, ds, b = L.global_setup(mesh, L.PRESETS["fig2"], 3)
            fingerprints[f"fig2_{dims[0]}x{dims[1]}_{ren}"] = chain.fingerprint
            L.execute_untiled(chain, b, ds, reg)
            for n, d in ds.items():
                values[f"fig2_{dims[0]}x{dims[1]}_{ren}/untiled/{n}"] = d.values.copy()
            for ts in (1, 4, 16, 64) if ren == "rcm" else (2, 3, 8):
                for mode in MODES:
                    record(f"fig2_{dims[0]}x{dims[1]}_{ren}_ts{ts}_{mode}", chain, ts, mode,
                           check=dims[0] * dims[1] <= 32)
    # conflict back-tracking regression (tests/test_acceptance.py:83-92)
    mesh = L.rcm_renumber(L.generate_rect_mesh(4, 1))
    chain, _, _ = L.global_setup(mesh, L.PRESETS["fig2"], 3)
    s = record("fig2_4x1_rcm_ts2_shared", chain, 2, "shared")
    assert s.recolor_rounds >= 2

    # EIGHT_LOOP
    for dims in [(8, 4), (16, 8)]:
        mesh = L.rcm_renumber(L.generate_rect_mesh(*dims))
        chain, ds, b = L.global_setup(mesh, L.PRESETS["eight_loop"], 8)
        fingerprints[f"eight_{dims[0]}x{dims[1]}_rcm"] = chain.fingerprint
        L.execute_untiled(chain, b, ds, reg)
        for n, d in ds.items():
            values[f"eight_{dims[0]}x{dims[1]}_rcm/untiled/{n}"] = d.values.copy()
        for ts in (3, 8, 16):
            for mode in MODES:
                record(f"eight_{dims[0]}x{dims[1]}_rcm_ts{ts}_{mode}", chain, ts, mode,
                       check=False)

    # shipped value dumps (pkg/out/fig2_report.txt.*): FIG2 16x8 rcm shared ts16
    mesh = L.rcm_renumber(L.generate_rect_mesh(16, 8))
    chain, ds, b = L.global_setup(mesh, L.PRESETS["fig2"], 3)
    s = L.inspect_chain(chain, 16, ExecMode.SHARED)
    L.execute_schedule(s, chain, b, ds, reg)
    for suffix in ("tiled", "untiled"):
        dumped = {}
        with open(os.path.join(REF, "out", f"fig2_report.txt.{suffix}")) as fh:
            for line in fh:
                name, i, v = line.split()
                dumped.setdefault(name, []).append(float(v))
        for n in dumped:
            assert np.array_equal(np.array(dumped[n]), ds[n].values), (suffix, n)
    meta["shipped_fig2_report_reproduces"] = True

    # toy chain, BASELINE config 1 (32x32) + a small variant
    treg = toy_registry()
    for dims, ts_list in (((32, 32), (64,)), ((8, 8), (8, 16))):
        for ren in ("none", "rcm"):
            mesh = L.generate_rect_mesh(*dims)
            if ren == "rcm":
                mesh = L.rcm_renumber(mesh)
            tag = f"toy_{dims[0]}x{dims[1]}_{ren}"
            chain, ds, b = toy_setup(mesh)
            fingerprints[tag] = chain.fingerprint
            base = {n: d.copy() for n, d in ds.items()}
            L.execute_untiled(chain, b, ds, treg)
            for n, d in ds.items():
                values[f"{tag}/untiled/{n}"] = d.values.copy()
            for ts in ts_list:
                for mode in MODES:
                    sname = f"{tag}_ts{ts}_{mode}"
                    s = record(sname, chain, ts, mode, check=dims[0] <= 8)
                    run = {n: d.copy() for n, d in base.items()}
                    L.execute_schedule(s, chain, b, run, treg)
                    for n, d in run.items():
                        values[f"{sname}/tiled/{n}"] = d.values.copy()

    # DG-shaped elastic-wave chain: the builder's numpy bodies in the reference executor
    for p in (1, 2, 3):
        for dims, ts, steps in (((4, 4), 8, 1), ((8, 6), 16, 1), ((6, 6), 12, 2)):
            if p == 3 and dims != (4, 4):
                continue
            prob = dg_oracle.build_problem_reference(L, dims, p, steps=steps, seed=1)
            tag = f"dg{p}s{steps}_{dims[0]}x{dims[1]}_none"
            fingerprints[tag] = prob.chain.fingerprint
            run = {n: d.copy() for n, d in prob.datasets.items()}
            L.execute_untiled(prob.chain, prob.bindings, run, prob.registry)
            for n in ("u", "s", "ru", "rs"):
                values[f"{tag}/untiled/{n}"] = run[n].values.copy()
            for mode in MODES:
                s = record(f"{tag}_ts{ts}_{mode}", prob.chain, ts, mode, check=False)
                run = {n: d.copy() for n, d in prob.datasets.items()}
                L.execute_schedule(s, prob.chain, prob.bindings, run, prob.registry)
                for n in ("u", "s", "ru", "rs"):
                    values[f"{tag}_ts{ts}_{mode}/tiled/{n}"] = run[n].values.copy()

    # invert_map round trips (seed 2024, 100 random maps)
    rng = np.random.default_rng(2024)
    inv = {}
    for i in range(100):
        n_src, n_tgt, arity = int(rng.integers(1, 40)), int(rng.integers(1, 30)), \
            int(rng.integers(1, 5))
        vals = rng.integers(0, n_tgt, size=n_src * arity)
        src = L.IterationSpace("s", n_src)
        tgt = L.IterationSpace("t", n_tgt)
        im = L.invert_map(MeshMap("m", src, tgt, arity, vals))
        inv[f"{i}/shape"] = np.array([n_src, n_tgt, arity])
        inv[f"{i}/values"] = vals
        inv[f"{i}/inv_offsets"] = im.offsets
        inv[f"{i}/inv_values"] = im.values

    # RCM orders
    from looptile.mesh import rcm_ordering, vertex_adjacency
    rcm = {}
    for dims in [(1, 1), (3, 2), (8, 4), (16, 8), (32, 32), (7, 13)]:
        mesh = L.generate_rect_mesh(*dims)
        rcm[f"{dims[0]}x{dims[1]}"] = rcm_ordering(vertex_adjacency(mesh))

    # distributed: partition tables + gathered values
    dist = {}
    for tag, dims, ren, nranks, depth in (("fig2_8x4_rcm", (8, 4), "rcm", 2, 3),
                                          ("fig2_8x4_rcm", (8, 4), "rcm", 4, 3),
                                          ("p_16x8_none", (16, 8), "none", 3, 2),
                                          ("p_12x10_rcm", (12, 10), "rcm", 4, 5),
                                          ("p_16x8_rcm", (16, 8), "rcm", 8, 2),
                                          ("p_9x7_none", (9, 7), "none", 5, 1)):
        mesh = L.generate_rect_mesh(*dims)
        if ren == "rcm":
            mesh = L.rcm_renumber(mesh)
        lms = L.partition_for_ranks(mesh, nranks, depth)
        pre = f"{tag}/n{nranks}"
        dist[f"{pre}/depth"] = np.array([depth])
        for lm in lms:
            for space, sz in lm.sizes.items():
                key = f"{pre}/r{lm.rank}/{space}"
                dist[key + "/sizes"] = np.array([sz.core, sz.owned, sz.exec, sz.nonexec])
                dist[key + "/gids"] = lm.global_ids[space]
            dist[f"{pre}/r{lm.rank}/c2v"] = lm.cells_to_vertices
            dist[f"{pre}/r{lm.rank}/e2v"] = lm.edges_to_vertices
            for (space, nbr), table in lm.exchange_table.items():
                dist[f"{pre}/r{lm.rank}/x/{space}/{nbr}"] = table
        if tag.startswith("fig2"):
            res = L.run_distributed(mesh, L.PRESETS["fig2"], nranks, 4, depth=depth,
                                    registry=reg, poison_halo=True)
            for n, v in res.datasets.items():
                dist[f"{pre}/gathered/{n}"] = v

    with gzip.open(os.path.join(HERE, "schedules.json.gz"), "wt") as fh:
        json.dump({"schedules": schedules, "meta": meta, "fingerprints": fingerprints}, fh)
    np.savez_compressed(os.path.join(HERE, "values.npz"), **values)
    np.savez_compressed(os.path.join(HERE, "invert.npz"), **inv)
    np.savez_compressed(os.path.join(HERE, "rcm.npz"), **rcm)
    np.savez_compressed(os.path.join(HERE, "distributed.npz"), **dist)
    print(f"{len(schedules)} schedules, {len(values)} value arrays, "
          f"{len(fingerprints)} fingerprints")


if __name__ == "__main__":
    main()
