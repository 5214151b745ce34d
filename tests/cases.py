"""Chain builders shared by the oracle and GPU parity tests (host-side only)."""

import paper_1708_03183_b200 as lt

DEPTH = {"fig2": 3, "eight": 8, "toy": 6}
PROBLEM = {"fig2": lt.FIG2, "eight": lt.EIGHT_LOOP, "toy": lt.TOY}


def build_case(prob: str, dims, ren: str):
    if prob.startswith("dg"):
        st, chain = dg_setup(f"{prob}_{dims[0]}x{dims[1]}_{ren}")
        return st.mesh, (chain, {n: v.copy() for n, v in st.data.items()}, dict(st.vpe),
                         st.bindings)
    mesh = lt.generate_rect_mesh(*dims)
    if ren == "rcm":
        mesh = lt.rcm_renumber(mesh)
    return mesh, setup(mesh, prob)


def setup(mesh, prob: str):
    import numpy as np
    p = PROBLEM[prob]
    spaces = lt.mesh_spaces(mesh)
    from paper_1708_03183_b200.problems import problem_maps
    maps = problem_maps(mesh, spaces, p, lt.mesh_maps(mesh, spaces))
    gids = {n: np.arange(s.total) for n, s in spaces.items()}
    totals = {n: s.total for n, s in spaces.items()}
    return host_instantiate(p, spaces, maps, gids, DEPTH[prob], totals)


def host_instantiate(problem, spaces, maps, gids, depth, totals):
    """(chain, {name: numpy values}, {name: vpe}, bindings) without touching a GPU."""
    from paper_1708_03183_b200.chain import Descriptor, Loop, build_chain
    from paper_1708_03183_b200.executor import KernelBinding
    from paper_1708_03183_b200.problems import init_values
    loops = []
    for i, spec in enumerate(problem.loops):
        loops.append(Loop(i, spaces[spec.space],
                          tuple(Descriptor(None if a.map is None else maps[a.map], a.mode)
                                for a in spec.accesses), spec.kernel))
    chain = build_chain(tuple(spaces.values()), tuple(maps.values()), loops, depth)
    data = {d.name: init_values(d, gids[d.space], totals[d.space]) for d in problem.datasets}
    vpe = {d.name: d.values_per_element for d in problem.datasets}
    bindings = tuple(KernelBinding(s.kernel, tuple(a.dataset for a in s.accesses))
                     for s in problem.loops)
    return chain, data, vpe, bindings


def dg_setup(tag: str):
    """'dg2s1_8x6_none' -> host ElasticSetup + chain, identical to make_golden's instance."""
    from paper_1708_03183_b200.dg import elastic_setup
    from paper_1708_03183_b200.chain import build_chain
    head, d, ren = tag.split("_")[:3]
    p, steps = int(head[2]), int(head[4:])
    dims = tuple(int(v) for v in d.split("x"))
    st = elastic_setup(dims[0], dims[1], p, steps, noise_seed=1, sigma=max(dims) / 8.0,
                       renumbering=None if ren == "none" else ren)
    chain = build_chain(tuple(st.spaces.values()), tuple(st.maps.values()), st.loops,
                        len(st.loops))
    st.chain = chain
    return st, chain
