"""Elastic-wave DG kernel bodies for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

numpy restatement of the native ``dg_*_p{P}`` kernels (see
``paper_1708_03183_b200/dg.py`` for the discretisation).  The reference has
no elastic-wave implementation, so DG arithmetic parity is
"unpinned" by the reference; these bodies are registered in the REAL
reference ``KernelRegistry`` by ``tests/golden/make_golden.py`` so the
reference's own loop machinery (``execute_untiled``/``execute_schedule``,
executor.py:128-245) produces the DG golden values.  The operator tables
are the same float64 arrays the CUDA kernels receive (``dg_tables``).

Bodies follow the reference calling convention (executor.py:142-159): one
numpy view per direct descriptor, a list of views per mapped descriptor.
"""

from __future__ import annotations

import numpy as np

from paper_1708_03183_b200.dg import chain_loops, dg_tables, elastic_setup


def bodies(p: int, dt: float) -> dict:
    tab = dg_tables(p)
    nd, nq = tab.nd, tab.nq
    Sr, Ss, E, LIFT = tab.Sr, tab.Ss, tab.E, tab.LIFT

    def vol(cgeo, mat, u, s, ru, rs):
        rx, ry, sx, sy, det = cgeo
        lam, mu = mat[1], mat[2]
        f = np.concatenate([u, s]).reshape(5, nd)
        dr = f @ Sr.T
        ds = f @ Ss.T
        dx = rx * dr + sx * ds
        dy = ry * dr + sy * ds
        vx, vy, sxx, syy, sxy = range(5)
        ru[:nd] = det * (dx[sxx] + dy[sxy])
        ru[nd:] = det * (dx[sxy] + dy[syy])
        rs[:nd] = det * ((lam + 2 * mu) * dx[vx] + lam * dy[vy])
        rs[nd:2 * nd] = det * (lam * dx[vx] + (lam + 2 * mu) * dy[vy])
        rs[2 * nd:] = det * mu * (dy[vx] + dx[vy])

    def traces(face, u, s):
        f = np.concatenate([u, s]).reshape(5, nd)
        return f @ E[face].T  # (5, nq)

    def stress_corr(dvx, dvy, nx, ny, lam, mu):
        dvn = dvx * nx + dvy * ny
        return (lam * dvn + 2 * mu * dvx * nx, lam * dvn + 2 * mu * dvy * ny,
                mu * (dvx * ny + dvy * nx))

    def add_lift(face, jf, tx, ty, cxx, cyy, cxy, ru, rs, rev=False):
        Lf = LIFT[face]
        if rev:
            tx, ty, cxx, cyy, cxy = (a[::-1] for a in (tx, ty, cxx, cyy, cxy))
        ru[:nd] += jf * (Lf @ tx)
        ru[nd:] += jf * (Lf @ ty)
        rs[:nd] += jf * (Lf @ cxx)
        rs[nd:2 * nd] += jf * (Lf @ cyy)
        rs[2 * nd:] += jf * (Lf @ cxy)

    def iflux(fgeo, mat, u, s, ru, rs):
        nx, ny, jf, fa, fb = fgeo
        fa, fb = int(fa), int(fb)
        ta = traces(fa, u[0], s[0])
        tb = traces(fb, u[1], s[1])[:, ::-1]  # neighbour points in reversed order
        ra, la, ma, zpa, zsa = mat[0]
        rb, lb, mb, zpb, zsb = mat[1]
        tnx, tny = -ny, nx
        vxa, vya, sxxa, syya, sxya = ta
        vxb, vyb, sxxb, syyb, sxyb = tb
        Tax, Tay = sxxa * nx + sxya * ny, sxya * nx + syya * ny
        Tbx, Tby = sxxb * nx + sxyb * ny, sxyb * nx + syyb * ny
        vna, vta = vxa * nx + vya * ny, vxa * tnx + vya * tny
        vnb, vtb = vxb * nx + vyb * ny, vxb * tnx + vyb * tny
        Tna, Tta = Tax * nx + Tay * ny, Tax * tnx + Tay * tny
        Tnb, Ttb = Tbx * nx + Tby * ny, Tbx * tnx + Tby * tny
        dvn = (Tnb - Tna + zpb * (vnb - vna)) / (zpa + zpb)
        dvt = (Ttb - Tta + zsb * (vtb - vta)) / (zsa + zsb)
        dTax = zpa * dvn * nx + zsa * dvt * tnx
        dTay = zpa * dvn * ny + zsa * dvt * tny
        dvax = dvn * nx + dvt * tnx
        dvay = dvn * ny + dvt * tny
        cxx, cyy, cxy = stress_corr(dvax, dvay, nx, ny, la, ma)
        add_lift(fa, jf, dTax, dTay, cxx, cyy, cxy, ru[0], rs[0])
        dTbx = (Tbx - Tax) - dTax
        dTby = (Tby - Tay) - dTay
        dvbx = vxa + dvax - vxb
        dvby = vya + dvay - vyb
        cxx, cyy, cxy = stress_corr(dvbx, dvby, -nx, -ny, lb, mb)
        add_lift(fb, jf, dTbx, dTby, cxx, cyy, cxy, ru[1], rs[1], rev=True)

    def eflux(fgeo, mat, u, s, ru, rs):
        nx, ny, jf, fa, _ = fgeo
        fa = int(fa)
        vx, vy, sxx, syy, sxy = traces(fa, u[0], s[0])
        rho, lam, mu, zp, zs = mat[0]
        tnx, tny = -ny, nx
        Tx, Ty = sxx * nx + sxy * ny, sxy * nx + syy * ny
        dvn = -(Tx * nx + Ty * ny) / zp
        dvt = -(Tx * tnx + Ty * tny) / zs
        dvx = dvn * nx + dvt * tnx
        dvy = dvn * ny + dvt * tny
        cxx, cyy, cxy = stress_corr(dvx, dvy, nx, ny, lam, mu)
        add_lift(fa, jf, -Tx, -Ty, cxx, cyy, cxy, ru[0], rs[0])

    def minv(cgeo, mat, ru, rs):
        det = cgeo[4]
        ru *= 1.0 / (mat[0] * det)
        rs *= 1.0 / det

    def axpy(u, s, ru, rs):
        u += dt * ru
        s += dt * rs

    return {f"dg_vol_p{p}": vol, f"dg_iflux_p{p}": iflux, f"dg_eflux_p{p}": eflux,
            f"dg_minv_p{p}": minv, f"dg_axpy_p{p}": axpy}


class RefProblem:
    """A DG chain declared with the REFERENCE's classes (module ``L``)."""

    def __init__(self, chain, datasets, bindings, registry, setup):
        self.chain, self.datasets, self.bindings = chain, datasets, bindings
        self.registry, self.setup = registry, setup


def build_problem_reference(L, dims, p: int, steps: int = 1, seed: int = 1,
                            material="homogeneous", sigma: float | None = None) -> RefProblem:
    """Declare the elastic chain on the reference API with numpy bodies.

    ``sigma`` defaults to max(dims)/8 (small fixtures); BASELINE config 2 uses 8."""
    st = elastic_setup(dims[0], dims[1], p, steps, material=material, noise_seed=seed,
                       sigma=max(dims) / 8.0 if sigma is None else sigma)
    sp = {n: L.IterationSpace(n, s.core_size, s.boundary_size, s.nonexec_size)
          for n, s in st.spaces.items()}
    mp = {n: L.MeshMap(n, sp[m.source.name], sp[m.target.name], m.arity, m.values)
          for n, m in st.maps.items()}
    modes = {"R": L.AccessMode.READ, "W": L.AccessMode.WRITE, "I": L.AccessMode.INC,
             "RW": L.AccessMode.WRITE}
    loops, bindings = chain_loops(p, steps, sp, mp, loop_cls=L.Loop, desc_cls=L.Descriptor,
                                  binding_cls=L.KernelBinding, modes=modes)
    chain = L.build_chain(tuple(sp.values()), tuple(mp.values()), loops, len(loops))
    reg = L.KernelRegistry()
    for name, fn in bodies(p, st.dt).items():
        nargs = 6 if ("vol" in name or "flux" in name) else 4
        reg.register(name, fn, nargs)
    ds = {n: L.Dataset(n, sp[st.space_of[n]], st.vpe[n], v.copy()) for n, v in st.data.items()}
    return RefProblem(chain, ds, bindings, reg, st)
