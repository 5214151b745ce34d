// lt_dg.cuh — elastic-wave DG kernel bodies (velocity-stress, modal P1..P4).
//
// Discretisation: paper_1708_03183_b200/dg.py (module docstring); numpy twin:
// oracle/dg_oracle.py.  One thread per element (cell or facet); operator
// tables (S_r, S_s, face traces E, lifts) come from the kernel's parameter
// block (read-only, warp-uniform loads -> L1 broadcast).  Facet kernels write
// their per-side increments into the executor's contribution slots; the
// executor applies them in reference order.
#pragma once

#include "lt_kernels.cuh"

namespace lt {

template <int P>
struct DGShape {
  static constexpr int ND = (P + 1) * (P + 2) / 2;
  static constexpr int NQ = P + 1;
};

// L0: R = |J| (div sigma ; C:grad v)   [cgeo R, mat R, u R, s R, ru W, rs W]
template <int P, class C>
__device__ __forceinline__ void dg_vol(C &c) {
  constexpr int ND = DGShape<P>::ND;
  const double *g = c.rd(0), *m = c.rd(1), *u = c.rd(2), *s = c.rd(3);
  double *ru = c.wr(4), *rs = c.wr(5);
  const double *__restrict__ Sr = c.params();
  const double *__restrict__ Ss = Sr + ND * ND;
  double f[5][ND];
#pragma unroll
  for (int j = 0; j < ND; ++j) {
    f[0][j] = u[j];
    f[1][j] = u[ND + j];
    f[2][j] = s[j];
    f[3][j] = s[ND + j];
    f[4][j] = s[2 * ND + j];
  }
  const double rx = g[0], ry = g[1], sx = g[2], sy = g[3], det = g[4];
  const double lam = m[1], mu = m[2], l2m = lam + 2.0 * mu;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    double dr[5], ds[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) { dr[q] = 0.0; ds[q] = 0.0; }
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      const double a = __ldg(Sr + i * ND + j), b = __ldg(Ss + i * ND + j);
#pragma unroll
      for (int q = 0; q < 5; ++q) { dr[q] += a * f[q][j]; ds[q] += b * f[q][j]; }
    }
    double dx[5], dy[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) { dx[q] = rx * dr[q] + sx * ds[q]; dy[q] = ry * dr[q] + sy * ds[q]; }
    ru[i] = det * (dx[2] + dy[4]);
    ru[ND + i] = det * (dx[4] + dy[3]);
    rs[i] = det * (l2m * dx[0] + lam * dy[1]);
    rs[ND + i] = det * (lam * dx[0] + l2m * dy[1]);
    rs[2 * ND + i] = det * mu * (dy[0] + dx[1]);
  }
}

template <int ND, int NQ>
__device__ __forceinline__ void dg_traces(const double *__restrict__ E, int face, const double *u,
                                          const double *s, double t[5][NQ], bool reversed) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int qq = reversed ? NQ - 1 - q : q;
    const double *e = E + (face * NQ + qq) * ND;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      const double w = __ldg(e + j);
      a0 += w * u[j];
      a1 += w * u[ND + j];
      a2 += w * s[j];
      a3 += w * s[ND + j];
      a4 += w * s[2 * ND + j];
    }
    t[0][q] = a0; t[1][q] = a1; t[2][q] = a2; t[3][q] = a3; t[4][q] = a4;
  }
}

// increments: out_u = jf * LIFT_face * (tx, ty); out_s = jf * LIFT_face * (cxx, cyy, cxy)
template <int ND, int NQ>
__device__ __forceinline__ void dg_lift(const double *__restrict__ LIFT, int face, double jf,
                                        const double corr[5][NQ], bool reversed, double *out_u,
                                        double *out_s) {
  const double *Lf = LIFT + face * ND * NQ;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double w = __ldg(Lf + i * NQ + q);
      const int qq = reversed ? NQ - 1 - q : q;
      a0 += w * corr[0][qq];
      a1 += w * corr[1][qq];
      a2 += w * corr[2][qq];
      a3 += w * corr[3][qq];
      a4 += w * corr[4][qq];
    }
    out_u[i] = jf * a0;
    out_u[ND + i] = jf * a1;
    out_s[i] = jf * a2;
    out_s[ND + i] = jf * a3;
    out_s[2 * ND + i] = jf * a4;
  }
}

// L1: interior facets, upwind flux   [fgeo R, mat R@2, u R@2, s R@2, ru I@2, rs I@2]
template <int P, class C>
__device__ __forceinline__ void dg_iflux(C &c) {
  constexpr int ND = DGShape<P>::ND, NQ = DGShape<P>::NQ;
  const double *g = c.rd(0);
  const double nx = g[0], ny = g[1], jf = g[2];
  const int fa = (int)g[3], fb = (int)g[4];
  const double *ma = c.rdm(1, 0), *mb = c.rdm(1, 1);
  const double *__restrict__ E = c.params();
  const double *__restrict__ LIFT = E + 3 * NQ * ND;
  double ta[5][NQ], tb[5][NQ];
  dg_traces<ND, NQ>(E, fa, c.rdm(2, 0), c.rdm(3, 0), ta, false);
  dg_traces<ND, NQ>(E, fb, c.rdm(2, 1), c.rdm(3, 1), tb, true);
  const double la = ma[1], mua = ma[2], lb = mb[1], mub = mb[2];
  const double zpa = ma[3], zsa = ma[4], zpb = mb[3], zsb = mb[4];  // impedances rho*c_p, rho*c_s
  const double ip = 1.0 / (zpa + zpb), is = 1.0 / (zsa + zsb);
  const double tnx = -ny, tny = nx;
  double ca[5][NQ], cb[5][NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double Tax = ta[2][q] * nx + ta[4][q] * ny, Tay = ta[4][q] * nx + ta[3][q] * ny;
    const double Tbx = tb[2][q] * nx + tb[4][q] * ny, Tby = tb[4][q] * nx + tb[3][q] * ny;
    const double vna = ta[0][q] * nx + ta[1][q] * ny, vta = ta[0][q] * tnx + ta[1][q] * tny;
    const double vnb = tb[0][q] * nx + tb[1][q] * ny, vtb = tb[0][q] * tnx + tb[1][q] * tny;
    const double Tna = Tax * nx + Tay * ny, Tta = Tax * tnx + Tay * tny;
    const double Tnb = Tbx * nx + Tby * ny, Ttb = Tbx * tnx + Tby * tny;
    const double dvn = (Tnb - Tna + zpb * (vnb - vna)) * ip;
    const double dvt = (Ttb - Tta + zsb * (vtb - vta)) * is;
    const double dTax = zpa * dvn * nx + zsa * dvt * tnx;
    const double dTay = zpa * dvn * ny + zsa * dvt * tny;
    const double dvax = dvn * nx + dvt * tnx, dvay = dvn * ny + dvt * tny;
    const double dna = dvax * nx + dvay * ny;
    ca[0][q] = dTax;
    ca[1][q] = dTay;
    ca[2][q] = la * dna + 2.0 * mua * dvax * nx;
    ca[3][q] = la * dna + 2.0 * mua * dvay * ny;
    ca[4][q] = mua * (dvax * ny + dvay * nx);
    const double dvbx = ta[0][q] + dvax - tb[0][q], dvby = ta[1][q] + dvay - tb[1][q];
    const double dnb = -(dvbx * nx + dvby * ny);
    cb[0][q] = (Tbx - Tax) - dTax;
    cb[1][q] = (Tby - Tay) - dTay;
    cb[2][q] = lb * dnb - 2.0 * mub * dvbx * nx;
    cb[3][q] = lb * dnb - 2.0 * mub * dvby * ny;
    cb[4][q] = -mub * (dvbx * ny + dvby * nx);
  }
  dg_lift<ND, NQ>(LIFT, fa, jf, ca, false, c.inc(4, 0), c.inc(5, 0));
  dg_lift<ND, NQ>(LIFT, fb, jf, cb, true, c.inc(4, 1), c.inc(5, 1));
}

// L2: exterior facets, traction-free mirror state
template <int P, class C>
__device__ __forceinline__ void dg_eflux(C &c) {
  constexpr int ND = DGShape<P>::ND, NQ = DGShape<P>::NQ;
  const double *g = c.rd(0);
  const double nx = g[0], ny = g[1], jf = g[2];
  const int fa = (int)g[3];
  const double *m = c.rdm(1, 0);
  const double *__restrict__ E = c.params();
  const double *__restrict__ LIFT = E + 3 * NQ * ND;
  double t[5][NQ];
  dg_traces<ND, NQ>(E, fa, c.rdm(2, 0), c.rdm(3, 0), t, false);
  const double lam = m[1], mu = m[2];
  const double izp = 1.0 / m[3], izs = 1.0 / m[4];
  const double tnx = -ny, tny = nx;
  double cr[5][NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double Tx = t[2][q] * nx + t[4][q] * ny, Ty = t[4][q] * nx + t[3][q] * ny;
    const double dvn = -(Tx * nx + Ty * ny) * izp;
    const double dvt = -(Tx * tnx + Ty * tny) * izs;
    const double dvx = dvn * nx + dvt * tnx, dvy = dvn * ny + dvt * tny;
    const double dn = dvx * nx + dvy * ny;
    cr[0][q] = -Tx;
    cr[1][q] = -Ty;
    cr[2][q] = lam * dn + 2.0 * mu * dvx * nx;
    cr[3][q] = lam * dn + 2.0 * mu * dvy * ny;
    cr[4][q] = mu * (dvx * ny + dvy * nx);
  }
  dg_lift<ND, NQ>(LIFT, fa, jf, cr, false, c.inc(4, 0), c.inc(5, 0));
}

// L3: inverse mass (M_ref = I): ru /= rho |J|, rs /= |J|   [cgeo R, mat R, ru RW, rs RW]
template <int P, class C>
__device__ __forceinline__ void dg_minv(C &c) {
  constexpr int ND = DGShape<P>::ND;
  const double det = c.rd(0)[4], rho = c.rd(1)[0];
  double *ru = c.wr(2), *rs = c.wr(3);
  const double iu = 1.0 / (rho * det), is = 1.0 / det;
#pragma unroll
  for (int i = 0; i < 2 * ND; ++i) ru[i] *= iu;
#pragma unroll
  for (int i = 0; i < 3 * ND; ++i) rs[i] *= is;
}

// L4: forward Euler   [u RW, s RW, ru R, rs R]  params: dt
template <int P, class C>
__device__ __forceinline__ void dg_axpy(C &c) {
  constexpr int ND = DGShape<P>::ND;
  const double dt = c.params()[0];
  double *u = c.wr(0), *s = c.wr(1);
  const double *ru = c.rd(2), *rs = c.rd(3);
#pragma unroll
  for (int i = 0; i < 2 * ND; ++i) u[i] += dt * ru[i];
#pragma unroll
  for (int i = 0; i < 3 * ND; ++i) s[i] += dt * rs[i];
}

template <int P, class C>
__device__ __forceinline__ void dg_dispatch_p(int which, C &c) {
  switch (which) {
    case 0: dg_vol<P>(c); break;
    case 1: dg_iflux<P>(c); break;
    case 2: dg_eflux<P>(c); break;
    case 3: dg_minv<P>(c); break;
    case 4: dg_axpy<P>(c); break;
  }
}

// family: 0 none, 1..4 only degree P, 5 all degrees
template <int FAM, class C>
__device__ __forceinline__ void dg_dispatch(int k, C &c) {
  const int p = k / 5 + 1, which = k % 5;
  if (FAM == 1 || (FAM == 5 && p == 1)) dg_dispatch_p<1>(which, c);
  else if (FAM == 2 || (FAM == 5 && p == 2)) dg_dispatch_p<2>(which, c);
  else if (FAM == 3 || (FAM == 5 && p == 3)) dg_dispatch_p<3>(which, c);
  else if (FAM == 4 || (FAM == 5 && p == 4)) dg_dispatch_p<4>(which, c);
}

inline int dg_nd(int p) { return (p + 1) * (p + 2) / 2; }

inline int64_t dg_param_count(int k) {
  const int p = k / 5 + 1, which = k % 5, nd = dg_nd(p), nq = p + 1;
  switch (which) {
    case 0: return 2 * nd * nd;
    case 1:
    case 2: return 6 * nq * nd;
    case 4: return 1;
    default: return 0;
  }
}

inline void dg_validate(int k, size_t j, const ChainView &cv, const LoopDesc &L,
                        const lt_arg *args) {
  const int p = k / 5 + 1, which = k % 5, nd = dg_nd(p);
  static const int want[5][6] = {{5, 5, 2, 3, 2, 3}, {5, 5, 2, 3, 2, 3}, {5, 5, 2, 3, 2, 3},
                                 {5, 5, 2, 3, 0, 0}, {2, 3, 2, 3, 0, 0}};
  static const bool scaled[5][6] = {{0, 0, 1, 1, 1, 1}, {0, 0, 1, 1, 1, 1}, {0, 0, 1, 1, 1, 1},
                                    {0, 0, 1, 1, 0, 0}, {1, 1, 1, 1, 0, 0}};
  for (size_t d = 0; d < L.desc.size(); ++d) {
    const int v = scaled[which][d] ? want[which][d] * nd : want[which][d];
    if (args[d].vpe != v)
      fail(LT_E_EXECUTION, "loop " + std::to_string(j) + " arg " + std::to_string(d) +
                               ": DG P" + std::to_string(p) + " kernel needs values_per_element " +
                               std::to_string(v) + ", got " + std::to_string(args[d].vpe));
  }
  if (which == 1 || which == 2) {
    const int want_ar = which == 1 ? 2 : 1;
    for (size_t d = 1; d < L.desc.size(); ++d)
      if (cv.maps[L.desc[d].map].arity != want_ar)
        fail(LT_E_EXECUTION, "loop " + std::to_string(j) + ": facet kernel needs a map of arity " +
                                 std::to_string(want_ar));
  }
}

}  // namespace lt
