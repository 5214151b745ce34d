// lt_dg.cuh — elastic-wave DG kernel bodies (velocity-stress, modal P1..P4).
//
// Discretisation: paper_1708_03183_b200/dg.py (module docstring); numpy twin:
// oracle/dg_oracle.py.  G lanes per element (cell or facet), lane i owning
// DoF row i; operator tables (S_r, S_s, face traces E, lifts) come from the
// kernel's parameter block (read-only, L1-cached).  Facet kernels produce
// per-side increments that the executor applies in reference order: from
// contribution slots (untiled / global executors) or straight from registers
// in rank rounds (staged executors).
#pragma once

#include "lt_kernels.cuh"

namespace lt {

template <int P>
struct DGShape {
  static constexpr int ND = (P + 1) * (P + 2) / 2;
  static constexpr int NQ = P + 1;
};

// Work items ("lanes") per element: cell kernels one per DoF row i < ND (lane
// i owns component f*ND + i of u, s, ru, rs), facet kernels one per facet
// point q < NQ.  Lanes never communicate: each writes its own outputs.
// L0: R = |J| (div sigma ; C:grad v)   [cgeo R, mat R, u R, s R, ru W, rs W]
#ifndef LT_VEC_DG
#define LT_VEC_DG 1  // 16-byte shared/global loads of DoF pairs when ND is even
#endif

// Rows whose field segments start at even offsets (ND even) and whose base is
// 16-byte aligned can be read two DoFs per load (LDS.128 / LDG.128): half the
// load instructions of the contractions, same arithmetic order.
// (measured: +1 % at P3 in the 168-register build, -2.4 % at P2; P1 and P4
// have odd ND; so only ND >= 10)
template <int ND>
__device__ __forceinline__ bool dg_pairs(const double *a, const double *b) {
  return LT_VEC_DG && ND % 2 == 0 && ND >= 10 &&
         ((((uintptr_t)a) | ((uintptr_t)b)) & 15) == 0;
}

__device__ __forceinline__ double2 ld2(const double *p) {
  return *reinterpret_cast<const double2 *>(p);
}

template <int P, class C>
__device__ __forceinline__ void dg_vol(C &c, int i) {
  constexpr int ND = DGShape<P>::ND;
  if (i >= ND) return;
  const double *g = c.rd(0), *m = c.rd(1), *u = c.rd(2), *s = c.rd(3);
  double *ru = c.wr(4), *rs = c.wr(5);
  const double *__restrict__ Sr = c.params() + i * ND;
  const double *__restrict__ Ss = Sr + ND * ND;
  double dr[5], ds[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) { dr[q] = 0.0; ds[q] = 0.0; }
  if (dg_pairs<ND>(u, s)) {
#pragma unroll
    for (int j = 0; j < ND; j += 2) {
      const double2 a = __ldg(reinterpret_cast<const double2 *>(Sr + j));
      const double2 b = __ldg(reinterpret_cast<const double2 *>(Ss + j));
      const double2 f0 = ld2(u + j), f1 = ld2(u + ND + j), f2 = ld2(s + j),
                    f3 = ld2(s + ND + j), f4 = ld2(s + 2 * ND + j);
      const double fa[5] = {f0.x, f1.x, f2.x, f3.x, f4.x};
      const double fb[5] = {f0.y, f1.y, f2.y, f3.y, f4.y};
#pragma unroll
      for (int q = 0; q < 5; ++q) { dr[q] += a.x * fa[q]; ds[q] += b.x * fa[q]; }
#pragma unroll
      for (int q = 0; q < 5; ++q) { dr[q] += a.y * fb[q]; ds[q] += b.y * fb[q]; }
    }
  } else {
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      const double a = __ldg(Sr + j), b = __ldg(Ss + j);
      const double f[5] = {u[j], u[ND + j], s[j], s[ND + j], s[2 * ND + j]};
#pragma unroll
      for (int q = 0; q < 5; ++q) { dr[q] += a * f[q]; ds[q] += b * f[q]; }
    }
  }
  const double rx = g[0], ry = g[1], sx = g[2], sy = g[3], det = g[4];
  const double lam = m[1], mu = m[2], l2m = lam + 2.0 * mu;
  double dx[5], dy[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) { dx[q] = rx * dr[q] + sx * ds[q]; dy[q] = ry * dr[q] + sy * ds[q]; }
  ru[i] = det * (dx[2] + dy[4]);
  ru[ND + i] = det * (dx[4] + dy[3]);
  rs[i] = det * (l2m * dx[0] + lam * dy[1]);
  rs[ND + i] = det * (lam * dx[0] + l2m * dy[1]);
  rs[2 * ND + i] = det * mu * (dy[0] + dx[1]);
}

// One output row of a lifted facet correction:
//   o[f] = jf * sum_q LIFT[face][i][q] * corr[f][q]   (corr in the side's own point order)
template <int ND, int NQ>
__device__ __forceinline__ void dg_lift_row(const double *__restrict__ LIFT, int face, int i,
                                            double jf, const double *corr, double o[5]) {
  const double *Lr = LIFT + (face * ND + i) * NQ;
  double a[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double w = __ldg(Lr + q);
#pragma unroll
    for (int f = 0; f < 5; ++f) a[f] += w * corr[f * NQ + q];
  }
#pragma unroll
  for (int f = 0; f < 5; ++f) o[f] = jf * a[f];
}

// trace of the 5 fields at point `pt` of `face`
template <int ND, int NQ>
__device__ __forceinline__ void dg_trace(const double *__restrict__ E, int face, int pt,
                                         const double *u, const double *s, double t[5]) {
  const double *e = E + (face * NQ + pt) * ND;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
  if (dg_pairs<ND>(u, s)) {
#pragma unroll
    for (int j = 0; j < ND; j += 2) {
      const double2 w = __ldg(reinterpret_cast<const double2 *>(e + j));
      const double2 f0 = ld2(u + j), f1 = ld2(u + ND + j), f2 = ld2(s + j),
                    f3 = ld2(s + ND + j), f4 = ld2(s + 2 * ND + j);
      a0 += w.x * f0.x;
      a1 += w.x * f1.x;
      a2 += w.x * f2.x;
      a3 += w.x * f3.x;
      a4 += w.x * f4.x;
      a0 += w.y * f0.y;
      a1 += w.y * f1.y;
      a2 += w.y * f2.y;
      a3 += w.y * f3.y;
      a4 += w.y * f4.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      const double w = __ldg(e + j);
      a0 += w * u[j];
      a1 += w * u[ND + j];
      a2 += w * s[j];
      a3 += w * s[ND + j];
      a4 += w * s[2 * ND + j];
    }
  }
  t[0] = a0; t[1] = a1; t[2] = a2; t[3] = a3; t[4] = a4;
}

// Per-side correction record of a facet (the deferred form of its increment):
// [corr f=0..4][q=0..NQ-1] in the side's own point order, jf, face.  The
// executor's deferred apply lifts records per (target, DoF row) and adds them
// in the reference's (element, k) order.

// Upwind flux of one interior facet point from the two traces (side a's point
// q, side b's own point NQ-1-q): per-side corrections ra[f*NQ], rb[f*NQ].
template <int NQ>
__device__ __forceinline__ void dg_iflux_point(double nx, double ny, const double *ma,
                                               const double *mb, const double ta[5],
                                               const double tb[5], double *ra, double *rb) {
  const double la = ma[1], mua = ma[2], lb = mb[1], mub = mb[2];
  const double zpa = ma[3], zsa = ma[4], zpb = mb[3], zsb = mb[4];  // impedances rho*c_p, rho*c_s
  const double ip = 1.0 / (zpa + zpb), is = 1.0 / (zsa + zsb);
  const double tnx = -ny, tny = nx;
  const double Tax = ta[2] * nx + ta[4] * ny, Tay = ta[4] * nx + ta[3] * ny;
  const double Tbx = tb[2] * nx + tb[4] * ny, Tby = tb[4] * nx + tb[3] * ny;
  const double vna = ta[0] * nx + ta[1] * ny, vta = ta[0] * tnx + ta[1] * tny;
  const double vnb = tb[0] * nx + tb[1] * ny, vtb = tb[0] * tnx + tb[1] * tny;
  const double Tna = Tax * nx + Tay * ny, Tta = Tax * tnx + Tay * tny;
  const double Tnb = Tbx * nx + Tby * ny, Ttb = Tbx * tnx + Tby * tny;
  const double dvn = (Tnb - Tna + zpb * (vnb - vna)) * ip;
  const double dvt = (Ttb - Tta + zsb * (vtb - vta)) * is;
  const double dTax = zpa * dvn * nx + zsa * dvt * tnx;
  const double dTay = zpa * dvn * ny + zsa * dvt * tny;
  const double dvax = dvn * nx + dvt * tnx, dvay = dvn * ny + dvt * tny;
  const double dna = dvax * nx + dvay * ny;
  ra[0] = dTax;
  ra[NQ] = dTay;
  ra[2 * NQ] = la * dna + 2.0 * mua * dvax * nx;
  ra[3 * NQ] = la * dna + 2.0 * mua * dvay * ny;
  ra[4 * NQ] = mua * (dvax * ny + dvay * nx);
  const double dvbx = ta[0] + dvax - tb[0], dvby = ta[1] + dvay - tb[1];
  const double dnb = -(dvbx * nx + dvby * ny);
  rb[0] = (Tbx - Tax) - dTax;
  rb[NQ] = (Tby - Tay) - dTay;
  rb[2 * NQ] = lb * dnb - 2.0 * mub * dvbx * nx;
  rb[3 * NQ] = lb * dnb - 2.0 * mub * dvby * ny;
  rb[4 * NQ] = -mub * (dvbx * ny + dvby * nx);
}

// L1: interior facets, upwind flux at point q (side a's order; side b's own
// point is NQ-1-q)   [fgeo R, mat R@2, u R@2, s R@2, ru I@2, rs I@2]
template <int P, class C>
__device__ __forceinline__ void dg_iflux(C &c, int q) {
  constexpr int ND = DGShape<P>::ND, NQ = DGShape<P>::NQ;
  if (q >= NQ) return;
  const double *g = c.rd(0);
  const double nx = g[0], ny = g[1];
  const int fa = (int)g[3], fb = (int)g[4];
  const double *ma = c.rdm(1, 0), *mb = c.rdm(1, 1);
  const double *__restrict__ E = c.params();
  double ta[5], tb[5];
  dg_trace<ND, NQ>(E, fa, q, c.rdm(2, 0), c.rdm(3, 0), ta);
  dg_trace<ND, NQ>(E, fb, NQ - 1 - q, c.rdm(2, 1), c.rdm(3, 1), tb);
  dg_iflux_point<NQ>(nx, ny, ma, mb, ta, tb, c.rec(0) + q, c.rec(1) + (NQ - 1 - q));
  if (C::kRecGeo && q == 0) {  // staged records omit |f|/2 and the face (read from fgeo)
    double *r0 = c.rec(0) + 5 * NQ, *r1 = c.rec(1) + 5 * NQ;
    r0[0] = g[2];
    r0[1] = g[3];
    r1[0] = g[2];
    r1[1] = g[4];
  }
}

// Traction-free mirror state at one exterior facet point: corrections r[f*NQ].
template <int NQ>
__device__ __forceinline__ void dg_eflux_point(double nx, double ny, const double *m,
                                               const double t[5], double *r) {
  const double lam = m[1], mu = m[2];
  const double izp = 1.0 / m[3], izs = 1.0 / m[4];
  const double tnx = -ny, tny = nx;
  const double Tx = t[2] * nx + t[4] * ny, Ty = t[4] * nx + t[3] * ny;
  const double dvn = -(Tx * nx + Ty * ny) * izp;
  const double dvt = -(Tx * tnx + Ty * tny) * izs;
  const double dvx = dvn * nx + dvt * tnx, dvy = dvn * ny + dvt * tny;
  const double dn = dvx * nx + dvy * ny;
  r[0] = -Tx;
  r[NQ] = -Ty;
  r[2 * NQ] = lam * dn + 2.0 * mu * dvx * nx;
  r[3 * NQ] = lam * dn + 2.0 * mu * dvy * ny;
  r[4 * NQ] = mu * (dvx * ny + dvy * nx);
}

// L2: exterior facets, traction-free mirror state, point q
template <int P, class C>
__device__ __forceinline__ void dg_eflux(C &c, int q) {
  constexpr int ND = DGShape<P>::ND, NQ = DGShape<P>::NQ;
  if (q >= NQ) return;
  const double *g = c.rd(0);
  const double nx = g[0], ny = g[1];
  const int fa = (int)g[3];
  const double *m = c.rdm(1, 0);
  const double *__restrict__ E = c.params();
  double t[5];
  dg_trace<ND, NQ>(E, fa, q, c.rdm(2, 0), c.rdm(3, 0), t);
  dg_eflux_point<NQ>(nx, ny, m, t, c.rec(0) + q);
  if (C::kRecGeo && q == 0) {
    c.rec(0)[5 * NQ] = g[2];
    c.rec(0)[5 * NQ + 1] = g[3];
  }
}

// L3: inverse mass (M_ref = I): ru /= rho |J|, rs /= |J|   [cgeo R, mat R, ru RW, rs RW]
template <int P, class C>
__device__ __forceinline__ void dg_minv(C &c, int i) {
  constexpr int ND = DGShape<P>::ND;
  if (i >= ND) return;
  const double det = c.rd(0)[4], rho = c.rd(1)[0];
  double *ru = c.wr(2), *rs = c.wr(3);
  const double iu = 1.0 / (rho * det), is = 1.0 / det;
  ru[i] *= iu;
  ru[ND + i] *= iu;
  rs[i] *= is;
  rs[ND + i] *= is;
  rs[2 * ND + i] *= is;
}

// L4: forward Euler   [u RW, s RW, ru R, rs R]  params: dt
template <int P, class C>
__device__ __forceinline__ void dg_axpy(C &c, int i) {
  constexpr int ND = DGShape<P>::ND;
  if (i >= ND) return;
  const double dt = c.params()[0];
  double *u = c.wr(0), *s = c.wr(1);
  const double *ru = c.rd(2), *rs = c.rd(3);
  u[i] += dt * ru[i];
  u[ND + i] += dt * ru[ND + i];
  s[i] += dt * rs[i];
  s[ND + i] += dt * rs[ND + i];
  s[2 * ND + i] += dt * rs[2 * ND + i];
}

// ---- grouped work items (shared-memory tile executors) ------------------------------
// The tile executors run a DG loop as (element, group) items with the element
// index fastest across lanes: a cell item owns RV DoF rows and reads the cell's
// fields once for all of them; a facet item owns QF facet points and reads both
// cells' fields once for all of them.  Per accumulator the summation order is
// that of the one-row / one-point bodies above (j ascending), so the arithmetic
// is the same; only the number of shared-memory and table loads per DFMA drops
// (P3: 9 loads per 40 DFMA instead of 7 per 10).
template <int P>
struct DGGroup {
  static constexpr int ND = DGShape<P>::ND, NQ = DGShape<P>::NQ;
  static constexpr int RV = P == 1 ? 1 : 2;               // DoF rows per cell item
  static constexpr int GV = (ND + RV - 1) / RV;           // cell items per cell
  static constexpr int QF = P <= 2 ? NQ : (NQ + 1) / 2;   // facet points per facet item
  static constexpr int GF = (NQ + QF - 1) / QF;           // facet items per facet
  static constexpr int RA = P <= 2 ? 3 : 5;               // DoF rows per deferred-apply item
  static constexpr int GA = (ND + RA - 1) / RA;           // apply items per target
};

template <int ND>
__device__ __forceinline__ bool dg_pairs_g(const double *a, const double *b) {
  return ND % 2 == 0 && ((((uintptr_t)a) | ((uintptr_t)b)) & 15) == 0;
}

template <int P, class C>
__device__ __forceinline__ void dg_vol_g(C &c, int g) {
  constexpr int ND = DGShape<P>::ND, RV = DGGroup<P>::RV;
  const double *gm = c.rd(0), *m = c.rd(1), *u = c.rd(2), *s = c.rd(3);
  double *ru = c.wr(4), *rs = c.wr(5);
  const double *__restrict__ Sr = c.params();
  const double *__restrict__ Ss = Sr + ND * ND;
  const int i0 = g * RV;
  const double *a[RV], *b[RV];  // operator rows (the last group of an odd ND repeats a row)
  double dr[RV][5], ds[RV][5];
#pragma unroll
  for (int r = 0; r < RV; ++r) {
    const int row = min(i0 + r, ND - 1);
    a[r] = Sr + row * ND;
    b[r] = Ss + row * ND;
#pragma unroll
    for (int q = 0; q < 5; ++q) { dr[r][q] = 0.0; ds[r][q] = 0.0; }
  }
  if (dg_pairs_g<ND>(u, s)) {
#pragma unroll
    for (int j = 0; j < ND - 1; j += 2) {
      const double2 f0 = ld2(u + j), f1 = ld2(u + ND + j), f2 = ld2(s + j),
                    f3 = ld2(s + ND + j), f4 = ld2(s + 2 * ND + j);
      const double fa[5] = {f0.x, f1.x, f2.x, f3.x, f4.x};
      const double fb[5] = {f0.y, f1.y, f2.y, f3.y, f4.y};
#pragma unroll
      for (int r = 0; r < RV; ++r) {
        const double2 x = __ldg(reinterpret_cast<const double2 *>(a[r] + j));
        const double2 y = __ldg(reinterpret_cast<const double2 *>(b[r] + j));
#pragma unroll
        for (int q = 0; q < 5; ++q) { dr[r][q] += x.x * fa[q]; ds[r][q] += y.x * fa[q]; }
#pragma unroll
        for (int q = 0; q < 5; ++q) { dr[r][q] += x.y * fb[q]; ds[r][q] += y.y * fb[q]; }
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      const double f[5] = {u[j], u[ND + j], s[j], s[ND + j], s[2 * ND + j]};
#pragma unroll
      for (int r = 0; r < RV; ++r) {
        const double x = __ldg(a[r] + j), y = __ldg(b[r] + j);
#pragma unroll
        for (int q = 0; q < 5; ++q) { dr[r][q] += x * f[q]; ds[r][q] += y * f[q]; }
      }
    }
  }
  const double rx = gm[0], ry = gm[1], sx = gm[2], sy = gm[3], det = gm[4];
  const double lam = m[1], mu = m[2], l2m = lam + 2.0 * mu;
#pragma unroll
  for (int r = 0; r < RV; ++r) {
    const int i = i0 + r;
    if (i < ND) {
      double dx[5], dy[5];
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        dx[q] = rx * dr[r][q] + sx * ds[r][q];
        dy[q] = ry * dr[r][q] + sy * ds[r][q];
      }
      ru[i] = det * (dx[2] + dy[4]);
      ru[ND + i] = det * (dx[4] + dy[3]);
      rs[i] = det * (l2m * dx[0] + lam * dy[1]);
      rs[ND + i] = det * (lam * dx[0] + l2m * dy[1]);
      rs[2 * ND + i] = det * mu * (dy[0] + dx[1]);
    }
  }
}

// traces of the 5 fields at QF points pt[k] of `face`, the cell's fields read once
template <int ND, int NQ, int QF>
__device__ __forceinline__ void dg_trace_g(const double *__restrict__ E, int face,
                                           const int (&pt)[QF], const double *u, const double *s,
                                           double (&t)[QF][5]) {
  const double *e[QF];
#pragma unroll
  for (int k = 0; k < QF; ++k) {
    e[k] = E + (face * NQ + pt[k]) * ND;
#pragma unroll
    for (int f = 0; f < 5; ++f) t[k][f] = 0.0;
  }
  if (dg_pairs_g<ND>(u, s)) {
#pragma unroll
    for (int j = 0; j < ND - 1; j += 2) {
      const double2 f0 = ld2(u + j), f1 = ld2(u + ND + j), f2 = ld2(s + j),
                    f3 = ld2(s + ND + j), f4 = ld2(s + 2 * ND + j);
#pragma unroll
      for (int k = 0; k < QF; ++k) {
        const double2 w = __ldg(reinterpret_cast<const double2 *>(e[k] + j));
        t[k][0] += w.x * f0.x;
        t[k][1] += w.x * f1.x;
        t[k][2] += w.x * f2.x;
        t[k][3] += w.x * f3.x;
        t[k][4] += w.x * f4.x;
        t[k][0] += w.y * f0.y;
        t[k][1] += w.y * f1.y;
        t[k][2] += w.y * f2.y;
        t[k][3] += w.y * f3.y;
        t[k][4] += w.y * f4.y;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      const double f[5] = {u[j], u[ND + j], s[j], s[ND + j], s[2 * ND + j]};
#pragma unroll
      for (int k = 0; k < QF; ++k) {
        const double w = __ldg(e[k] + j);
#pragma unroll
        for (int q = 0; q < 5; ++q) t[k][q] += w * f[q];
      }
    }
  }
}

// interior facet item: points pg*QF .. pg*QF+QF-1 (side a's order)
template <int P, class C>
__device__ __forceinline__ void dg_iflux_g(C &c, int pg) {
  constexpr int ND = DGShape<P>::ND, NQ = DGShape<P>::NQ, QF = DGGroup<P>::QF;
  static_assert(!C::kRecGeo, "grouped facet items: records without geometry");
  const double *g = c.rd(0);
  const double nx = g[0], ny = g[1];
  const int fa = (int)g[3], fb = (int)g[4];
  const double *ma = c.rdm(1, 0), *mb = c.rdm(1, 1);
  const double *__restrict__ E = c.params();
  const int q0 = pg * QF;
  int pa[QF], pb[QF];
#pragma unroll
  for (int k = 0; k < QF; ++k) {
    pa[k] = min(q0 + k, NQ - 1);
    pb[k] = NQ - 1 - pa[k];
  }
  double ta[QF][5], tb[QF][5];
  dg_trace_g<ND, NQ, QF>(E, fa, pa, c.rdm(2, 0), c.rdm(3, 0), ta);
  dg_trace_g<ND, NQ, QF>(E, fb, pb, c.rdm(2, 1), c.rdm(3, 1), tb);
  double *ra = c.rec(0), *rb = c.rec(1);
#pragma unroll
  for (int k = 0; k < QF; ++k)
    if (q0 + k < NQ) dg_iflux_point<NQ>(nx, ny, ma, mb, ta[k], tb[k], ra + pa[k], rb + pb[k]);
}

template <int P, class C>
__device__ __forceinline__ void dg_eflux_g(C &c, int pg) {
  constexpr int ND = DGShape<P>::ND, NQ = DGShape<P>::NQ, QF = DGGroup<P>::QF;
  static_assert(!C::kRecGeo, "grouped facet items: records without geometry");
  const double *g = c.rd(0);
  const double nx = g[0], ny = g[1];
  const int fa = (int)g[3];
  const double *m = c.rdm(1, 0);
  const double *__restrict__ E = c.params();
  const int q0 = pg * QF;
  int pa[QF];
#pragma unroll
  for (int k = 0; k < QF; ++k) pa[k] = min(q0 + k, NQ - 1);
  double t[QF][5];
  dg_trace_g<ND, NQ, QF>(E, fa, pa, c.rdm(2, 0), c.rdm(3, 0), t);
  double *r = c.rec(0);
#pragma unroll
  for (int k = 0; k < QF; ++k)
    if (q0 + k < NQ) dg_eflux_point<NQ>(nx, ny, m, t[k], r + pa[k]);
}

// ---- field-lane volume items: operator tables as constant-bank operands ------------
// One lane per (cell, field f < 5): the lane reads the ND values of its field
// once and applies every row of S_r and S_s to them.  The operator entries are
// then the same for all lanes, so they come from the constant bank as DFMA
// operands (no load instruction, no shared-memory or L1 traffic): a cell costs
// 5 x ND/2 16-byte shared loads instead of 10 lanes x 5 ND/2 broadcast loads
// plus ND^2 table loads.  The five fields of a cell sit in adjacent lanes of
// one warp (6 cells per warp, lanes 30-31 idle); the output field g needs one
// x- and one y-derivative of two other fields, fetched with two shuffles per
// DoF.  Same products and sums per value as dg_vol (j ascending).
// The tables are mirrored from the kernel's parameter block before every launch
// (refresh_const_tables); one mirror per degree.
__constant__ double c_dg_vol_p1[2 * 3 * 3];
__constant__ double c_dg_vol_p2[2 * 6 * 6];
__constant__ double c_dg_vol_p3[2 * 10 * 10];
__constant__ double c_dg_vol_p4[2 * 15 * 15];

template <int P>
__device__ __forceinline__ double dg_cvol(int k) {
  if constexpr (P == 1) return c_dg_vol_p1[k];
  else if constexpr (P == 2) return c_dg_vol_p2[k];
  else if constexpr (P == 3) return c_dg_vol_p3[k];
  else return c_dg_vol_p4[k];
}

// f: the lane's field (0 vx, 1 vy, 2 sxx, 3 syy, 4 sxy); base: first lane of the
// cell's five; valid: the lane owns a cell of the list (others only shuffle)
template <int P, class C>
__device__ __forceinline__ void dg_vol_f(C &c, int f, int base, bool valid) {
  constexpr int ND = DGShape<P>::ND;
  const double *gm = c.rd(0), *m = c.rd(1);
  const double *col = f < 2 ? c.rd(2) + f * ND : c.rd(3) + (f - 2) * ND;
  double F[ND];
  if (dg_pairs_g<ND>(col, col)) {
#pragma unroll
    for (int j = 0; j < ND - 1; j += 2) {
      const double2 v = ld2(col + j);
      F[j] = v.x;
      F[j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < ND; ++j) F[j] = col[j];
  }
  const double rx = gm[0], ry = gm[1], sx = gm[2], sy = gm[3], det = gm[4];
  const double lam = m[1], mu = m[2], l2m = lam + 2.0 * mu;
  double dx[ND], dy[ND];
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      a += dg_cvol<P>(i * ND + j) * F[j];
      b += dg_cvol<P>(ND * ND + i * ND + j) * F[j];
    }
    dx[i] = rx * a + sx * b;
    dy[i] = ry * a + sy * b;
  }
  // output g = f:  ru_x = det (dx[sxx] + dy[sxy])      ru_y = det (dx[sxy] + dy[syy])
  //   rs_xx = det (l2m dx[vx] + lam dy[vy])   rs_yy = det (lam dx[vx] + l2m dy[vy])
  //   rs_xy = det mu (dy[vx] + dx[vy])
  const int sxl = (base + (f == 0 ? 2 : f == 1 ? 4 : f == 4 ? 1 : 0)) & 31;
  const int syl = (base + (f == 0 ? 4 : f == 1 ? 3 : f == 4 ? 0 : 1)) & 31;
  const double cx = f == 2 ? l2m : f == 3 ? lam : 1.0;
  const double cy = f == 2 ? lam : f == 3 ? l2m : 1.0;
  const double sc = f == 4 ? det * mu : det;
  double *out = f < 2 ? c.wr(4) + f * ND : c.wr(5) + (f - 2) * ND;
  double o[ND];
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    const double X = __shfl_sync(0xffffffffu, dx[i], sxl);
    const double Y = __shfl_sync(0xffffffffu, dy[i], syl);
    o[i] = f < 2 || f == 4 ? sc * (f == 4 ? Y + X : X + Y) : sc * (cx * X + cy * Y);
  }
  if (!valid) return;
  if (dg_pairs_g<ND>(out, out)) {
#pragma unroll
    for (int i = 0; i < ND - 1; i += 2)
      *reinterpret_cast<double2 *>(out + i) = make_double2(o[i], o[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < ND; ++i) out[i] = o[i];
  }
}

// inverse mass / forward Euler as (cell, field f < 5) items: the ND values of
// one field, contiguous in the cell's row (16-byte pairs when ND is even)
template <int P, class C>
__device__ __forceinline__ void dg_minv_g(C &c, int f) {
  constexpr int ND = DGShape<P>::ND;
  const double det = c.rd(0)[4], rho = c.rd(1)[0];
  const double iu = 1.0 / (rho * det), is = 1.0 / det;
  double *r = f < 2 ? c.wr(2) + f * ND : c.wr(3) + (f - 2) * ND;
  const double sc = f < 2 ? iu : is;
  if (dg_pairs_g<ND>(r, r)) {
#pragma unroll
    for (int j = 0; j < ND - 1; j += 2) {
      double2 v = ld2(r + j);
      v.x *= sc;
      v.y *= sc;
      *reinterpret_cast<double2 *>(r + j) = v;
    }
  } else {
#pragma unroll
    for (int j = 0; j < ND; ++j) r[j] *= sc;
  }
}

template <int P, class C>
__device__ __forceinline__ void dg_axpy_g(C &c, int f) {
  constexpr int ND = DGShape<P>::ND;
  const double dt = c.params()[0];
  double *x = f < 2 ? c.wr(0) + f * ND : c.wr(1) + (f - 2) * ND;
  const double *r = f < 2 ? c.rd(2) + f * ND : c.rd(3) + (f - 2) * ND;
  if (dg_pairs_g<ND>(x, r)) {
#pragma unroll
    for (int j = 0; j < ND - 1; j += 2) {
      double2 v = ld2(x + j);
      const double2 w = ld2(r + j);
      v.x += dt * w.x;
      v.y += dt * w.y;
      *reinterpret_cast<double2 *>(x + j) = v;
    }
  } else {
#pragma unroll
    for (int j = 0; j < ND; ++j) x[j] += dt * r[j];
  }
}

// deferred apply of one record to RA rows of its target: the record is read
// once; acc[r][f] += jf * sum_q LIFT[face][i0+r][q] * corr[f][q]
template <int P>
__device__ __forceinline__ void dg_lift_rows_g(const double *__restrict__ params, int face, int i0,
                                               double jf, const double *rec,
                                               double (&acc)[DGGroup<P>::RA][5]) {
  constexpr int ND = DGShape<P>::ND, NQ = DGShape<P>::NQ, RV = DGGroup<P>::RA;
  const double *__restrict__ LIFT = params + 3 * NQ * ND;
  double corr[5][NQ];
#pragma unroll
  for (int f = 0; f < 5; ++f)
#pragma unroll
    for (int q = 0; q < NQ; ++q) corr[f][q] = rec[f * NQ + q];
#pragma unroll
  for (int r = 0; r < RV; ++r) {
    const double *Lr = LIFT + (face * ND + min(i0 + r, ND - 1)) * NQ;
    double a[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double w = __ldg(Lr + q);
#pragma unroll
      for (int f = 0; f < 5; ++f) a[f] += w * corr[f][q];
    }
#pragma unroll
    for (int f = 0; f < 5; ++f) acc[r][f] += jf * a[f];
  }
}

template <int P, class C>
__device__ __forceinline__ void dg_dispatch_p(int which, C &c, int lane) {
  switch (which) {
    case 0: dg_vol<P>(c, lane); break;
    case 1: dg_iflux<P>(c, lane); break;
    case 2: dg_eflux<P>(c, lane); break;
    case 3: dg_minv<P>(c, lane); break;
    case 4: dg_axpy<P>(c, lane); break;
  }
}

// family: 0 none, 1..4 only degree P, 5 all degrees
#define LT_DG_FAMILY(FAM, k, CALL)                                  \
  do {                                                              \
    const int p_ = (k) / 5 + 1;                                     \
    if (FAM == 1 || (FAM == 5 && p_ == 1)) { constexpr int P = 1; CALL; } \
    else if (FAM == 2 || (FAM == 5 && p_ == 2)) { constexpr int P = 2; CALL; } \
    else if (FAM == 3 || (FAM == 5 && p_ == 3)) { constexpr int P = 3; CALL; } \
    else if (FAM == 4 || (FAM == 5 && p_ == 4)) { constexpr int P = 4; CALL; } \
  } while (0)

template <int FAM, class C>
__device__ __forceinline__ void dg_dispatch(int k, C &c, int lane) {
  LT_DG_FAMILY(FAM, k, (dg_dispatch_p<P>(k % 5, c, lane)));
}

// deferred apply of one (target row i): acc[f] += lift of each record, in order
// same with |f|/2 and the face given (staged records carry corrections only)
template <int FAM>
__device__ __forceinline__ void dg_lift_acc_g(int k, const double *__restrict__ params, int i,
                                              const double *rec, double jf, int face,
                                              double acc[5]) {
  LT_DG_FAMILY(FAM, k, ({
                 constexpr int ND = DGShape<P>::ND, NQ = DGShape<P>::NQ;
                 const double *__restrict__ LIFT = params + 3 * NQ * ND;
                 double o[5];
                 dg_lift_row<ND, NQ>(LIFT, face, i, jf, rec, o);
#pragma unroll
                 for (int f = 0; f < 5; ++f) acc[f] += o[f];
               }));
}

template <int FAM>
__device__ __forceinline__ void dg_lift_acc(int k, const double *__restrict__ params, int i,
                                            const double *rec, double acc[5]) {
  LT_DG_FAMILY(FAM, k, ({
                 constexpr int ND = DGShape<P>::ND, NQ = DGShape<P>::NQ;
                 const double *__restrict__ LIFT = params + 3 * NQ * ND;
                 double o[5];
                 dg_lift_row<ND, NQ>(LIFT, (int)rec[5 * NQ + 1], i, rec[5 * NQ], rec, o);
#pragma unroll
                 for (int f = 0; f < 5; ++f) acc[f] += o[f];
               }));
}

inline int dg_nd(int p) { return (p + 1) * (p + 2) / 2; }
// work items per element of DG kernel k: DoF rows (cells) or facet points
inline int dg_lanes(int k) {
  if (k % 5 == 1 || k % 5 == 2) return k / 5 + 2;
  return dg_nd(k / 5 + 1);
}
// doubles of one per-side correction record: 5 NQ corrections, jf, face
// (record stride rounded up to odd: conflict-free 64-bit shared-memory reads)
inline int dg_corr_size(int k) { return (5 * (k / 5 + 2) + 2) | 1; }
// staged executors: corrections only (|f|/2 and the face come from the facet's
// geometry row), stride rounded up to odd
inline int dg_corr_size_staged(int k) { return (5 * (k / 5 + 2)) | 1; }
inline bool dg_is_flux(int k) { return k % 5 == 1 || k % 5 == 2; }

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
    if (L.desc[4].map != L.desc[5].map || L.desc[4].mode != LT_INC || L.desc[5].mode != LT_INC)
      fail(LT_E_EXECUTION, "loop " + std::to_string(j) +
                               ": facet kernel increments ru and rs (INC) through one map");
  }
}

}  // namespace lt
