// lt_kernels.cuh — native kernel bodies (the executor's plugin surface).
//
// The reference registers Python callables by kernel id (executor.py:46-61;
// bodies problems.py:49-64).  Here a kernel id names a device function; the
// executor hands it an access context `C` that resolves each descriptor:
//   C::rd(d)      const double* of the element's own values      (direct)
//   C::wr(d)      double*       of the element's own values      (direct W/RW)
//   C::rdm(d, k)  const double* of the k-th mapped target         (mapped READ)
//   C::inc(d, k)  double*       contribution slot for target k    (mapped INC / WRITE)
// Bodies are called once per (element, lane), lane < the kernel's lanes
// (scalar bodies: 1 lane); lanes of an element write disjoint outputs.
// Mapped INC/WRITE bodies never touch the target itself: they fill their
// contribution slot and the executor applies the slots in the reference's
// sequential order (element ascending, then k) -- no atomics anywhere.
//
// Scalar bodies are restated with __dadd_rn/__dmul_rn/__ddiv_rn so no FMA
// contraction can occur: results are bitwise equal to numpy's.
#pragma once

#include "lt_internal.cuh"

namespace lt {

enum KernelId : int32_t {
  K_EDGE_INC = 0,   // problems.py:49-51  verts[k] += x
  K_CELL_INC,       // problems.py:54-56  v += res for v in verts
  K_EDGE_READ,      // problems.py:59-60  out = verts[0] + verts[1]
  K_CELL_READ,      // problems.py:63-64  out = verts[0] + verts[1] + verts[2]
  K_TOY_K1,         // BASELINE config 1, L1: v_k += a / 3
  K_TOY_K2,         // BASELINE config 1, L2: e = 0.5 * (v0 + v1)
  K_TOY_K3,         // BASELINE config 1, L3: a += (e0 + e1 + e2) / 3
  K_DG_FIRST,       // elastic-wave DG kernels, see lt_dg.cuh
};

struct KernelInfo {
  const char *name;
  int32_t nargs;
};

// Per-descriptor binding resolved for the device
struct DArg {
  double *data;
  const int32_t *map;   // global map values (nullptr if direct)
  const int32_t *lmap;  // local map (tile-list order), tiled executor only
  double *scr;          // untiled: global contribution scratch of this descriptor
  int32_t arity;
  int32_t vpe;
  int32_t mode;
  int32_t inc_off;      // tiled: offset (doubles) of this descriptor's slots in smem
  const int32_t *slot;  // staged: footprint slot per list position (direct) or (position, k)
  int32_t ds;           // staged: index of the staged dataset this descriptor binds
  int32_t sstride;      // staged: shared-memory row stride (odd: conflict-free 64-bit rows)
};

#define LT_MAX_STAGED 16  // distinct datasets staged in shared memory
#ifndef LT_SBLOCK
#define LT_SBLOCK 128     // threads per CTA of the staged tile executor
#endif

// One dataset staged in shared memory: the tile's footprint rows of it are
// gathered at tile start and the rows the tile wrote are stored back at the end.
#define LT_MAX_SPACES 8   // spaces with a staged footprint
#define LT_MAX_SLOOPS 24  // loops of a chain run by the staged executor

struct StageDS {
  double *data;
  int32_t vpe;
  int32_t stride;          // shared-memory row stride (vpe | 1)
  int32_t sp;              // footprint space index
  int32_t load;            // 1: gather every footprint row; 2: only the tile's load list
                           // (rows its first, full-writing loop does not overwrite)
  int32_t written;         // the tile writes some rows of it (store-back flags present)
  int32_t ro;              // never written by the chain: gathered before dependency waits
  // gather/store-back thread mapping: thread = (row offset < di, component < unit)
  int32_t di, dc;          // rows per pass LT_SBLOCK / unit, LT_SBLOCK % unit (unit: vpe or pairs)
  uint32_t magic;          // x / vpe == umulhi(x, magic) for x < 2^16 (vpe >= 2)
  int32_t vec;             // even vpe, 16-byte aligned: rows moved as 16-byte pairs
                           // (di, dc, magic then count pairs, vpe / 2 per row)
  int32_t tma;             // full-footprint gathers by TMA tile::gather4 (vec rows, dense
                           // shared stride, footprint rounded up to 4 rows)
};

// x / d for 0 <= x < 2^16, 1 <= d < 256, with magic = 2^32 / d + 1 (host: lt_magic)
__host__ __device__ __forceinline__ uint32_t lt_magic(int d) {
  return d > 1 ? (uint32_t)((1ull << 32) / (unsigned)d + 1) : 0u;
}
__device__ __forceinline__ int lt_div(int x, int d, uint32_t magic) {
  return d == 1 ? x : (int)__umulhi((unsigned)x, magic);
}

struct IncPlan {
  int32_t desc;
  int32_t plan;           // staged: index of the (loop, map) apply plan in the tile program
  const int32_t *gc_off;  // per global chunk: range of unique targets
  const int32_t *utgt;    // unique target ids
  const int32_t *ut_off;  // per unique target: range of contributor slots
  const int32_t *slots;   // contributor slot = pos_in_chunk*arity + k, ascending
};

struct DLoop {
  int32_t kernel;
  int32_t n_desc;
  int32_t chunk;            // tiled: elements per chunk (<= LT_BLOCK)
  int32_t n_inc;
  int32_t use_local;
  int32_t exec_size;
  int32_t n_plans;          // staged: distinct ordered-gather plans (maps) of the loop
  int32_t deferred;         // staged: INC applied by the kernel's deferred (lifting) apply
  int32_t lanes;            // work items (lanes) per element
  int32_t rec;              // deferred: doubles per (element, k) record in the scratch
  uint32_t lane_magic;      // lt_magic(lanes)
  int32_t lane_dq, lane_dr; // LT_SBLOCK / lanes, LT_SBLOCK % lanes
  uint32_t row_magic;       // deferred apply: lt_magic(rows per target)
  int32_t row_dq, row_dr;   // LT_SBLOCK / rows, LT_SBLOCK % rows
  int32_t nobar;            // staged: no barrier before the next loop (1: independent data,
                            // 2: same items, lane-local kernels -- fused per item)
  const double *params;
  const int32_t *offsets;   // tiled: per-tile list offsets
  const int32_t *elements;  // tiled: concatenated lists
  const int32_t *chunk_base;
  IncPlan inc[LT_MAX_INC];
  DArg a[LT_MAX_DESC];
};

// ---- scalar bodies -----------------------------------------------------------
template <class C>
__device__ __forceinline__ void body_edge_inc(C &c) {
  const double *x = c.rd(0);
  const int vpe = c.vpe(1);
  for (int k = 0; k < c.arity(1); ++k) {
    double *o = c.inc(1, k);
    for (int i = 0; i < vpe; ++i) o[i] = x[i];
  }
}

template <class C>
__device__ __forceinline__ void body_sum_read(C &c) {  // edge_read / cell_read
  double *out = c.wr(0);
  const int vpe = c.vpe(0);
  const int a = c.arity(1);
  for (int i = 0; i < vpe; ++i) {
    double s = c.rdm(1, 0)[i];
    for (int k = 1; k < a; ++k) s = __dadd_rn(s, c.rdm(1, k)[i]);
    out[i] = s;
  }
}

template <class C>
__device__ __forceinline__ void body_toy_k1(C &c) {
  const double *a = c.rd(0);
  const int vpe = c.vpe(1);
  for (int k = 0; k < c.arity(1); ++k) {
    double *o = c.inc(1, k);
    for (int i = 0; i < vpe; ++i) o[i] = __ddiv_rn(a[i], 3.0);
  }
}

template <class C>
__device__ __forceinline__ void body_toy_k2(C &c) {
  double *e = c.wr(0);
  const int vpe = c.vpe(0);
  for (int i = 0; i < vpe; ++i) e[i] = __dmul_rn(0.5, __dadd_rn(c.rdm(1, 0)[i], c.rdm(1, 1)[i]));
}

template <class C>
__device__ __forceinline__ void body_toy_k3(C &c) {
  double *a = c.wr(0);
  const int vpe = c.vpe(0);
  for (int i = 0; i < vpe; ++i) {
    double s = __dadd_rn(__dadd_rn(c.rdm(1, 0)[i], c.rdm(1, 1)[i]), c.rdm(1, 2)[i]);
    a[i] = __dadd_rn(a[i], __ddiv_rn(s, 3.0));
  }
}

}  // namespace lt
