// lt_exec.cu — executors: untiled per-loop kernels (execute_untiled,
// executor.py:163-169) and the fused tiled executor (execute_schedule,
// executor.py:185-245; Alg. 2).
//
// Fused tiled executor: one launch per colour phase, one CTA per tile.  The
// CTA runs every loop of the chain over its tile's iteration lists in chain
// order, separated by CTA barriers.  Mapped INC (and mapped WRITE)
// contributions of a chunk of <= LT_BLOCK elements go to shared memory; the
// chunk's unique targets are then updated by one thread each, applying the
// contributions in (element, k) order -- exactly the order of the reference's
// sequential per-tile execution, so results are bitwise those of
// execute_schedule.  No global atomics, no cross-CTA traffic: equal-coloured
// tiles touch disjoint written data by construction of the schedule.
#include <cub/cub.cuh>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <tuple>

#include "lt_dg.cuh"
#include "lt_kernels.cuh"
#include "lt_pairs.cuh"

namespace lt {

// ---- kernel table -------------------------------------------------------------
// signature tokens per descriptor: D* direct any, DR direct read, DW direct
// write/rw, DF direct write of every component (a WRITE binding then needs no
// load of the rows it writes), MR mapped read, MI mapped inc (or write)
struct KernelSpec {
  const char *name;
  const char *sig;
};

static const KernelSpec kSpecs[] = {
    {"edge_inc", "D*,MI"},  {"cell_inc", "D*,MI"},  {"edge_read", "DF,MR"},
    {"cell_read", "DF,MR"}, {"toy_k1", "D*,MI"},    {"toy_k2", "DF,MR"},
    {"toy_k3", "DW,MR"},
#define LT_DG_SPEC(P)                                                                  \
  {"dg_vol_p" #P, "DR,DR,DR,DR,DF,DF"}, {"dg_iflux_p" #P, "DR,MR,MR,MR,MI,MI"},        \
      {"dg_eflux_p" #P, "DR,MR,MR,MR,MI,MI"}, {"dg_minv_p" #P, "DR,DR,DW,DW"},         \
      {"dg_axpy_p" #P, "DW,DW,DR,DR"}
    LT_DG_SPEC(1), LT_DG_SPEC(2), LT_DG_SPEC(3), LT_DG_SPEC(4),
#undef LT_DG_SPEC
};
static const int kNumKernels = (int)(sizeof(kSpecs) / sizeof(kSpecs[0]));

static int sig_count(const char *sig) {
  int n = 1;
  for (const char *p = sig; *p; ++p) n += (*p == ',');
  return n;
}

// ---- access contexts ------------------------------------------------------------
struct TileCtx {
  static constexpr bool kRecGeo = true;  // records carry |f|/2 and the face
  const DLoop &L;
  int e, gpos, lpos;
  double *smem;
  __device__ int vpe(int d) const { return L.a[d].vpe; }
  __device__ int arity(int d) const { return L.a[d].arity; }
  __device__ const double *params() const { return L.params; }
  __device__ int elem() const { return e; }
  __device__ const double *rd(int d) const { return L.a[d].data + (size_t)e * L.a[d].vpe; }
  __device__ double *wr(int d) const { return L.a[d].data + (size_t)e * L.a[d].vpe; }
  __device__ int tgt(int d, int k) const {
    const DArg &A = L.a[d];
    return L.use_local ? A.lmap[(size_t)gpos * A.arity + k] : A.map[(size_t)e * A.arity + k];
  }
  __device__ const double *rdm(int d, int k) const {
    return L.a[d].data + (size_t)tgt(d, k) * L.a[d].vpe;
  }
  __device__ double *inc(int d, int k) const {
    const DArg &A = L.a[d];
    return smem + A.inc_off + (lpos * A.arity + k) * A.vpe;
  }
  __device__ double *rec(int k) const { return smem + (lpos * L.a[4].arity + k) * L.rec; }
};

struct FlatCtx {  // untiled: element ids, global scratch
  static constexpr bool kRecGeo = true;
  const DLoop &L;
  int e;
  __device__ int vpe(int d) const { return L.a[d].vpe; }
  __device__ int arity(int d) const { return L.a[d].arity; }
  __device__ const double *params() const { return L.params; }
  __device__ int elem() const { return e; }
  __device__ const double *rd(int d) const { return L.a[d].data + (size_t)e * L.a[d].vpe; }
  __device__ double *wr(int d) const { return L.a[d].data + (size_t)e * L.a[d].vpe; }
  __device__ int tgt(int d, int k) const { return L.a[d].map[(size_t)e * L.a[d].arity + k]; }
  __device__ const double *rdm(int d, int k) const {
    return L.a[d].data + (size_t)tgt(d, k) * L.a[d].vpe;
  }
  __device__ double *inc(int d, int k) const {
    const DArg &A = L.a[d];
    return A.scr + ((size_t)e * A.arity + k) * A.vpe;
  }
  __device__ double *rec(int k) const {
    return L.a[4].scr + ((size_t)e * L.a[4].arity + k) * L.rec;
  }
};

// staged: every dataset row the tile touches lives in shared memory; slots are
// footprint-local row indices produced by the plan.  A loop's descriptors are
// resolved once per loop (resolve_descs: first row, row stride, slot map,
// arity) into registers, so an item's row address is one shared-memory slot
// load and one multiply-add (was: three dependent shared loads and two
// constant-bank loads per descriptor access)
struct StagedDesc {
  double *row0;     // first row of the bound dataset in shared memory
  const int *slot;  // slot map of the descriptor in the tile program
  int stride;       // shared-memory row stride (doubles)
  int arity;
};

__device__ __forceinline__ void resolve_descs(const DLoop &L, const int *sb, double *smem,
                                              const int *base, const int *B, StagedDesc *D) {
#pragma unroll
  for (int d = 0; d < LT_MAX_DESC; ++d)
    if (d < L.n_desc) {
      D[d].row0 = smem + base[L.a[d].ds];
      D[d].slot = B + sb[d];
      D[d].stride = L.a[d].sstride;
      D[d].arity = L.a[d].arity;
    }
}

#ifndef LT_RESOLVE_MINB
// builds with <= this many CTAs/SM resolve descriptors per loop; off: measured
// 4.6 % slower at config 3 and 3.4 % at config 4 (168-register build) -- the
// shorter address chains do not pay for the registers they hold across items
#define LT_RESOLVE_MINB 0
#endif

// R: descriptors resolved per loop (wide builds: the registers are there); else
// every access walks the tile program (the 80-register builds, which would spill)
template <bool R>
struct StagedCtxT {
  static constexpr bool kRecGeo = false;  // |f|/2 and face read from the facet geometry row
  const DLoop &L;
  int e, pos, lpos;  // pos: position in the tile's list
  double *scratch;
  const StagedDesc *D;
  double *smem;
  const int *base;   // per staged dataset: first double of its rows in smem
  const int *B;      // tile program in smem
  const int *sbase;  // per descriptor: base of its slot map in B
  __device__ int vpe(int d) const { return L.a[d].vpe; }
  __device__ int arity(int d) const { return R ? D[d].arity : L.a[d].arity; }
  __device__ const double *params() const { return L.params; }
  __device__ int elem() const { return e; }
  __device__ double *row(int d, int slot) const {
    if constexpr (R) return D[d].row0 + slot * D[d].stride;
    else return smem + base[L.a[d].ds] + slot * L.a[d].sstride;
  }
  __device__ int slot_at(int d, int i) const {
    if constexpr (R) return D[d].slot[i];
    else return B[sbase[d] + i];
  }
  __device__ const double *rd(int d) const { return row(d, slot_at(d, pos)); }
  __device__ double *wr(int d) const { return row(d, slot_at(d, pos)); }
  __device__ const double *rdm(int d, int k) const {
    return row(d, slot_at(d, pos * arity(d) + k));
  }
  __device__ double *inc(int d, int k) const {
    const DArg &A = L.a[d];
    return scratch + A.inc_off + (lpos * A.arity + k) * A.vpe;
  }
  __device__ double *rec(int k) const { return scratch + (lpos * L.a[4].arity + k) * L.rec; }
};

// FAM selects which DG degree is compiled into an instantiation (0: scalar
// kernels only, 1..4: scalar + DG P, 5: everything) so a P1 chain does not
// pay the register footprint of P4 bodies.
template <int FAM, class C>
__device__ __forceinline__ void dispatch(int kernel, C &c, int lane) {
  switch (kernel) {
    case K_EDGE_INC: body_edge_inc(c); break;
    case K_CELL_INC: body_edge_inc(c); break;  // same body: every target += own value
    case K_EDGE_READ: body_sum_read(c); break;
    case K_CELL_READ: body_sum_read(c); break;
    case K_TOY_K1: body_toy_k1(c); break;
    case K_TOY_K2: body_toy_k2(c); break;
    case K_TOY_K3: body_toy_k3(c); break;
    default:
      if (FAM > 0) dg_dispatch<FAM>(kernel - K_DG_FIRST, c, lane);
      break;
  }
}

// Deferred apply of DG facet records for one (target, DoF row i): the target's
// ru/rs row values (du, ds: component i) plus every contributor's lifted record
// in (element, k) order.
template <int FAM>
__device__ __forceinline__ void lift_apply_item(const DLoop &L, double *du, double *ds, int nd,
                                                int i, const double *recs, const int *slots,
                                                int s0, int s1) {
  double acc[5] = {du[0], du[nd], ds[0], ds[nd], ds[2 * nd]};
  for (int s = s0; s < s1; ++s)
    dg_lift_acc<FAM>(L.kernel - K_DG_FIRST, L.params, i, recs + (size_t)slots[s] * L.rec, acc);
  du[0] = acc[0];
  du[nd] = acc[1];
  ds[0] = acc[2];
  ds[nd] = acc[3];
  ds[2 * nd] = acc[4];
}

// Work items (element, lane) of cnt elements with `lanes` items each, strided
// over `step` threads, stepped incrementally (no division per item).
template <class F>
__device__ __forceinline__ void for_items(int cnt, int lanes, int step, F &&f) {
  const int dq = step / lanes, dr = step - dq * lanes;
  int e = threadIdx.x / lanes, l = threadIdx.x - e * lanes;
  while (e < cnt) {
    f(e, l);
    e += dq;
    l += dr;
    if (l >= lanes) { l -= lanes; ++e; }
  }
}

// same over LT_SBLOCK threads with the loop's precomputed stepping constants
template <class F>
__device__ __forceinline__ void for_items_s(int cnt, const DLoop &L, F &&f) {
  const int lanes = L.lanes;
  int e = lt_div(threadIdx.x, lanes, L.lane_magic), l = threadIdx.x - e * lanes;
  while (e < cnt) {
    f(e, l);
    e += L.lane_dq;
    l += L.lane_dr;
    if (l >= lanes) { l -= lanes; ++e; }
  }
}

// (element, group) items of cnt elements x groups, element index fastest across
// lanes (adjacent lanes: adjacent list positions, distinct shared-memory rows)
template <class F>
__device__ __forceinline__ void for_flat(int cnt, int groups, F &&f) {
  const int total = cnt * groups;
  for (int x = threadIdx.x; x < total; x += LT_SBLOCK) {
    const int g = groups == 1 ? 0 : x / cnt;
    f(x - g * cnt, g);
  }
}

#ifndef LT_APPLY_BATCH
// > 1: a deferred-apply item resolves the slot -> facet -> geometry chains of
// that many contributors before lifting them (independent loads in flight).
// Measured slower (3: config 4 cut 40.78 -> 41.36 ms, config 3 12.17 -> 12.34 ms:
// the extra live registers cost more than the overlapped loads save); off
#define LT_APPLY_BATCH 1
#endif

#ifndef LT_TMA_GATHER
// 1: compile the TMA tile::gather4 footprint gathers (UTMALDG; then opt-in at run
// time with LT_TMA=1).  Off by default: measured 7 % slower than the cp.async
// gathers when used, and its scaffolding (run-time aligned shared-memory base,
// second mbarrier, tensor maps in the kernel parameters) cost 13-23 % even when
// unused (config 2: 0.552 -> 0.677 ms; config 4 cut ts 12: 47.9 -> 54.3 ms)
#define LT_TMA_GATHER 0
#endif

#ifndef LT_GROUPED
// DG loops of the shared-memory tile executors as grouped items (lt_dg.cuh), per
// phase: 1 volume, 2 facet records, 4 deferred apply, 8 inverse mass / update.
// Measured (B200, dataflow executor, round 2): the tile phases are latency-bound
// with one to three rounds of items per thread, so the fine items (one DoF row /
// one facet point per lane) win for the contractions -- grouped volume, records
// and apply items are 40-70 % slower per phase at P3 despite 3x fewer shared
// loads -- while the per-field inverse-mass/update items are 20 % faster
// (conflict-free 16-byte rows).  At the bench configurations (block layout, 3-4
// CTAs/SM) grouped volume items gain 2.6 % at P2 (mask 9: 10.78 -> 10.50 ms) and
// grouped apply items 0.9 % at P3 (mask 12: 39.46 -> 39.10 ms on the config 4
// cut); profiles/r02_ab_masks_final_config.txt.
// (evaluated inside run_tile<FAM, ...>)
#define LT_GROUPED (FAM == 2 ? 9 : FAM == 3 ? 12 : 8)
#endif

// ---- fused tiled executor ------------------------------------------------------
__device__ __forceinline__ void apply_chunk(const DLoop &L, const IncPlan &P, int gc,
                                            const double *smem) {
  const DArg &A = L.a[P.desc];
  const int vpe = A.vpe;
  const int u0 = P.gc_off[gc], u1 = P.gc_off[gc + 1];
  const int work = (u1 - u0) * vpe;
  for (int w = threadIdx.x; w < work; w += blockDim.x) {
    const int u = u0 + w / vpe, c = w - (w / vpe) * vpe;
    double *dst = A.data + (size_t)P.utgt[u] * vpe + c;
    const int s0 = P.ut_off[u], s1 = P.ut_off[u + 1];
    if (A.mode == LT_INC) {
      double v = *dst;
      for (int s = s0; s < s1; ++s) v = __dadd_rn(v, smem[A.inc_off + P.slots[s] * vpe + c]);
      *dst = v;
    } else {  // mapped WRITE: last writer in sequential order wins
      *dst = smem[A.inc_off + P.slots[s1 - 1] * vpe + c];
    }
  }
}

template <int FAM>
__global__ void __launch_bounds__(LT_BLOCK) k_fused_tiles(const DLoop *__restrict__ loops,
                                                          int n_loops,
                                                          const int32_t *__restrict__ tile_ids) {
  extern __shared__ double smem[];
  const int t = tile_ids[blockIdx.x];
  for (int j = 0; j < n_loops; ++j) {
    const DLoop &L = loops[j];
    const int beg = L.offsets[t];
    const int n = L.offsets[t + 1] - beg;
    if (n == 0) continue;
    const int CH = L.chunk;
    for (int c0 = 0; c0 < n; c0 += CH) {
      for_items(min(CH, n - c0), L.lanes, blockDim.x, [&](int lp, int lane) {
        const int gpos = beg + c0 + lp;
        TileCtx cx{L, L.elements[gpos], gpos, lp, smem};
        dispatch<FAM>(L.kernel, cx, lane);
      });
      if (L.n_inc) {
        __syncthreads();
        const int gc = L.chunk_base[t] + c0 / CH;
        if (L.deferred) {
          const IncPlan &P = L.inc[0];
          const int nd = L.a[4].vpe >> 1, u0 = P.gc_off[gc];
          const int work = (P.gc_off[gc + 1] - u0) * nd;
          for (int w = threadIdx.x; w < work; w += blockDim.x) {
            const int u = u0 + w / nd, i = w - (w / nd) * nd;
            lift_apply_item<FAM>(L, L.a[4].data + (size_t)P.utgt[u] * L.a[4].vpe + i,
                                 L.a[5].data + (size_t)P.utgt[u] * L.a[5].vpe + i, nd, i, smem,
                                 P.slots, P.ut_off[u], P.ut_off[u + 1]);
          }
        } else {
          for (int i = 0; i < L.n_inc; ++i) apply_chunk(L, L.inc[i], gc, smem);
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

// ---- staged tiled executor ------------------------------------------------------------
// One CTA per tile: gather the tile footprint of every bound dataset into
// shared memory (coalesced along the ascending footprint rows), run the whole
// chain on it, store back the rows the tile wrote.  Global traffic per tile is
// one read of its footprint and one write of its outputs, independent of the
// chain length; the loops themselves only see shared-memory latency.
__device__ __forceinline__ void apply_chunk_staged(const DLoop &L, const IncPlan &P, int gc,
                                                   const double *scratch, double *smem,
                                                   const int *base) {
  const DArg &A = L.a[P.desc];
  const int vpe = A.vpe;
  double *rows = smem + base[A.ds];
  const int u0 = P.gc_off[gc], u1 = P.gc_off[gc + 1];
  const int work = (u1 - u0) * vpe;
  for (int w = threadIdx.x; w < work; w += blockDim.x) {
    const int u = u0 + w / vpe, c = w - (w / vpe) * vpe;
    double *dst = rows + P.utgt[u] * vpe + c;
    const int s0 = P.ut_off[u], s1 = P.ut_off[u + 1];
    if (A.mode == LT_INC) {
      double v = *dst;
      for (int s = s0; s < s1; ++s) v = __dadd_rn(v, scratch[A.inc_off + P.slots[s] * vpe + c]);
      *dst = v;
    } else {
      *dst = scratch[A.inc_off + P.slots[s1 - 1] * vpe + c];
    }
  }
}

__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem_dst, const void *gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

#ifdef LT_PHASE_TIMING
// profiling build only: per-phase cycle totals of the staged executor (thread 0)
__device__ unsigned long long g_phase_cycles[64];
#define LT_TSTAMP(var) long long var = clock64()
#define LT_TACC(slot, t0)                                                  \
  do {                                                                     \
    if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[slot], clock64() - (t0)); \
  } while (0)
#else
#define LT_TSTAMP(var)
#define LT_TACC(slot, t0)
#endif

// Kernel parameters of the staged executor: lives in the constant bank, so the
// per-loop descriptor fields every thread reads are uniform broadcasts.
//
// Tile program: every executable tile owns a contiguous, 16-byte aligned int32
// blob in HBM holding everything the tile needs besides the dataset rows:
//   header   [per space: fp count, fp base]
//            [per loop: list length, chunk count, slot base per descriptor,
//                       (gc, ut, uo, sl) bases per apply plan]
//            [per staged dataset: written-flag base or -1]
//   sections footprint element ids per space, slot maps per (loop, descriptor),
//            ordered-gather plans per (loop, map), written flags per dataset.
// One cp.async.bulk (TMA 1-D bulk copy) brings the blob into shared memory;
// after it every index the tile touches is a shared-memory access.
struct StagedParams {
  int32_t n_loops, n_ds, n_sp, hs;   // hs: header ints
  int32_t loop_pos[LT_MAX_SLOOPS];   // header position of each loop's block
  int32_t ds_pos;                    // header position of the written-row lists
  int32_t prog_pos;                  // header position of the program length (ints)
  int32_t ro_packed;                 // rows of read-only datasets follow the program in the blob
  int32_t dep_pos;                   // header position of the dependency list (dataflow)
  int32_t ld_pos;                    // header position of the per-dataset load lists
  int32_t base_pos;                  // header position of the per-dataset row bases
  int32_t n_gather, n_store;         // datasets gathered after the dependency wait / stored back
#if LT_TMA_GATHER
  int32_t n_tma;                     // datasets gathered by TMA gather4 (0: none)
#endif
  int8_t gather_ds[LT_MAX_STAGED];   // their indices (no per-dataset flag tests in the tile)
  int8_t store_ds[LT_MAX_STAGED];
  int32_t pad;
  const int32_t *blob;
  const int64_t *blob_off;           // per tile: first int of its blob
  const int32_t *blob_len;           // per tile: ints (multiple of 4)
  StageDS ds[LT_MAX_STAGED];
  DLoop loops[LT_MAX_SLOOPS];
#if LT_TMA_GATHER
  CUtensorMap tmap[LT_MAX_STAGED];   // per TMA-gathered dataset: [rows x vpe] f64, box vpe x 1
#endif
};

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes,
                                          uint64_t *bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// mbar_wait for the TMA gathers: a transaction that never completes (a byte
// count that does not match what the copies deliver) traps after ~2^26
// suspended polls (seconds) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait_guarded(uint64_t *bar, unsigned phase) {
  for (unsigned spins = 0;; ++spins) {
    unsigned done;
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (done) return;
    if (spins > (1u << 26)) __trap();
  }
}

// the dynamic shared memory of the staged kernels starts 128-byte aligned
// (TMA destinations); plans reserve the 112 bytes this may skip
__device__ __forceinline__ double *lt_align128(double *p) {
#if LT_TMA_GATHER
  return reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(p) + 127) & ~uintptr_t(127));
#else
  return p;  // compile-time shared-memory base: addresses fold into the instructions
#endif
}

#if LT_TMA_GATHER
// TMA gather: four rows (global ids r0..r3) of a [rows x vpe] float64 tensor
// into four consecutive shared-memory rows at dst (UTMALDG gather4 in SASS).
__device__ __forceinline__ void tma_gather4(double *dst, const CUtensorMap *map, int r0, int r1,
                                            int r2, int r3, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

// Full-footprint gathers of the TMA datasets in `list` by warp 0: one
// expect_tx for all their bytes, then each lane issues gather4s for every 32nd
// group of four footprint rows (a short tail repeats the last row id: the
// footprint is padded to four rows).  Every thread later waits on `gbar`.
__device__ __forceinline__ void tma_gather_list(const StagedParams &P, const int8_t *list, int n,
                                                const int *B, double *smem, const int *base,
                                                uint64_t *gbar) {
  if (threadIdx.x >= 32) return;
  unsigned bytes = 0;
  for (int q = 0; q < n; ++q) {
    const StageDS &S = P.ds[list[q]];
    // a gather4 writes (and counts) four full boxes: stride doubles per row
    if (S.tma && S.load == 1) bytes += (unsigned)((B[2 * S.sp] + 3) & ~3) * S.stride * 8u;
  }
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic smem use
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(gbar)),
                 "r"(bytes)
                 : "memory");
  }
  __syncwarp();
  for (int q = 0; q < n; ++q) {
    const int d = list[q];
    const StageDS &S = P.ds[d];
    if (!(S.tma && S.load == 1)) continue;
    const int nrow = B[2 * S.sp];
    const int *idx = B + B[2 * S.sp + 1];
    double *rows = smem + base[d];
    for (int g = threadIdx.x * 4; g < nrow; g += 128) {
      const int last = nrow - 1;
      tma_gather4(rows + g * S.stride, &P.tmap[d], idx[g], idx[min(g + 1, last)],
                  idx[min(g + 2, last)], idx[min(g + 3, last)], gbar);
    }
  }
}

#endif  // LT_TMA_GATHER

// Apply the contributions of one chunk for every INC/WRITE descriptor that
// shares ordered-gather plan `p` (e.g. ru and rs through if2c): one thread per
// unique target, contributions added in (element, k) order.
__device__ __forceinline__ void apply_item(const DLoop &L, int desc, int cc, int u,
                                           const int *utgt, const int *ut_off, const int *slots,
                                           const double *scratch, double *smem, const int *base) {
  const DArg &A = L.a[desc];
  const int vpe = A.vpe;
  const int s0 = ut_off[u], s1 = ut_off[u + 1];
  double *dst = smem + base[A.ds] + utgt[u] * A.sstride + cc;
  const double *sc = scratch + A.inc_off + cc;
  if (A.mode == LT_INC) {
    double v = *dst;
    for (int s = s0; s < s1; ++s) v = __dadd_rn(v, sc[slots[s] * vpe]);
    *dst = v;
  } else {
    *dst = sc[slots[s1 - 1] * vpe];
  }
}

__device__ __forceinline__ void apply_plan(const DLoop &L, int p, const int *gc_off,
                                           const int *utgt, const int *ut_off, const int *slots,
                                           int c, const double *scratch, double *smem,
                                           const int *base) {
  // descriptors sharing plan p (<= LT_MAX_INC = 4) and their offsets in the
  // concatenated component space, kept in scalars (no local memory)
  int d0 = -1, d1 = -1, d2 = -1, d3 = -1, c1 = 0, c2 = 0, c3 = 0, vt = 0;
#pragma unroll
  for (int i = 0; i < LT_MAX_INC; ++i) {
    if (i >= L.n_inc || L.inc[i].plan != p) continue;
    const int d = L.inc[i].desc;
    if (d0 < 0) { d0 = d; vt += L.a[d].vpe; c1 = vt; }
    else if (d1 < 0) { d1 = d; vt += L.a[d].vpe; c2 = vt; }
    else if (d2 < 0) { d2 = d; vt += L.a[d].vpe; c3 = vt; }
    else { d3 = d; vt += L.a[d].vpe; }
  }
  if (d1 < 0) c1 = c2 = c3 = vt;
  else if (d2 < 0) c2 = c3 = vt;
  else if (d3 < 0) c3 = vt;
  const int u0 = gc_off[c], nu = gc_off[c + 1] - u0;
  // one work item per (target, component), walked incrementally (no division)
  const int dq = LT_SBLOCK / vt, dr = LT_SBLOCK - dq * vt;
  int q = threadIdx.x / vt, r = threadIdx.x - q * vt;
  while (q < nu) {
    const int desc = r < c1 ? d0 : r < c2 ? d1 : r < c3 ? d2 : d3;
    const int cc = r - (r < c1 ? 0 : r < c2 ? c1 : r < c3 ? c2 : c3);
    apply_item(L, desc, cc, u0 + q, utgt, ut_off, slots, scratch, smem, base);
    q += dq;
    r += dr;
    if (r >= vt) { r -= vt; ++q; }
  }
}

// Gather the footprint rows of dataset d into its shared rows with
// asynchronous copies.  Each thread owns one component (or 16-byte pair) c and
// a row offset r0 < S.di = LT_SBLOCK / unit, and walks rows r0, r0 + di, ...:
// consecutive threads copy consecutive components of a row (coalesced within
// rows and along runs of consecutive ids), and the loop carries no division
// or component wrap-around (4-5 instructions per copy).
// no "memory" clobber: the index loads may move across the copies (the rows
// they fill are read only after cp_async_wait_all + a barrier)
template <int BYTES>
__device__ __forceinline__ void cp_async_nc(double *smem_dst, const double *gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  if (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src));
}

template <int BYTES>
__device__ __forceinline__ void gather_loop(const double *__restrict__ src, double *dst,
                                            const int *__restrict__ idx, int i, int n, int rpp,
                                            int step, uint32_t v, uint32_t c) {
  // four rows per trip: their index loads are independent and overlap
  for (; i + 3 * rpp < n; i += 4 * rpp, dst += 4 * step) {
    const uint32_t g0 = (uint32_t)idx[i], g1 = (uint32_t)idx[i + rpp];
    const uint32_t g2 = (uint32_t)idx[i + 2 * rpp], g3 = (uint32_t)idx[i + 3 * rpp];
    cp_async_nc<BYTES>(dst, src + (g0 * v + c));
    cp_async_nc<BYTES>(dst + step, src + (g1 * v + c));
    cp_async_nc<BYTES>(dst + 2 * step, src + (g2 * v + c));
    cp_async_nc<BYTES>(dst + 3 * step, src + (g3 * v + c));
  }
  for (; i < n; i += rpp, dst += step) cp_async_nc<BYTES>(dst, src + ((uint32_t)idx[i] * v + c));
}

__device__ __forceinline__ void gather_rows(const StageDS &S, const int *B, double *rows) {
  const uint32_t v = (uint32_t)S.vpe;
  const int rpp = S.di;
  const int nrow = B[2 * S.sp];
  const int *idx = B + B[2 * S.sp + 1];
  const int unit = S.vec ? (int)v >> 1 : (int)v;
  const int r0 = lt_div(threadIdx.x, unit, S.magic);
  if (r0 >= rpp) return;
  const uint32_t c = (uint32_t)(threadIdx.x - r0 * unit) << S.vec;  // thread's first double
  double *dst = rows + r0 * S.stride + c;
  const int step = rpp * S.stride;
  if (S.vec)  // 16-byte pairs: even rows, 16-byte aligned in HBM and shared memory
    gather_loop<16>(S.data, dst, idx, r0, nrow, rpp, step, v, c);
  else
    gather_loop<8>(S.data, dst, idx, r0, nrow, rpp, step, v, c);
}

// Gather only the listed footprint rows (load == 2: rows the first writer of
// the dataset does not overwrite), same thread mapping.
__device__ __forceinline__ void gather_rows_listed(const StageDS &S, const int *B, const int *ll,
                                                   int nl, double *rows) {
  const uint32_t v = (uint32_t)S.vpe;
  const int rpp = S.di;
  const int *idx = B + B[2 * S.sp + 1];
  const int unit = S.vec ? (int)v >> 1 : (int)v;
  const int r0 = lt_div(threadIdx.x, unit, S.magic);
  if (r0 >= rpp) return;
  const uint32_t c = (uint32_t)(threadIdx.x - r0 * unit) << S.vec;
  double *dst = rows + c;
  int i = r0;
  for (; i + rpp < nl; i += 2 * rpp) {  // two rows per trip: list and index loads overlap
    const int ra = ll[i], rb = ll[i + rpp];
    const uint32_t ga = (uint32_t)idx[ra], gb = (uint32_t)idx[rb];
    if (S.vec) {
      cp_async_nc<16>(dst + ra * S.stride, S.data + (ga * v + c));
      cp_async_nc<16>(dst + rb * S.stride, S.data + (gb * v + c));
    } else {
      cp_async_nc<8>(dst + ra * S.stride, S.data + (ga * v + c));
      cp_async_nc<8>(dst + rb * S.stride, S.data + (gb * v + c));
    }
  }
  for (; i < nl; i += rpp) {
    const int r = ll[i];
    if (S.vec)
      cp_async_nc<16>(dst + r * S.stride, S.data + ((uint32_t)idx[r] * v + c));
    else
      cp_async_nc<8>(dst + r * S.stride, S.data + ((uint32_t)idx[r] * v + c));
  }
}

// Store back the rows of dataset S the tile wrote (compact list wl of
// footprint positions), same thread mapping as the gather.  SB = 2: two rows
// per trip with both rows' shared-memory loads issued before the global
// stores, so the wl -> idx -> row load chains overlap.
template <int SB, class T>
__device__ __forceinline__ void store_rows_t(double *__restrict__ dst,
                                            const double *__restrict__ src,
                                            const int *__restrict__ idx,
                                            const int *__restrict__ wl, int nw, int r0, int rpp,
                                            uint32_t v, int sv) {
  int i = r0;
  if (SB >= 2)
    for (; i + rpp < nw; i += 2 * rpp) {  // two rows per trip, loads before stores
      const int ra = wl[i], rb = wl[i + rpp];
      const uint32_t ga = (uint32_t)idx[ra] * v, gb = (uint32_t)idx[rb] * v;
      const T xa = *reinterpret_cast<const T *>(src + ra * sv);
      const T xb = *reinterpret_cast<const T *>(src + rb * sv);
      *reinterpret_cast<T *>(dst + ga) = xa;
      *reinterpret_cast<T *>(dst + gb) = xb;
    }
  for (; i < nw; i += rpp) {
    const int r = wl[i];
    *reinterpret_cast<T *>(dst + (uint32_t)idx[r] * v) = *reinterpret_cast<const T *>(src + r * sv);
  }
}

template <int SB>
__device__ __forceinline__ void store_rows(const StageDS &S, const int *idx, const int *wl, int nw,
                                          const double *rows) {
  const uint32_t v = (uint32_t)S.vpe;
  const int rpp = S.di;
  const int unit = S.vec ? (int)v >> 1 : (int)v;
  const int r0 = lt_div(threadIdx.x, unit, S.magic);
  if (r0 >= rpp) return;
  const uint32_t c = (uint32_t)(threadIdx.x - r0 * unit) << S.vec;
  if (S.vec)
    store_rows_t<SB, double2>(S.data + c, rows + c, idx, wl, nw, r0, rpp, v, S.stride);
  else
    store_rows_t<SB, double>(S.data + c, rows + c, idx, wl, nw, r0, rpp, v, S.stride);
}

// Phase 1 of a tile (no dependency on other tiles): tile program via TMA,
// shared-memory layout, and the gather of datasets the chain never writes.
__device__ __forceinline__ void tile_program_issue(const StagedParams &P, int t, double *smem,
                                                   uint64_t *bar) {  // one thread
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of smem
  bulk_load(smem, P.blob + P.blob_off[t], 4u * (unsigned)P.blob_len[t], bar);
}

// After the program arrived: the per-dataset row bases are in its header
// (host-computed, base_pos), so no thread computes them and no barrier is
// needed -- every thread waits on the program's mbarrier itself.
__device__ __forceinline__ const int *tile_prefetch(const StagedParams &P, int t, double *smem,
                                                    uint64_t *bar, unsigned phase,
                                                    bool issued = false) {
  int *B = reinterpret_cast<int *>(smem);
  LT_TSTAMP(t_blob);
  if (threadIdx.x == 0 && !issued) tile_program_issue(P, t, smem, bar);
  mbar_wait(bar, phase);
  LT_TACC(0, t_blob);
  const int *base = B + P.base_pos;
  if (!P.ro_packed) {
    for (int d = 0; d < P.n_ds; ++d)
      if (P.ds[d].ro) gather_rows(P.ds[d], B, smem + base[d]);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  return base;
}

// Deferred apply of a DG facet loop's chunk: one work item per (unique target,
// DoF row); each contributor's correction record is lifted and added in
// (element, k) order -- the reference's sequential order -- straight into the
// target's ru/rs rows in shared memory.
template <int FAM>
__device__ __forceinline__ void apply_deferred(const DLoop &L, const int *gc_off, const int *utgt,
                                               const int *ut_off, const int *slots, int c,
                                               const double *scratch, double *smem,
                                               const int *base, const int *fslot) {
  if (FAM == 0) return;
  const DArg &Au = L.a[4], &As = L.a[5], &Ag = L.a[0];
  const int nd = Au.vpe >> 1;
  const bool two = Au.arity == 2;
  double *ru = smem + base[Au.ds], *rs = smem + base[As.ds];
  const double *geo = smem + base[Ag.ds];
  const int u0 = gc_off[c], nu = gc_off[c + 1] - u0;
  int q = lt_div(threadIdx.x, nd, L.row_magic), i = threadIdx.x - q * nd;
  while (q < nu) {
    const int u = u0 + q;
    double *du = ru + utgt[u] * Au.sstride + i, *ds = rs + utgt[u] * As.sstride + i;
    double acc[5] = {du[0], du[nd], ds[0], ds[nd], ds[2 * nd]};
#if LT_APPLY_BATCH > 1
    // contributors in batches: the slot -> facet slot -> geometry row -> (|f|/2,
    // face) chains of a batch are independent loads issued together (a cell has
    // three facets: one batch), the lifts then add in (element, k) order
    for (int s = ut_off[u], s1 = ut_off[u + 1]; s < s1; s += LT_APPLY_BATCH) {
      int sl[LT_APPLY_BATCH], face[LT_APPLY_BATCH];
      double jf[LT_APPLY_BATCH];
#pragma unroll
      for (int b = 0; b < LT_APPLY_BATCH; ++b) sl[b] = slots[min(s + b, s1 - 1)];
#pragma unroll
      for (int b = 0; b < LT_APPLY_BATCH; ++b) {
        const int lp = two ? sl[b] >> 1 : sl[b], k = two ? sl[b] & 1 : 0;
        const double *g = geo + fslot[lp] * Ag.sstride;  // facet geometry [nx ny |f|/2 fa fb]
        jf[b] = g[2];
        face[b] = (int)g[3 + k];
      }
#pragma unroll
      for (int b = 0; b < LT_APPLY_BATCH; ++b)
        if (s + b < s1)
          dg_lift_acc_g<FAM>(L.kernel - K_DG_FIRST, L.params, i, scratch + (size_t)sl[b] * L.rec,
                             jf[b], face[b], acc);
    }
#else
    for (int s = ut_off[u], s1 = ut_off[u + 1]; s < s1; ++s) {
      const int sl = slots[s], lp = two ? sl >> 1 : sl, k = two ? sl & 1 : 0;
      const double *g = geo + fslot[lp] * Ag.sstride;  // facet geometry [nx ny |f|/2 fa fb]
      dg_lift_acc_g<FAM>(L.kernel - K_DG_FIRST, L.params, i, scratch + (size_t)sl * L.rec, g[2],
                         (int)g[3 + k], acc);
    }
#endif
    du[0] = acc[0];
    du[nd] = acc[1];
    ds[0] = acc[2];
    ds[nd] = acc[3];
    ds[2 * nd] = acc[4];
    q += L.row_dq;
    i += L.row_dr;
    if (i >= nd) { i -= nd; ++q; }
  }
}

// Grouped form: one work item per (unique target, group of RA DoF rows), the
// target index fastest across lanes; every contributor's record is read once
// for the item's rows.  Same (element, k) order per target row.
template <int P>
__device__ __forceinline__ void apply_deferred_g(const DLoop &L, const int *gc_off,
                                                 const int *utgt, const int *ut_off,
                                                 const int *slots, int c, const double *scratch,
                                                 double *smem, const int *base,
                                                 const int *fslot) {
  constexpr int ND = DGShape<P>::ND, RV = DGGroup<P>::RA, GV = DGGroup<P>::GA;
  const DArg &Au = L.a[4], &As = L.a[5], &Ag = L.a[0];
  const bool two = Au.arity == 2;
  double *ru = smem + base[Au.ds], *rs = smem + base[As.ds];
  const double *geo = smem + base[Ag.ds];
  const int u0 = gc_off[c], nu = gc_off[c + 1] - u0;
  for_flat(nu, GV, [&](int q, int g) {
    const int u = u0 + q, i0 = g * RV;
    double *du = ru + utgt[u] * Au.sstride, *ds = rs + utgt[u] * As.sstride;
    double acc[RV][5];
#pragma unroll
    for (int r = 0; r < RV; ++r) {
      const int i = min(i0 + r, ND - 1);
      acc[r][0] = du[i];
      acc[r][1] = du[ND + i];
      acc[r][2] = ds[i];
      acc[r][3] = ds[ND + i];
      acc[r][4] = ds[2 * ND + i];
    }
#if LT_APPLY_BATCH > 1
    for (int s = ut_off[u], s1 = ut_off[u + 1]; s < s1; s += LT_APPLY_BATCH) {
      int sl[LT_APPLY_BATCH], face[LT_APPLY_BATCH];
      double jf[LT_APPLY_BATCH];
#pragma unroll
      for (int b = 0; b < LT_APPLY_BATCH; ++b) sl[b] = slots[min(s + b, s1 - 1)];
#pragma unroll
      for (int b = 0; b < LT_APPLY_BATCH; ++b) {
        const int lp = two ? sl[b] >> 1 : sl[b], k = two ? sl[b] & 1 : 0;
        const double *gf = geo + fslot[lp] * Ag.sstride;  // facet geometry [nx ny |f|/2 fa fb]
        jf[b] = gf[2];
        face[b] = (int)gf[3 + k];
      }
#pragma unroll
      for (int b = 0; b < LT_APPLY_BATCH; ++b)
        if (s + b < s1)
          dg_lift_rows_g<P>(L.params, face[b], i0, jf[b], scratch + (size_t)sl[b] * L.rec, acc);
    }
#else
    for (int s = ut_off[u], s1 = ut_off[u + 1]; s < s1; ++s) {
      const int sl = slots[s], lp = two ? sl >> 1 : sl, k = two ? sl & 1 : 0;
      const double *gf = geo + fslot[lp] * Ag.sstride;  // facet geometry [nx ny |f|/2 fa fb]
      dg_lift_rows_g<P>(L.params, (int)gf[3 + k], i0, gf[2], scratch + (size_t)sl * L.rec, acc);
    }
#endif
#pragma unroll
    for (int r = 0; r < RV; ++r) {
      const int i = i0 + r;
      if (i < ND) {
        du[i] = acc[r][0];
        du[ND + i] = acc[r][1];
        ds[i] = acc[r][2];
        ds[ND + i] = acc[r][3];
        ds[2 * ND + i] = acc[r][4];
      }
    }
  });
}

// Phase 2: gather the datasets the chain writes, run every loop on shared
// memory, store back the rows this tile wrote.
template <int FAM, int SB = 1, bool RES = false>
__device__ __forceinline__ void run_tile(const StagedParams &P, int t, double *smem,
                                         const int *base, uint64_t *gbar, unsigned &gphase) {
  const int *B = reinterpret_cast<const int *>(smem);
  LT_TSTAMP(t_gather);
#if LT_TMA_GATHER
  if (P.n_tma) tma_gather_list(P, P.gather_ds, P.n_gather, B, smem, base, gbar);
#endif
  for (int q = 0; q < P.n_gather; ++q) {
    const int d = P.gather_ds[q];
    const StageDS &S = P.ds[d];
    if (S.load == 2)
      gather_rows_listed(S, B, B + B[P.ld_pos + 2 * d + 1], B[P.ld_pos + 2 * d], smem + base[d]);
    else if (!S.tma)
      gather_rows(S, B, smem + base[d]);
  }
  cp_async_wait_all();
#if LT_TMA_GATHER
  if (P.n_tma) {
    mbar_wait_guarded(gbar, gphase);
    gphase ^= 1u;
  }
#endif
  __syncthreads();
  LT_TACC(1, t_gather);
  double *scratch = smem + base[P.n_ds];
  for (int j = 0; j < P.n_loops; ++j) {
    const DLoop &L = P.loops[j];
    const int *LH = B + P.loop_pos[j];
    const int n = LH[0];
    if (n == 0) continue;
    LT_TSTAMP(t_loop);
    StagedDesc Dd[LT_MAX_DESC];
    if constexpr (RES) resolve_descs(L, LH + 2, smem, base, B, Dd);
    if (L.deferred) {  // DG facet loop: records, then lifted ordered apply
      const int CH = LH[1];  // per-tile chunk (tile program header)
      const int *pb = LH + 2 + L.n_desc;
      for (int c0 = 0, ci = 0; c0 < n; c0 += CH, ++ci) {
        LT_TSTAMP(t_rec);
        if (FAM >= 1 && FAM <= 4) {  // kernel selected once per loop, not per item
          constexpr int PP = FAM >= 1 && FAM <= 4 ? FAM : 1;
          if (LT_GROUPED & 2) {
            if ((L.kernel - K_DG_FIRST) % 5 == 1)
              for_flat(min(CH, n - c0), DGGroup<PP>::GF, [&](int lp, int pg) {
                StagedCtxT<RES> cx{L, 0, c0 + lp, lp, scratch, Dd, smem, base, B, LH + 2};
                dg_iflux_g<PP>(cx, pg);
              });
            else
              for_flat(min(CH, n - c0), DGGroup<PP>::GF, [&](int lp, int pg) {
                StagedCtxT<RES> cx{L, 0, c0 + lp, lp, scratch, Dd, smem, base, B, LH + 2};
                dg_eflux_g<PP>(cx, pg);
              });
          } else if ((L.kernel - K_DG_FIRST) % 5 == 1)
            for_items_s(min(CH, n - c0), L, [&](int lp, int lane) {
              StagedCtxT<RES> cx{L, 0, c0 + lp, lp, scratch, Dd, smem, base, B, LH + 2};
              dg_iflux<PP>(cx, lane);
            });
          else
            for_items_s(min(CH, n - c0), L, [&](int lp, int lane) {
              StagedCtxT<RES> cx{L, 0, c0 + lp, lp, scratch, Dd, smem, base, B, LH + 2};
              dg_eflux<PP>(cx, lane);
            });
        } else {
          for_items_s(min(CH, n - c0), L, [&](int lp, int lane) {
            StagedCtxT<RES> cx{L, 0, c0 + lp, lp, scratch, Dd, smem, base, B, LH + 2};
            dispatch<FAM>(L.kernel, cx, lane);
          });
        }
        __syncthreads();
        LT_TACC(40 + (j < 23 ? j : 23), t_rec);
        // fslot: the chunk's facet-geometry slots (descriptor 0, direct)
        if constexpr ((LT_GROUPED & 4) && FAM >= 1 && FAM <= 4)
          apply_deferred_g<FAM>(L, B + pb[0], B + pb[1], B + pb[2], B + pb[3], ci, scratch, smem,
                                base, B + LH[2] + c0);
        else
          apply_deferred<FAM>(L, B + pb[0], B + pb[1], B + pb[2], B + pb[3], ci, scratch, smem,
                              base, B + LH[2] + c0);
        __syncthreads();
      }
      LT_TACC(8 + (j < 24 ? j : 23), t_loop);
      continue;
    }
    if (!L.n_inc) {  // direct / mapped-read loop: all items of the list at once
      const int which = (L.kernel - K_DG_FIRST) % 5;
      if (FAM >= 1 && FAM <= 4 && L.kernel >= K_DG_FIRST) {  // kernel selected once per loop
        constexpr int PP = FAM >= 1 && FAM <= 4 ? FAM : 1;
        if (which == 3 && L.nobar == 2 && (P.loops[j + 1].kernel - K_DG_FIRST) % 5 == 4) {
          // inverse mass and update over the same items, lane-local: one pass
          const DLoop &L2 = P.loops[j + 1];
          const int *LH2 = B + P.loop_pos[j + 1];
          StagedDesc Dd2[LT_MAX_DESC];
          if constexpr (RES) resolve_descs(L2, LH2 + 2, smem, base, B, Dd2);
          if (LT_GROUPED & 8)
            for_flat(n, 5, [&](int pos, int f) {
              StagedCtxT<RES> cx{L, 0, pos, 0, scratch, Dd, smem, base, B, LH + 2};
              dg_minv_g<PP>(cx, f);
              StagedCtxT<RES> cy{L2, 0, pos, 0, scratch, Dd2, smem, base, B, LH2 + 2};
              dg_axpy_g<PP>(cy, f);
            });
          else
            for_items_s(n, L, [&](int pos, int lane) {
              StagedCtxT<RES> cx{L, 0, pos, 0, scratch, Dd, smem, base, B, LH + 2};
              dg_minv<PP>(cx, lane);
              StagedCtxT<RES> cy{L2, 0, pos, 0, scratch, Dd2, smem, base, B, LH2 + 2};
              dg_axpy<PP>(cy, lane);
            });
          ++j;
          if (!L2.nobar || (j + 1 < P.n_loops && B[P.loop_pos[j + 1]] == 0)) __syncthreads();
          LT_TACC(8 + (j < 24 ? j : 23), t_loop);
          continue;
        }
        if (which == 0 && (LT_GROUPED & 16)) {
          // field lanes: 6 cells x 5 fields per warp, warp-uniform trip count
          // (every lane takes part in the shuffles)
          const int lane = threadIdx.x & 31, cw = lane / 5, f = lane - 5 * cw;
          constexpr int kCells = 6 * (LT_SBLOCK / 32);
          for (int c0 = 6 * (threadIdx.x >> 5); c0 - 6 * (int)(threadIdx.x >> 5) < n;
               c0 += kCells) {
            const bool valid = cw < 6 && c0 + cw < n;
            StagedCtxT<RES> cx{L, 0, valid ? c0 + cw : n - 1, 0, scratch, Dd, smem, base, B,
                               LH + 2};
            dg_vol_f<PP>(cx, f, lane - f, valid);
          }
        } else if (which == 0 && (LT_GROUPED & 1))
          for_flat(n, DGGroup<PP>::GV, [&](int pos, int g) {
            StagedCtxT<RES> cx{L, 0, pos, 0, scratch, Dd, smem, base, B, LH + 2};
            dg_vol_g<PP>(cx, g);
          });
        else if (which == 0)
          for_items_s(n, L, [&](int pos, int lane) {
            StagedCtxT<RES> cx{L, 0, pos, 0, scratch, Dd, smem, base, B, LH + 2};
            dg_vol<PP>(cx, lane);
          });
        else if (which == 3 && (LT_GROUPED & 8))
          for_flat(n, 5, [&](int pos, int f) {
            StagedCtxT<RES> cx{L, 0, pos, 0, scratch, Dd, smem, base, B, LH + 2};
            dg_minv_g<PP>(cx, f);
          });
        else if (which == 3)
          for_items_s(n, L, [&](int pos, int lane) {
            StagedCtxT<RES> cx{L, 0, pos, 0, scratch, Dd, smem, base, B, LH + 2};
            dg_minv<PP>(cx, lane);
          });
        else if (LT_GROUPED & 8)
          for_flat(n, 5, [&](int pos, int f) {
            StagedCtxT<RES> cx{L, 0, pos, 0, scratch, Dd, smem, base, B, LH + 2};
            dg_axpy_g<PP>(cx, f);
          });
        else
          for_items_s(n, L, [&](int pos, int lane) {
            StagedCtxT<RES> cx{L, 0, pos, 0, scratch, Dd, smem, base, B, LH + 2};
            dg_axpy<PP>(cx, lane);
          });
      } else {
        for_items_s(n, L, [&](int pos, int lane) {
          StagedCtxT<RES> cx{L, 0, pos, 0, scratch, Dd, smem, base, B, LH + 2};
          dispatch<FAM>(L.kernel, cx, lane);
        });
      }
      // no barrier when the next loop's first phase cannot conflict with this
      // one (plan: barrier_free_pair); an empty next loop needs the barrier
      if (!L.nobar || (j + 1 < P.n_loops && B[P.loop_pos[j + 1]] == 0)) __syncthreads();
      LT_TACC(8 + (j < 24 ? j : 23), t_loop);
      continue;
    }
    const int CH = L.chunk;
    for (int c0 = 0, ci = 0; c0 < n; c0 += CH, ++ci) {
      LT_TSTAMP(t_body);
      for_items_s(min(CH, n - c0), L, [&](int lp, int lane) {
        StagedCtxT<RES> cx{L, 0, c0 + lp, lp, scratch, Dd, smem, base, B, LH + 2};
        dispatch<FAM>(L.kernel, cx, lane);
      });
      LT_TACC(32 + (j < 4 ? j : 3), t_body);
      if (L.n_inc) {
        __syncthreads();
        LT_TACC(36 + (j < 2 ? j : 1), t_body);
        for (int pl = 0; pl < L.n_plans; ++pl) {
          const int *pb = LH + 2 + L.n_desc + 4 * pl;
          apply_plan(L, pl, B + pb[0], B + pb[1], B + pb[2], B + pb[3], ci, scratch, smem, base);
        }
      }
      __syncthreads();
    }
    LT_TACC(8 + (j < 24 ? j : 23), t_loop);
  }
  LT_TSTAMP(t_wb);
  // store back the rows this tile wrote (coalesced like the gather)
  for (int q = 0; q < P.n_store; ++q) {
    const int d = P.store_ds[q];
    const StageDS &S = P.ds[d];
    store_rows<SB>(S, B + B[2 * S.sp + 1], B + B[P.ds_pos + 2 * d + 1], B[P.ds_pos + 2 * d],
               smem + base[d]);
  }
  LT_TACC(2, t_wb);
}

// one colour phase per launch, one CTA per tile
template <int FAM>
__global__ void __launch_bounds__(LT_SBLOCK) k_staged_tiles(const __grid_constant__ StagedParams P,
                                                            const int32_t *__restrict__ tile_ids) {
  extern __shared__ __align__(16) double smem_raw[];
  double *smem = lt_align128(smem_raw);
  __shared__ __align__(8) uint64_t bar, gbar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    if (LT_TMA_GATHER) mbar_init(&gbar, 1);
  }
  __syncthreads();
  unsigned gphase = 0;
  const int *base = tile_prefetch(P, tile_ids[blockIdx.x], smem, &bar, 0);
  run_tile<FAM>(P, tile_ids[blockIdx.x], smem, base, &gbar, gphase);
}

// Pack the rows of the read-only datasets of every tile to be run behind its
// tile program, in the shared-memory layout tile_prefetch computes, so that
// the tile's single bulk copy brings them along.  Runs once per execution call
// (datasets may change between calls; they cannot change within one).
__global__ void __launch_bounds__(256) k_pack_ro(const __grid_constant__ StagedParams P,
                                                 const int32_t *__restrict__ order, int n) {
  for (int it = blockIdx.x; it < n; it += gridDim.x) {
    const int t = order[it];
    const int32_t *B = P.blob + P.blob_off[t];
    double *tile = reinterpret_cast<double *>(const_cast<int32_t *>(B));
    for (int d = 0; d < P.n_ds; ++d) {
      const StageDS &S = P.ds[d];
      if (!S.ro) continue;
      const int acc = B[P.base_pos + d];  // the layout tile_prefetch uses (header)
      const int v = S.vpe, nrow = B[2 * S.sp];
      const int32_t *idx = B + B[2 * S.sp + 1];
      double *rows = tile + acc;
      for (int w = threadIdx.x; w < nrow * v; w += blockDim.x) {
        const int r = w / v, c = w - r * v;
        rows[r * S.stride + c] = __ldg(S.data + ((uint32_t)idx[r] * (uint32_t)v + c));
      }
    }
  }
}

// Persistent dataflow executor: CTAs pop tile instances (repeat k, tile) from a
// queue ordered by (repeat, region, colour, id) and wait only for the
// overlapping tiles that precede them: an overlapping tile of lower colour must
// have finished this repeat, any other overlapping tile (and the tile itself)
// the previous repeat.  Waits only target earlier queue items, which are held
// by running CTAs, so the schedule cannot deadlock.  Replaces the grid-wide
// barrier between colour classes by point-to-point tile dependencies.
struct DataflowArgs {
  const int64_t *item_tk;  // per queue item: repeat << 32 | tile
  const int64_t *item_ol;  // per queue item: program ints to bulk-copy << 40 | program offset
  const int32_t *order;    // executable tiles in queue order
  int32_t *done;           // per tile: completed repeats
  int32_t *queue;          // next item
  int32_t n_exec;
  int32_t n_items;
};

#ifndef LT_POLL_NS
#define LT_POLL_NS 32  // back-off between polls of an unfinished dependency
#endif
__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// MINB: CTAs per SM the register budget is sized for (6: 80 registers -- at P1
// this beats 72 registers at 7 CTAs/SM, which spill, by 1.5 %; 3: 168
// registers for footprints whose shared memory allows at most 3 CTAs per SM --
// config 3, 0.7 % faster than 128 registers)
template <int FAM, int MINB>
__global__ void __launch_bounds__(LT_SBLOCK, MINB) k_dataflow(const __grid_constant__ StagedParams P,
                                                        const DataflowArgs D) {
  extern __shared__ __align__(16) double smem_raw[];
  double *smem = lt_align128(smem_raw);
  __shared__ __align__(8) uint64_t bar, gbar;
  __shared__ int item;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    if (LT_TMA_GATHER) mbar_init(&gbar, 1);
  }
  unsigned phase = 0, gphase = 0;
  // the next queue item is popped one tile ahead, hiding the atomic's latency;
  // a CTA still runs its items in queue order, so waits only target items
  // held by running CTAs and the schedule stays deadlock-free
  int next = threadIdx.x == 0 ? atomicAdd(D.queue, 1) : 0;
  int prev = -1;  // tile whose completion is still to be released
  // release: the barrier at the top of the loop orders every thread's
  // store-back before thread 0's cumulative gpu-scope release increment
  // (CUTLASS GenericBarrier's arrive); it is issued after the next tile
  // program's TMA so its latency overlaps that load
  auto release = [&](int tile) {
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(D.done + tile) : "memory");
  };
  for (;;) {
    if (threadIdx.x == 0) {
      item = next;
      next = atomicAdd(D.queue, 1);
    }
    __syncthreads();
    const int it = item;
    if (it >= D.n_items) {
      if (threadIdx.x == 0 && prev >= 0) release(prev);
      return;
    }
    // the item's tile and its program's offset/length are independent loads
    // (one global round trip before the program's bulk copy)
    const long long tk = D.item_tk[it];
    const int t = (int)(uint32_t)tk, k = (int)(tk >> 32);
    if (threadIdx.x == 0) {
      const long long ol = D.item_ol[it];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic smem reads
      bulk_load(smem, P.blob + (ol & ((1ll << 40) - 1)), 4u * (unsigned)(ol >> 40), &bar);
      if (prev >= 0) release(prev);
    }
    const int *base = tile_prefetch(P, t, smem, &bar, phase, true);  // overlaps the dep. wait
    phase ^= 1u;
    LT_TSTAMP(t_wait);
    // the tile's dependency list arrived with its program (one global round
    // trip per wait: the done counter).  ld.acquire.gpu also invalidates this
    // SM's L1 (CCTL.IVALL), so the gathers below cannot see stale lines of
    // rows other tiles wrote
    const int *Bt = reinterpret_cast<const int *>(smem);
    const int n_dep = Bt[P.dep_pos];
    const int *dep = Bt + Bt[P.dep_pos + 1];
    for (int i = threadIdx.x; i < n_dep; i += LT_SBLOCK) {
      const int e = dep[i];
      const int need = k + (e & 1);
      const int32_t *flag = D.done + (e >> 1);
      while (ld_acquire(flag) < need) __nanosleep(LT_POLL_NS);
    }
    __syncthreads();
    LT_TACC(3, t_wait);
    LT_TSTAMP(t_tile);
    run_tile<FAM, 2, (MINB <= LT_RESOLVE_MINB)>(P, t, smem, base, &gbar, gphase);
    prev = t;
    LT_TACC(4, t_tile);
#ifdef LT_PHASE_TIMING
    if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[5], 1ull);
#endif
  }
}

// ---- untiled executor --------------------------------------------------------------
template <int FAM>
__global__ void __launch_bounds__(256) k_untiled_body(const DLoop *__restrict__ Lp, int n) {
  const DLoop &L = *Lp;
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int e = (int)(w / L.lanes);
  if (e >= n) return;
  FlatCtx cx{L, e};
  dispatch<FAM>(L.kernel, cx, (int)(w - (int64_t)e * L.lanes));
}

// smallest instantiation covering every kernel of the chain
static int chain_family(const ChainView &cv) {
  int fam = 0;
  for (const LoopDesc &L : cv.loops) {
    if (L.kernel < K_DG_FIRST) continue;
    const int p = (L.kernel - K_DG_FIRST) / 5 + 1;
    fam = (fam == 0 || fam == p) ? p : 5;
  }
  return fam;
}

typedef void (*FusedFn)(const DLoop *, int, const int32_t *);
typedef void (*UntiledFn)(const DLoop *, int);
static FusedFn fused_fn(int fam) {
  switch (fam) {
    case 0: return k_fused_tiles<0>;
    case 1: return k_fused_tiles<1>;
    case 2: return k_fused_tiles<2>;
    case 3: return k_fused_tiles<3>;
    case 4: return k_fused_tiles<4>;
    default: return k_fused_tiles<5>;
  }
}
typedef void (*DeferredFn)(const DLoop *, const int32_t *, const int32_t *, int64_t, int);
static DeferredFn untiled_deferred_fn(int fam);
static UntiledFn untiled_fn(int fam) {
  switch (fam) {
    case 0: return k_untiled_body<0>;
    case 1: return k_untiled_body<1>;
    case 2: return k_untiled_body<2>;
    case 3: return k_untiled_body<3>;
    case 4: return k_untiled_body<4>;
    default: return k_untiled_body<5>;
  }
}

__global__ void k_untiled_apply(const DLoop *__restrict__ Lp, int d, const int32_t *inv_off,
                                const int32_t *inv_flat, int64_t n_target, int exec_size) {
  const DLoop &L = *Lp;
  const DArg &A = L.a[d];
  const int vpe = A.vpe;
  int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= n_target * vpe) return;
  const int64_t t = w / vpe;
  const int c = (int)(w - t * vpe);
  const int b = inv_off[t], e = inv_off[t + 1];
  double *dst = A.data + (size_t)t * vpe + c;
  if (A.mode == LT_INC) {
    double v = *dst;
    for (int i = b; i < e; ++i) {
      const int f = inv_flat[i];
      if (f / A.arity >= exec_size) break;  // ascending: the rest are non-exec too
      v = __dadd_rn(v, A.scr[(size_t)f * vpe + c]);
    }
    *dst = v;
  } else {
    int last = -1;
    for (int i = b; i < e; ++i) {
      const int f = inv_flat[i];
      if (f / A.arity >= exec_size) break;
      last = f;
    }
    if (last >= 0) *dst = A.scr[(size_t)last * vpe + c];
  }
}

// deferred DG facet records: one thread per (target, DoF row)
template <int FAM>
__global__ void k_untiled_apply_deferred(const DLoop *__restrict__ Lp, const int32_t *inv_off,
                                         const int32_t *inv_flat, int64_t n_target,
                                         int exec_size) {
  const DLoop &L = *Lp;
  const int nd = L.a[4].vpe >> 1, ar = L.a[4].arity;
  int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= n_target * nd) return;
  const int64_t t = w / nd;
  const int i = (int)(w - t * nd);
  int b = inv_off[t], e = inv_off[t + 1];
  while (e > b && inv_flat[e - 1] / ar >= exec_size) --e;  // ascending: non-exec sources last
  lift_apply_item<FAM>(L, L.a[4].data + t * L.a[4].vpe + i, L.a[5].data + t * L.a[5].vpe + i, nd,
                       i, L.a[4].scr, inv_flat, b, e);
}

static DeferredFn untiled_deferred_fn(int fam) {
  switch (fam) {
    case 1: return k_untiled_apply_deferred<1>;
    case 2: return k_untiled_apply_deferred<2>;
    case 3: return k_untiled_apply_deferred<3>;
    case 4: return k_untiled_apply_deferred<4>;
    default: return k_untiled_apply_deferred<5>;
  }
}

// ---- plan building -------------------------------------------------------------------
__global__ void k_inc_keys(const int32_t *elements, const int32_t *sigma, const int32_t *offsets,
                           const int32_t *chunk_base, const int32_t *map, int arity, int CH0,
                           const int32_t *tile_chunk, int64_t n, uint64_t *keys, int32_t *vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * arity) return;
  const int64_t p = i / arity;
  const int k = (int)(i - p * arity);
  const int e = elements[p];
  const int t = sigma[e];
  const int pos = (int)(p - offsets[t]);
  const int CH = tile_chunk ? tile_chunk[t] : CH0;  // per-tile chunks (staged deferred loops)
  const uint64_t gc = (uint64_t)(chunk_base[t] + pos / CH);
  keys[i] = (gc << 32) | (uint32_t)map[(int64_t)e * arity + k];
  vals[i] = (pos % CH) * arity + k;
}

__global__ void k_run_heads(const uint64_t *keys, int64_t n, int32_t *heads) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  heads[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_run_fill(const uint64_t *keys, const int32_t *heads, const int32_t *run_idx,
                           int64_t n, int32_t *utgt, int32_t *ut_off, uint32_t *run_gc) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (heads[i]) {
    const int r = run_idx[i];
    utgt[r] = (int32_t)(keys[i] & 0xffffffffu);
    run_gc[r] = (uint32_t)(keys[i] >> 32);
    ut_off[r] = (int32_t)i;
  }
}

__global__ void k_set_int(int32_t *p, int32_t v) { *p = v; }

struct IncBuffers {
  DevBuf<int32_t> gc_off, utgt, ut_off, slots;
  DevBuf<uint32_t> run_gc;  // global chunk of each unique target
  int64_t runs = 0;
};

// ---- tile footprints (staged executor plan) ------------------------------------------
// FP(t, S): ascending unique elements of space S that tile t touches in any loop,
// directly or through a map.  The extension of compute_local_maps
// (inspector.py:397-418) that makes tile-local numbering possible.
struct Footprint {
  DevBuf<int32_t> off;   // n_tiles + 1
  DevBuf<int32_t> elem;  // concatenated, ascending per tile
  DevBuf<uint32_t> tile; // tile of each entry
  int64_t n = 0;
  std::vector<int32_t> off_host;
};

static constexpr uint64_t kNoKey = ~0ull;

__global__ void k_fp_keys_direct(const int32_t *sigma, int64_t n, const int32_t *region,
                                 uint64_t *keys) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int t = sigma[e];
  keys[e] = (region[t] == LT_NONEXEC) ? kNoKey : (((uint64_t)t << 32) | (uint32_t)e);
}

__global__ void k_fp_keys_mapped(const int32_t *sigma, const int32_t *map, int arity, int64_t n,
                                 const int32_t *region, uint64_t *keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * arity) return;
  const int t = sigma[i / arity];
  keys[i] = (region[t] == LT_NONEXEC) ? kNoKey : (((uint64_t)t << 32) | (uint32_t)map[i]);
}

__global__ void k_fp_heads(const uint64_t *keys, int64_t n, int32_t *heads) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  heads[i] = (keys[i] != kNoKey && (i == 0 || keys[i] != keys[i - 1])) ? 1 : 0;
}

__global__ void k_fp_fill(const uint64_t *keys, const int32_t *heads, const int32_t *idx,
                          int64_t n, int32_t *elem, uint32_t *tile) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || !heads[i]) return;
  elem[idx[i]] = (int32_t)(keys[i] & 0xffffffffu);
  tile[idx[i]] = (uint32_t)(keys[i] >> 32);
}

__device__ __forceinline__ int fp_slot(const int32_t *fp_off, const int32_t *fp_elem, int t,
                                       int e) {
  int lo = fp_off[t], hi = fp_off[t + 1];
  const int b = lo;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (fp_elem[mid] < e) lo = mid + 1; else hi = mid;
  }
  return lo - b;
}

// slot of each list position (direct) or each (position, k) (mapped); -1 on T_ne
__global__ void k_slots(const int32_t *elements, const int32_t *sigma, const int32_t *map,
                        int arity, int64_t n, const int32_t *region, const int32_t *fp_off,
                        const int32_t *fp_elem, int32_t *slot) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * arity) return;
  const int e = elements[i / arity];
  const int t = sigma[e];
  if (region[t] == LT_NONEXEC) { slot[i] = -1; return; }
  const int target = map ? map[(int64_t)e * arity + (i % arity)] : e;
  slot[i] = fp_slot(fp_off, fp_elem, t, target);
}

__global__ void k_mark_written(const int32_t *elements, const int32_t *sigma, int arity,
                               int64_t n, const int32_t *fp_off, const int32_t *slot,
                               uint8_t *flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * arity) return;
  const int s = slot[i];
  if (s < 0) return;
  flag[fp_off[sigma[elements[i / arity]]] + s] = 1;
}

// unique INC targets of a chunk -> footprint slots of the chunk's tile
__global__ void k_utgt_to_slot(int32_t *utgt, const uint32_t *run_gc, int64_t R,
                               const int32_t *gc_tile, const int32_t *fp_off,
                               const int32_t *fp_elem) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int t = gc_tile[run_gc[r]];
  utgt[r] = fp_slot(fp_off, fp_elem, t, utgt[r]);
}

struct FpSource {
  int loop;
  int map;  // -1: direct (the loop's own elements)
};

static void build_footprint(Ctx &ctx, const lt_schedule *s, const ChainView &cv,
                            const std::vector<FpSource> &src, const DevBuf<int32_t> &region,
                            Footprint &fp) {
  int64_t nkeys = 0;
  for (const FpSource &f : src)
    nkeys += s->lists[f.loop].n * (f.map < 0 ? 1 : cv.maps[f.map].arity);
  DevBuf<uint64_t> keys(std::max<int64_t>(nkeys, 1), ctx.stream),
      sorted(std::max<int64_t>(nkeys, 1), ctx.stream);
  int64_t at = 0;
  for (const FpSource &f : src) {
    const LoopLists &L = s->lists[f.loop];
    if (f.map < 0) {
      if (L.n)
        k_fp_keys_direct<<<grid_for(L.n, 256), 256, 0, ctx.stream>>>(L.sigma.get(), L.n,
                                                                     region.get(), keys.get() + at);
      at += L.n;
    } else {
      const lt_map &mp = cv.maps[f.map];
      if (L.n)
        k_fp_keys_mapped<<<grid_for(L.n * mp.arity, 256), 256, 0, ctx.stream>>>(
            L.sigma.get(), mp.values, mp.arity, L.n, region.get(), keys.get() + at);
      at += L.n * mp.arity;
    }
    LT_CK_LAUNCH();
  }
  if (nkeys) {
    size_t tmp = 0;
    LT_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.get(), sorted.get(), (int)nkeys, 0, 64,
                                         ctx.stream));
    DevBuf<char> t((int64_t)tmp, ctx.stream);
    LT_CK(cub::DeviceRadixSort::SortKeys(t.get(), tmp, keys.get(), sorted.get(), (int)nkeys, 0, 64,
                                         ctx.stream));
  }
  DevBuf<int32_t> heads(std::max<int64_t>(nkeys, 1), ctx.stream),
      idx(std::max<int64_t>(nkeys, 1), ctx.stream);
  int64_t U = 0;
  if (nkeys) {
    k_fp_heads<<<grid_for(nkeys, 256), 256, 0, ctx.stream>>>(sorted.get(), nkeys, heads.get());
    LT_CK_LAUNCH();
    size_t tmp = 0;
    LT_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, heads.get(), idx.get(), (int)nkeys,
                                        ctx.stream));
    DevBuf<char> t((int64_t)tmp, ctx.stream);
    LT_CK(cub::DeviceScan::ExclusiveSum(t.get(), tmp, heads.get(), idx.get(), (int)nkeys,
                                        ctx.stream));
    int32_t li = 0, lh = 0;
    LT_CK(cudaMemcpyAsync(&li, idx.get() + nkeys - 1, 4, cudaMemcpyDeviceToHost, ctx.stream));
    LT_CK(cudaMemcpyAsync(&lh, heads.get() + nkeys - 1, 4, cudaMemcpyDeviceToHost, ctx.stream));
    LT_CK(cudaStreamSynchronize(ctx.stream));
    U = (int64_t)li + lh;
  }
  fp.elem.alloc(std::max<int64_t>(U, 1), ctx.stream);
  fp.tile.alloc(std::max<int64_t>(U, 1), ctx.stream);
  fp.n = U;
  DevBuf<uint32_t> &tile = fp.tile;
  if (nkeys) {
    k_fp_fill<<<grid_for(nkeys, 256), 256, 0, ctx.stream>>>(sorted.get(), heads.get(), idx.get(),
                                                            nkeys, fp.elem.get(), tile.get());
    LT_CK_LAUNCH();
  }
  fp.off.alloc(s->n_tiles + 1, ctx.stream);
  lower_bound_u32(ctx, tile.get(), U, s->n_tiles, fp.off.get());
  fp.off_host.resize(s->n_tiles + 1);
  LT_CK(cudaMemcpyAsync(fp.off_host.data(), fp.off.get(), sizeof(int32_t) * (s->n_tiles + 1),
                        cudaMemcpyDeviceToHost, ctx.stream));
  LT_CK(cudaStreamSynchronize(ctx.stream));
}

struct LoopPlan {
  int chunk = LT_BLOCK;
  bool deferred = false;    // staged: DG facet loop applied by its deferred lift
  int scratch_per_pos = 0;  // doubles
  DevBuf<int32_t> chunk_base;
  DevBuf<int32_t> gc_tile;  // staged: tile of each global chunk
  std::vector<int32_t> tile_chunk_host;  // staged deferred loops: chunk of each tile (else empty)
  DevBuf<int32_t> tile_chunk;
  std::vector<IncBuffers> inc;  // per apply plan
  std::vector<int> inc_desc;
  std::vector<int> plan_map;    // map of each apply plan
  std::vector<DevBuf<int32_t>> slots;  // staged: per descriptor footprint slots
};

struct ExecPlan {
  std::string key;
  bool staged = false;
  std::vector<LoopPlan> loops;
  std::vector<std::pair<int, DevBuf<int32_t>>> phases;  // (#tiles, tile ids) per colour phase
  std::vector<int> phase_region;
  std::vector<int> phase_color;
  DevBuf<DLoop> dloops;
  std::vector<DLoop> host_loops;
  size_t smem_bytes = 0;
  // staged
  std::map<int, Footprint> fp;               // per space
  std::vector<DevBuf<uint8_t>> wflags;        // per staged dataset
  std::vector<DevBuf<int32_t>> wlist;         // per dataset: written footprint positions
  std::vector<DevBuf<int32_t>> llist;         // per dataset (load == 2): rows to gather
  std::vector<std::vector<int32_t>> lbeg;     // per dataset, per tile: first entry in llist
  std::vector<std::vector<int32_t>> wbeg;     // per dataset, per tile: first entry in wlist
  StagedParams sp;
  DevBuf<int32_t> region;
  std::vector<int32_t> rank;  // execution order key: colour refined by write-conflict sub-colour
  int max_subcolor = 0;
  DevBuf<int32_t> blob, blob_len;
  DevBuf<int64_t> blob_off;
  size_t data_max = 0;  // largest per-tile dataset rows (bytes)
  size_t ds_bytes = 0;  // total bytes of the staged datasets (queue-order choice)
  size_t scratch_bytes = 0;  // contribution/record scratch per CTA
  std::vector<size_t> tile_rows;   // per tile: dataset-row bytes (diagnostics)
  std::vector<int32_t> tile_blob;  // per tile: tile-program ints (diagnostics)
  std::vector<int32_t> scratch_base_host;  // per tile: first double of its scratch in smem
  // dataflow
  bool dataflow = false;
  DevBuf<int32_t> order_all, order_core, order_bnd, nbr_off, nbr, done, queue;
  int last_call = -1;  // dataflow: 0 both phases, 1 core only, 2 boundary only
  std::vector<int32_t> nbr_off_host, nbr_host;  // dependency lists (queue-order construction)
  std::vector<int32_t> exec_host[3];            // tiles per call kind: all, core, boundary
  struct Items {
    DevBuf<int64_t> tk, ol;  // per queue item: repeat << 32 | tile; length << 40 | offset
  };
  std::map<std::pair<int, int>, Items> items;  // per (call kind, repeats)
  std::vector<int64_t> blob_off_host;          // per tile: program offset (ints)
  std::vector<int32_t> blob_len_host, blob_full_host;  // program / program + packed rows
  std::map<std::pair<int, int>, int> items_wave;  // 1: wavefront order chosen
  int n_all = 0, n_core = 0, n_bnd = 0, grid = 0;
  bool wide = false;  // wide build (tile programs allow <= LT_WIDE_MINB CTAs per SM)
};

static int choose_chunk(int scratch_per_pos, size_t smem_budget, int block, bool round = true) {
  if (scratch_per_pos == 0) return block;
  int ch = (int)(smem_budget / (sizeof(double) * (size_t)scratch_per_pos));
  ch = std::min(ch, block);
  if (round && ch >= 32) ch -= ch % 32;
  if (ch < 1) fail(LT_E_EXECUTION, "loop contributions exceed shared memory");
  return ch;
}

// Ordered-gather plan of one mapped INC/WRITE descriptor: per global chunk the
// unique targets and, per target, its contributor slots in (element, k) order.
// With a footprint, targets are converted to tile-local slots.
static void build_inc_plan(Ctx &ctx, const lt_schedule *s, int j, const lt_map &mp, int CH,
                           const std::vector<int32_t> &chunk_base_host,
                           const DevBuf<int32_t> &chunk_base, IncBuffers &out,
                           const Footprint *fp, const DevBuf<int32_t> *gc_tile,
                           const int32_t *tile_chunk = nullptr) {
  const LoopLists &Lj = s->lists[j];
  const int64_t n = Lj.n, nnz = n * mp.arity;
  const int64_t n_gc = chunk_base_host.back();
  DevBuf<uint64_t> kin(nnz, ctx.stream), kout(nnz, ctx.stream);
  DevBuf<int32_t> vin(nnz, ctx.stream);
  out.slots.alloc(std::max<int64_t>(nnz, 1), ctx.stream);
  out.gc_off.alloc(n_gc + 1, ctx.stream);
  if (nnz == 0) {
    LT_CK(cudaMemsetAsync(out.gc_off.get(), 0, sizeof(int32_t) * (n_gc + 1), ctx.stream));
    out.utgt.alloc(1, ctx.stream);
    out.ut_off.alloc(1, ctx.stream);
    LT_CK(cudaMemsetAsync(out.ut_off.get(), 0, sizeof(int32_t), ctx.stream));
    return;
  }
  k_inc_keys<<<grid_for(nnz, 256), 256, 0, ctx.stream>>>(
      Lj.elements.get(), Lj.sigma.get(), Lj.offsets.get(), chunk_base.get(), mp.values, mp.arity,
      CH, tile_chunk, n, kin.get(), vin.get());
  LT_CK_LAUNCH();
  sort_pairs_u64(ctx, kin.get(), vin.get(), nnz, 32 + bits_for(n_gc), kout.get(),
                 out.slots.get());
  DevBuf<int32_t> heads(nnz, ctx.stream), run_idx(nnz, ctx.stream);
  k_run_heads<<<grid_for(nnz, 256), 256, 0, ctx.stream>>>(kout.get(), nnz, heads.get());
  LT_CK_LAUNCH();
  size_t tmp = 0;
  LT_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, heads.get(), run_idx.get(), (int)nnz,
                                      ctx.stream));
  DevBuf<char> t((int64_t)tmp, ctx.stream);
  LT_CK(cub::DeviceScan::ExclusiveSum(t.get(), tmp, heads.get(), run_idx.get(), (int)nnz,
                                      ctx.stream));
  int32_t last_idx = 0, last_head = 0;
  LT_CK(cudaMemcpyAsync(&last_idx, run_idx.get() + nnz - 1, sizeof(int32_t),
                        cudaMemcpyDeviceToHost, ctx.stream));
  LT_CK(cudaMemcpyAsync(&last_head, heads.get() + nnz - 1, sizeof(int32_t),
                        cudaMemcpyDeviceToHost, ctx.stream));
  LT_CK(cudaStreamSynchronize(ctx.stream));
  const int64_t R = (int64_t)last_idx + last_head;
  out.utgt.alloc(R, ctx.stream);
  out.ut_off.alloc(R + 1, ctx.stream);
  out.run_gc.alloc(R, ctx.stream);
  out.runs = R;
  DevBuf<uint32_t> &run_gc = out.run_gc;
  k_run_fill<<<grid_for(nnz, 256), 256, 0, ctx.stream>>>(kout.get(), heads.get(), run_idx.get(),
                                                         nnz, out.utgt.get(), out.ut_off.get(),
                                                         run_gc.get());
  LT_CK_LAUNCH();
  k_set_int<<<1, 1, 0, ctx.stream>>>(out.ut_off.get() + R, (int32_t)nnz);
  LT_CK_LAUNCH();
  if (fp) {
    k_utgt_to_slot<<<grid_for(R, 256), 256, 0, ctx.stream>>>(
        out.utgt.get(), run_gc.get(), R, gc_tile->get(), fp->off.get(), fp->elem.get());
    LT_CK_LAUNCH();
  }
  lower_bound_u32(ctx, run_gc.get(), R, n_gc, out.gc_off.get());
  LT_CK(cudaStreamSynchronize(ctx.stream));
}

static void validate_bindings(const Ctx &ctx, const ChainView &cv, const lt_arg *args) {
  int a = 0;
  for (size_t j = 0; j < cv.loops.size(); ++j) {
    const LoopDesc &L = cv.loops[j];
    if (L.kernel < 0 || L.kernel >= kNumKernels)
      fail(LT_E_EXECUTION, "loop " + std::to_string(j) + ": unknown native kernel id");
    const KernelSpec &K = kSpecs[L.kernel];
    if (sig_count(K.sig) != (int)L.desc.size())
      fail(LT_E_EXECUTION, "kernel '" + std::string(K.name) + "' takes " +
                               std::to_string(sig_count(K.sig)) + " args, loop " +
                               std::to_string(j) + " has " + std::to_string(L.desc.size()) +
                               " descriptors");
    if ((int)L.desc.size() > LT_MAX_DESC) fail(LT_E_EXECUTION, "too many descriptors");
    const char *p = K.sig;
    int n_inc = 0;
    for (size_t d = 0; d < L.desc.size(); ++d, p += 3) {
      const lt_desc &D = L.desc[d];
      const lt_arg &A = args[a + d];
      const bool direct = D.map < 0;
      const std::string where = "loop " + std::to_string(j) + " arg " + std::to_string(d) +
                                " of kernel '" + K.name + "'";
      if ((p[0] == 'D') != direct)
        fail(LT_E_EXECUTION, where + (direct ? ": needs a mapped access" : ": needs a direct access"));
      const int64_t want = direct ? cv.total(L.space) : cv.total(cv.maps[D.map].target);
      if (A.n_elements != want || A.vpe < 1 || !A.values)
        fail(LT_E_EXECUTION, where + ": dataset size does not match its space");
      if (p[1] == 'R' && D.mode != LT_READ)
        fail(LT_E_EXECUTION, where + ": kernel only reads this argument");
      if ((p[1] == 'W' || p[1] == 'F') && D.mode != LT_WRITE && D.mode != LT_RW)
        fail(LT_E_EXECUTION, where + ": kernel writes this argument (WRITE/RW required)");
      if (p[1] == 'I' && D.mode != LT_INC && D.mode != LT_WRITE)
        fail(LT_E_EXECUTION, where + ": kernel increments this argument (INC required)");
      if (!direct && D.mode == LT_RW)
        fail(LT_E_EXECUTION, where + ": mapped RW access is not a parallel loop");
      if (p[1] == 'I') ++n_inc;
    }
    if (n_inc > LT_MAX_INC) fail(LT_E_EXECUTION, "too many indirect increments in one loop");
    // kernel-specific shape rules
    const std::string kn = K.name;
    if (kn == "edge_inc" || kn == "cell_inc" || kn == "toy_k1" || kn == "edge_read" ||
        kn == "cell_read" || kn == "toy_k2" || kn == "toy_k3") {
      if (args[a].vpe != args[a + 1].vpe)
        fail(LT_E_EXECUTION, "loop " + std::to_string(j) + ": kernel '" + kn +
                                 "' needs equal values_per_element on both arguments");
      int ar = cv.maps[L.desc[1].map].arity;
      if ((kn == "toy_k2" && ar != 2) || (kn == "toy_k3" && ar != 3))
        fail(LT_E_EXECUTION, "loop " + std::to_string(j) + ": kernel '" + kn +
                                 "' needs a map of arity " + (kn == "toy_k2" ? "2" : "3"));
    } else {
      dg_validate(L.kernel - K_DG_FIRST, j, cv, L, args + a);
      const int64_t np_ = dg_param_count(L.kernel - K_DG_FIRST);
      auto it = ctx.params.find(L.kernel);
      if (np_ > 0 && (it == ctx.params.end() || it->second.n < np_))
        fail(LT_E_EXECUTION, "loop " + std::to_string(j) + ": kernel '" + kn +
                                 "' needs its parameter block (" + std::to_string(np_) +
                                 " doubles) set with lt_ctx_set_kernel_params");
    }
    // a loop may not increment the same dataset through two descriptors, nor
    // read through a map what it increments (par_loop semantics)
    for (size_t d = 0; d < L.desc.size(); ++d) {
      if (L.desc[d].map < 0 || L.desc[d].mode == LT_READ) continue;
      for (size_t e = 0; e < L.desc.size(); ++e) {
        if (e == d || args[a + e].values != args[a + d].values) continue;
        if (L.desc[e].map >= 0)
          fail(LT_E_EXECUTION, "loop " + std::to_string(j) +
                                   ": a dataset incremented through a map may not be accessed "
                                   "through another descriptor of the same loop");
      }
    }
    a += (int)L.desc.size();
  }
}

static void fill_dloop(DLoop &D, const ChainView &cv, int j, const lt_arg *args, const Ctx &ctx,
                       int use_local) {
  const LoopDesc &L = cv.loops[j];
  std::memset(&D, 0, sizeof(D));
  D.kernel = L.kernel;
  D.n_desc = (int)L.desc.size();
  D.use_local = use_local;
  D.exec_size = (int)cv.exec_size(L.space);
  D.lanes = L.kernel >= K_DG_FIRST ? dg_lanes(L.kernel - K_DG_FIRST) : 1;
  D.lane_magic = lt_magic(D.lanes);
  D.lane_dq = LT_SBLOCK / D.lanes;
  D.lane_dr = LT_SBLOCK % D.lanes;
  if (L.kernel >= K_DG_FIRST && dg_is_flux(L.kernel - K_DG_FIRST)) {  // validated: one map, INC
    D.deferred = 1;
    D.rec = dg_corr_size(L.kernel - K_DG_FIRST);
    const int nd = dg_nd((L.kernel - K_DG_FIRST) / 5 + 1);
    D.row_magic = lt_magic(nd);
    D.row_dq = LT_SBLOCK / nd;
    D.row_dr = LT_SBLOCK % nd;
  }
  auto it = ctx.params.find(L.kernel);
  D.params = it == ctx.params.end() ? nullptr : it->second.get();
  for (int d = 0; d < D.n_desc; ++d) {
    DArg &A = D.a[d];
    A.data = args[d].values;
    A.vpe = args[d].vpe;
    A.mode = L.desc[d].mode;
    A.arity = L.desc[d].map < 0 ? 1 : cv.maps[L.desc[d].map].arity;
    A.map = L.desc[d].map < 0 ? nullptr : cv.maps[L.desc[d].map].values;
  }
}

static std::string plan_key(const Ctx &ctx, const ChainView &cv, const lt_arg *args,
                            int use_local) {
  std::string k = std::to_string(use_local) + "|" + std::to_string(ctx.params_gen) + "|";
  int a = 0;
  for (const LoopDesc &L : cv.loops) {
    k += std::to_string(L.kernel) + ":";
    for (const lt_desc &d : L.desc) {
      k += std::to_string(d.map) + "/" + std::to_string(d.mode) + "/" +
           std::to_string(args[a].vpe) + "/" + std::to_string((uintptr_t)args[a].values) + "/" +
           std::to_string(d.map < 0 ? 0 : (uintptr_t)cv.maps[d.map].values) + ",";
      ++a;
    }
    k += ";";
  }
  return k;
}

static const size_t kSmemBudget = 96 * 1024;
// shared scratch for one chunk of INC contributions in the staged executor
// (smaller chunks: more apply phases, more resident tiles per SM)
#ifndef LT_SCRATCH1_DEFAULT_KB
// 4 KB: with per-tile chunks the first pass only fixes the shortest chunk and
// the occupancy target; 8 KB cost config 3 (P2, Morton ts 32) its fourth CTA
// per SM (72.6 KB -> 56.6 KB per CTA: 12.13 -> 10.91 ms)
#define LT_SCRATCH1_DEFAULT_KB 4
#endif
// First-pass record/contribution scratch per CTA.  LT_SCRATCH_KB fixes it (and
// switches the later planning passes off); LT_SCRATCH1_KB only sets the first
// pass, i.e. the shortest chunk any tile gets and the shared memory the
// occupancy target is derived from (per-tile chunks still grow from there).
static size_t scratch_budget() {
  const char *e = getenv("LT_SCRATCH_KB");
  if (!e) e = getenv("LT_SCRATCH1_KB");
  return (e ? (size_t)atoi(e) : LT_SCRATCH1_DEFAULT_KB) * 1024;
}
static std::string g_last_fit;
static const size_t kSmemMax = 227 * 1024;
static const size_t kAlignSlack = LT_TMA_GATHER ? 128 : 0;  // skipped by lt_align128

__global__ void k_zero_at(int32_t *v, const int32_t *idx, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[idx[i]] = 0;
}

// ---- tile dependency graph of the dataflow executor ---------------------------------
// Two tiles depend on each other iff their footprints share an element of some
// space (every RAW/WAR/WAW hazard between tiles needs a shared element).
__global__ void k_elem_tile_keys(const int32_t *elem, const uint32_t *tile, int64_t n,
                                 uint64_t *keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) keys[i] = ((uint64_t)(uint32_t)elem[i] << 32) | tile[i];
}

__global__ void k_run_start(const uint64_t *keys, int64_t n, int32_t *r0) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  r0[i] = (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ? (int32_t)i : 0;
}

__global__ void k_pair_count(const int32_t *r0, int64_t n, int32_t *cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) cnt[i] = 2 * (int32_t)(i - r0[i]);
}

__global__ void k_pair_emit(const uint64_t *keys, const int32_t *r0, const int32_t *pos,
                            int64_t n, uint64_t *pairs) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t ti = (uint32_t)keys[i];
  int64_t o = pos[i];
  for (int64_t j = r0[i]; j < i; ++j) {
    const uint32_t tj = (uint32_t)keys[j];
    pairs[o++] = ((uint64_t)ti << 32) | tj;
    pairs[o++] = ((uint64_t)tj << 32) | ti;
  }
}

__global__ void k_self_pairs(const int32_t *order, int n, uint64_t *pairs) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) pairs[i] = ((uint64_t)(uint32_t)order[i] << 32) | (uint32_t)order[i];
}

__global__ void k_nbr_fill(const uint64_t *pairs, const int32_t *heads, const int32_t *idx,
                           int64_t n, const int32_t *color, int32_t *nbr, uint32_t *owner) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || !heads[i]) return;
  const int a = (int)(pairs[i] >> 32), b = (int)(uint32_t)pairs[i];
  nbr[idx[i]] = (b << 1) | (color[b] < color[a] ? 1 : 0);
  owner[idx[i]] = (uint32_t)a;
}

static void exclusive_sum(Ctx &ctx, const int32_t *in, int32_t *out, int64_t n) {
  size_t tmp = 0;
  LT_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, ctx.stream));
  DevBuf<char> t((int64_t)tmp, ctx.stream);
  LT_CK(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, (int)n, ctx.stream));
}

static int64_t last_plus(Ctx &ctx, const int32_t *scan, const int32_t *vals, int64_t n) {
  int32_t a = 0, b = 0;
  LT_CK(cudaMemcpyAsync(&a, scan + n - 1, 4, cudaMemcpyDeviceToHost, ctx.stream));
  LT_CK(cudaMemcpyAsync(&b, vals + n - 1, 4, cudaMemcpyDeviceToHost, ctx.stream));
  LT_CK(cudaStreamSynchronize(ctx.stream));
  return (int64_t)a + b;
}

template <class T>
static void to_host(Ctx &ctx, const DevBuf<T> &d, int64_t n, std::vector<T> &h);

static void build_dependencies(Ctx &ctx, lt_schedule *s, ExecPlan &P) {
  // queue orders: (region, colour, id)
  std::vector<int32_t> all, core, bnd;
  for (int reg : {LT_CORE, LT_BOUNDARY}) {
    std::vector<int32_t> v;
    for (int t = 0; t < s->n_tiles; ++t)
      if (s->region[t] == reg) v.push_back(t);
    std::stable_sort(v.begin(), v.end(),
                     [&](int a, int b) { return P.rank[a] < P.rank[b]; });
    (reg == LT_CORE ? core : bnd) = v;
    all.insert(all.end(), v.begin(), v.end());
  }
  P.n_all = (int)all.size();
  P.n_core = (int)core.size();
  P.n_bnd = (int)bnd.size();
  P.exec_host[0] = all;
  P.exec_host[1] = core;
  P.exec_host[2] = bnd;
  auto upload = [&](DevBuf<int32_t> &d, const std::vector<int32_t> &h) {
    d.alloc(std::max<int64_t>((int64_t)h.size(), 1), ctx.stream);
    if (!h.empty())
      LT_CK(cudaMemcpyAsync(d.get(), h.data(), 4 * h.size(), cudaMemcpyHostToDevice, ctx.stream));
  };
  upload(P.order_all, all);
  upload(P.order_core, core);
  upload(P.order_bnd, bnd);
  // overlapping tile pairs over every footprint space, plus (t, t)
  std::vector<DevBuf<uint64_t>> parts;
  std::vector<int64_t> sizes;
  for (auto &kv : P.fp) {
    Footprint &fp = kv.second;
    const int64_t n = fp.n;
    if (n == 0) continue;
    DevBuf<uint64_t> k(n, ctx.stream), ks(n, ctx.stream);
    k_elem_tile_keys<<<grid_for(n, 256), 256, 0, ctx.stream>>>(fp.elem.get(), fp.tile.get(), n,
                                                              k.get());
    LT_CK_LAUNCH();
    size_t tmp = 0;
    LT_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k.get(), ks.get(), (int)n, 0, 64,
                                         ctx.stream));
    DevBuf<char> tb((int64_t)tmp, ctx.stream);
    LT_CK(cub::DeviceRadixSort::SortKeys(tb.get(), tmp, k.get(), ks.get(), (int)n, 0, 64,
                                         ctx.stream));
    DevBuf<int32_t> r0(n, ctx.stream), r0m(n, ctx.stream), cnt(n, ctx.stream), pos(n, ctx.stream);
    k_run_start<<<grid_for(n, 256), 256, 0, ctx.stream>>>(ks.get(), n, r0.get());
    LT_CK_LAUNCH();
    tmp = 0;
    LT_CK(cub::DeviceScan::InclusiveScan(nullptr, tmp, r0.get(), r0m.get(), cub::Max(), (int)n,
                                         ctx.stream));
    DevBuf<char> tb2((int64_t)tmp, ctx.stream);
    LT_CK(cub::DeviceScan::InclusiveScan(tb2.get(), tmp, r0.get(), r0m.get(), cub::Max(), (int)n,
                                         ctx.stream));
    k_pair_count<<<grid_for(n, 256), 256, 0, ctx.stream>>>(r0m.get(), n, cnt.get());
    LT_CK_LAUNCH();
    exclusive_sum(ctx, cnt.get(), pos.get(), n);
    const int64_t total = last_plus(ctx, pos.get(), cnt.get(), n);
    DevBuf<uint64_t> pairs(std::max<int64_t>(total, 1), ctx.stream);
    k_pair_emit<<<grid_for(n, 256), 256, 0, ctx.stream>>>(ks.get(), r0m.get(), pos.get(), n,
                                                         pairs.get());
    LT_CK_LAUNCH();
    parts.push_back(std::move(pairs));
    sizes.push_back(total);
  }
  int64_t total = P.n_all;
  for (int64_t v : sizes) total += v;
  DevBuf<uint64_t> cat(std::max<int64_t>(total, 1), ctx.stream), srt(std::max<int64_t>(total, 1), ctx.stream);
  int64_t at = 0;
  for (size_t i = 0; i < parts.size(); ++i) {
    if (sizes[i])
      LT_CK(cudaMemcpyAsync(cat.get() + at, parts[i].get(), 8 * sizes[i], cudaMemcpyDeviceToDevice,
                            ctx.stream));
    at += sizes[i];
  }
  if (P.n_all) {
    k_self_pairs<<<grid_for(P.n_all, 256), 256, 0, ctx.stream>>>(P.order_all.get(), P.n_all,
                                                               cat.get() + at);
    LT_CK_LAUNCH();
  }
  size_t tmp = 0;
  if (total) {
    LT_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, cat.get(), srt.get(), (int)total, 0, 64,
                                         ctx.stream));
    DevBuf<char> tb((int64_t)tmp, ctx.stream);
    LT_CK(cub::DeviceRadixSort::SortKeys(tb.get(), tmp, cat.get(), srt.get(), (int)total, 0, 64,
                                         ctx.stream));
  }
  DevBuf<int32_t> heads(std::max<int64_t>(total, 1), ctx.stream), idx(std::max<int64_t>(total, 1), ctx.stream);
  int64_t U = 0;
  if (total) {
    k_run_heads<<<grid_for(total, 256), 256, 0, ctx.stream>>>(srt.get(), total, heads.get());
    LT_CK_LAUNCH();
    exclusive_sum(ctx, heads.get(), idx.get(), total);
    U = last_plus(ctx, idx.get(), heads.get(), total);
  }
  DevBuf<int32_t> color(s->n_tiles, ctx.stream);
  LT_CK(cudaMemcpyAsync(color.get(), P.rank.data(), 4 * s->n_tiles, cudaMemcpyHostToDevice,
                        ctx.stream));
  P.nbr.alloc(std::max<int64_t>(U, 1), ctx.stream);
  DevBuf<uint32_t> owner(std::max<int64_t>(U, 1), ctx.stream);
  if (total) {
    k_nbr_fill<<<grid_for(total, 256), 256, 0, ctx.stream>>>(srt.get(), heads.get(), idx.get(),
                                                            total, color.get(), P.nbr.get(),
                                                            owner.get());
    LT_CK_LAUNCH();
  }
  P.nbr_off.alloc(s->n_tiles + 1, ctx.stream);
  lower_bound_u32(ctx, owner.get(), U, s->n_tiles, P.nbr_off.get());
  P.done.alloc(s->n_tiles, ctx.stream);
  P.queue.alloc(1, ctx.stream);
  to_host(ctx, P.nbr_off, s->n_tiles + 1, P.nbr_off_host);
  to_host(ctx, P.nbr, U, P.nbr_host);
  LT_CK(cudaStreamSynchronize(ctx.stream));
}

// Queue items (repeat k, tile t) of one dataflow call.  Every dependency of an
// item must precede it in the queue (deadlock freedom); two orders qualify:
//  * colour-major: (k, colour, id) -- a colour class sweeps the whole mesh
//    before the next starts;
//  * wavefront: key = t + level * D with level = k * C + colour rank, D > the
//    largest tile-id distance to a dependency, so each colour (and repeat)
//    sweeps the mesh D tiles behind the previous one.  The live window is
//    ~C * D tiles instead of the whole mesh: rows shared by overlapping tiles
//    of successive colours are re-read from L2, not HBM.  D also adds two
//    grids of slack so a popped item rarely waits on a running dependency
//    (config 3: one grid is 31 % slower from dependency waits; two grids are
//    3.5 % faster than colour-major with 34 % less DRAM traffic; 4-8 grids
//    are as fast with more traffic).
// Wavefront is used when the staged datasets do not fit in half of L2 (or
// LT_ORDER=wave); the item list is checked against every dependency either way.
// read-only rows are packed behind the tile programs when every tile of the
// call runs more than once (packing costs one pass over those rows)
static bool pack_for(const ExecPlan &P, int repeats) {
  return P.sp.ro_packed && repeats >= 2 && !getenv("LT_NO_PACK");
}

static void build_items(Ctx &ctx, ExecPlan &P, int kind, int repeats, size_t ds_bytes) {
  const std::vector<int32_t> &tiles = P.exec_host[kind];
  const int n = (int)tiles.size();
  const int64_t ni = (int64_t)n * repeats;
  int l2 = 0;
  LT_CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx.device));
  const char *ord = getenv("LT_ORDER");
  bool wave = ord ? !strcmp(ord, "wave") : ds_bytes > (size_t)l2 / 2;
  std::vector<int32_t> it_t(ni), it_k(ni);
  // colour-major (the tiles are already sorted by rank within each region)
  for (int k = 0, q = 0; k < repeats; ++k)
    for (int i = 0; i < n; ++i, ++q) it_t[q] = tiles[i], it_k[q] = k;
  const int tmax = n ? *std::max_element(tiles.begin(), tiles.end()) + 1 : 1;
  std::vector<int32_t> pos_of((size_t)repeats * tmax, -1);
  // a same-repeat dependency outside this call's queue is only satisfied by an
  // earlier call when this is the boundary-only call and the dependency is a
  // core tile (its core-only call ran first: the host checks that order);
  // anything else would spin forever on the device
  std::vector<char> is_core;
  if (kind == 2) {
    is_core.assign(P.rank.size(), 0);
    for (int t : P.exec_host[1]) is_core[t] = 1;
  }
  auto outside_ok = [&](int u) { return kind == 2 && u < (int)is_core.size() && is_core[u]; };
  auto check = [&]() {
    for (int64_t q = 0; q < ni; ++q) pos_of[(size_t)it_k[q] * tmax + it_t[q]] = (int32_t)q;
    for (int64_t q = 0; q < ni; ++q) {
      const int t = it_t[q], k = it_k[q];
      for (int e = P.nbr_off_host[t]; e < P.nbr_off_host[t + 1]; ++e) {
        const int u = P.nbr_host[e] >> 1, rep = k + (P.nbr_host[e] & 1) - 1;
        if (rep < 0) continue;
        const int32_t pu = u < tmax ? pos_of[(size_t)rep * tmax + u] : -1;
        if (pu < 0) {
          if ((P.nbr_host[e] & 1) && !outside_ok(u))
            fail(LT_E_EXECUTION, "dataflow: tile " + std::to_string(t) + " depends on tile " +
                                     std::to_string(u) + " of a lower colour that this call "
                                     "does not execute (boundary colours must exceed core "
                                     "colours)");
          continue;
        }
        if (pu >= q) return false;
      }
    }
    return true;
  };
  if (wave) {
    std::vector<int32_t> ranks;
    for (int t : tiles) ranks.push_back(P.rank[t]);
    std::sort(ranks.begin(), ranks.end());
    ranks.erase(std::unique(ranks.begin(), ranks.end()), ranks.end());
    const int C = (int)ranks.size();
    int64_t reach = 0;
    for (int t : tiles)
      for (int e = P.nbr_off_host[t]; e < P.nbr_off_host[t + 1]; ++e)
        reach = std::max<int64_t>(reach, (int64_t)(P.nbr_host[e] >> 1) - t);
    const char *sl = getenv("LT_WAVE_SLACK");  // slack in grids
    const double slack = sl ? atof(sl) : 2.0;
    const int64_t Dst = reach + 1 + (int64_t)(slack * (P.grid > 0 ? P.grid : 0));
    std::vector<std::pair<int64_t, int64_t>> key(ni);  // (key, item)
    for (int64_t q = 0; q < ni; ++q) {
      const int t = it_t[q], k = it_k[q];
      const int lvl = k * C + (int)(std::lower_bound(ranks.begin(), ranks.end(), P.rank[t]) -
                                    ranks.begin());
      key[q] = {(int64_t)t + lvl * Dst, (int64_t)lvl << 32 | (uint32_t)t};
    }
    std::vector<int64_t> perm(ni);
    for (int64_t q = 0; q < ni; ++q) perm[q] = q;
    std::sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return key[a] < key[b]; });
    std::vector<int32_t> wt(ni), wk(ni);
    for (int64_t q = 0; q < ni; ++q) wt[q] = it_t[perm[q]], wk[q] = it_k[perm[q]];
    std::swap(wt, it_t);
    std::swap(wk, it_k);
    std::fill(pos_of.begin(), pos_of.end(), -1);
    if (!check()) {  // cannot happen by construction; keep the proven order
      for (int k = 0, q = 0; k < repeats; ++k)
        for (int i = 0; i < n; ++i, ++q) it_t[q] = tiles[i], it_k[q] = k;
      wave = false;
    }
  }
  std::fill(pos_of.begin(), pos_of.end(), -1);
  if (!check()) fail(LT_E_EXECUTION, "dataflow queue order violates a tile dependency");
  const bool packed = pack_for(P, repeats);
  std::vector<int64_t> tk(ni), ol(ni);
  for (int64_t q = 0; q < ni; ++q) {
    const int t = it_t[q];
    tk[q] = (int64_t)it_k[q] << 32 | (uint32_t)t;
    const int64_t len = packed ? P.blob_full_host[t] : P.blob_len_host[t];
    if (P.blob_off_host[t] >= (1ll << 40) || len >= (1ll << 23))
      fail(LT_E_EXECUTION, "tile program offset/length out of the queue item range");
    ol[q] = len << 40 | P.blob_off_host[t];
  }
  auto &dst = P.items[{kind, repeats}];
  dst.tk.alloc(std::max<int64_t>(ni, 1), ctx.stream);
  dst.ol.alloc(std::max<int64_t>(ni, 1), ctx.stream);
  if (ni) {
    LT_CK(cudaMemcpyAsync(dst.tk.get(), tk.data(), 8 * ni, cudaMemcpyHostToDevice, ctx.stream));
    LT_CK(cudaMemcpyAsync(dst.ol.get(), ol.data(), 8 * ni, cudaMemcpyHostToDevice, ctx.stream));
  }
  LT_CK(cudaStreamSynchronize(ctx.stream));
  P.items_wave[{kind, repeats}] = wave ? 1 : 0;
}

// ---- tile programs ------------------------------------------------------------------
static int64_t ds_rows(int64_t n, bool tma);
struct Section {
  const void *src = nullptr;
  bool u8 = false;
  std::vector<int64_t> src_off, dst_off;
  std::vector<int32_t> len, sub;
};

__global__ void k_seg_copy(const int32_t *src, const int64_t *src_off, const int32_t *len,
                           const int32_t *sub, int32_t *dst, const int64_t *dst_off, int n) {
  for (int s = blockIdx.x; s < n; s += gridDim.x) {
    const int32_t *a = src + src_off[s];
    int32_t *b = dst + dst_off[s];
    const int32_t v = sub[s];
    for (int i = threadIdx.x; i < len[s]; i += blockDim.x) b[i] = a[i] - v;
  }
}

__global__ void k_seg_copy_u8(const uint8_t *src, const int64_t *src_off, const int32_t *len,
                              int32_t *dst, const int64_t *dst_off, int n) {
  for (int s = blockIdx.x; s < n; s += gridDim.x) {
    const uint8_t *a = src + src_off[s];
    int32_t *b = dst + dst_off[s];
    for (int i = threadIdx.x; i < len[s]; i += blockDim.x) b[i] = a[i];
  }
}

template <class T>
static void to_host(Ctx &ctx, const DevBuf<T> &d, int64_t n, std::vector<T> &h) {
  h.resize(n);
  if (n) LT_CK(cudaMemcpyAsync(h.data(), d.get(), sizeof(T) * n, cudaMemcpyDeviceToHost, ctx.stream));
}


__global__ void k_differs(const int32_t *a, const int32_t *b, int64_t n, int32_t *flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && a[i] != b[i]) *flag = 1;
}

// No barrier is needed between a direct loop j (no INC) and the first phase of
// loop j+1 when either
//  (a) both are direct-only over the same space with identical tile lists and
//      the same lanes, and their kernels touch only their lane's components
//      (DG inverse mass -> axpy): every thread re-runs its own items; or
//  (b) loop j+1's first phase (its body; INC bodies write only scratch) neither
//      reads nor writes a dataset loop j writes, and writes nothing loop j
//      reads (DG volume -> interior-facet records).
// 0: loop j+1 needs a barrier after loop j; 1: independent datasets; 2: same
// items and lane-local kernels (the executor may run both bodies per item)
static int barrier_free_pair(Ctx &ctx, const lt_schedule *s, const ChainView &cv,
                             const lt_arg *args, int j) {
  const LoopDesc &A = cv.loops[j], &Bq = cv.loops[j + 1];
  for (const lt_desc &d : A.desc)
    if (d.map >= 0 && d.mode != LT_READ) return false;  // loop j must not have an apply phase
  int a0 = 0;
  for (int q = 0; q < j; ++q) a0 += (int)cv.loops[q].desc.size();
  const lt_arg *aa = args + a0, *ab = aa + A.desc.size();
  // (b) dataset independence
  bool indep = true;
  for (size_t x = 0; x < A.desc.size() && indep; ++x) {
    const bool a_writes = A.desc[x].mode != LT_READ;
    for (size_t y = 0; y < Bq.desc.size() && indep; ++y) {
      if (aa[x].values != ab[y].values) continue;
      const bool b_body_writes = Bq.desc[y].map < 0 && Bq.desc[y].mode != LT_READ;
      const bool b_body_reads = Bq.desc[y].mode == LT_READ || Bq.desc[y].mode == LT_RW;
      if (a_writes && (b_body_reads || b_body_writes)) indep = false;
      if (!a_writes && b_body_writes) indep = false;
    }
  }
  if (indep) return 1;
  // (a) same items, lane-local kernels
  auto lane_local = [](int k) {
    return k >= K_DG_FIRST && ((k - K_DG_FIRST) % 5 == 3 || (k - K_DG_FIRST) % 5 == 4);
  };
  if (A.space != Bq.space || !lane_local(A.kernel) || !lane_local(Bq.kernel)) return false;
  if (dg_lanes(A.kernel - K_DG_FIRST) != dg_lanes(Bq.kernel - K_DG_FIRST)) return false;
  for (const lt_desc &d : A.desc)
    if (d.map >= 0) return false;
  for (const lt_desc &d : Bq.desc)
    if (d.map >= 0) return false;
  const LoopLists &La = s->lists[j], &Lb = s->lists[j + 1];
  if (La.n != Lb.n) return false;
  DevBuf<int32_t> flag(1, ctx.stream);
  LT_CK(cudaMemsetAsync(flag.get(), 0, 4, ctx.stream));
  k_differs<<<grid_for(s->n_tiles + 1, 256), 256, 0, ctx.stream>>>(
      La.offsets.get(), Lb.offsets.get(), s->n_tiles + 1, flag.get());
  if (La.n)
    k_differs<<<grid_for(La.n, 256), 256, 0, ctx.stream>>>(La.elements.get(), Lb.elements.get(),
                                                          La.n, flag.get());
  LT_CK_LAUNCH();
  int32_t f = 1;
  LT_CK(cudaMemcpyAsync(&f, flag.get(), 4, cudaMemcpyDeviceToHost, ctx.stream));
  LT_CK(cudaStreamSynchronize(ctx.stream));
  return f == 0 ? 2 : 0;
}

__global__ void k_u8_to_i32(const uint8_t *a, int64_t n, int32_t *b) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

__global__ void k_compact_written(const uint8_t *flag, const int32_t *scan, const uint32_t *tile,
                                  const int32_t *fp_off, int64_t n, int32_t *out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && flag[i]) out[scan[i]] = (int32_t)(i - fp_off[tile[i]]);
}

__global__ void k_gather_at(const int32_t *src, const int32_t *idx, int64_t n, int32_t *out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = src[idx[i]];
}

// Lay out and fill the per-tile programs; returns the largest blob in bytes.
static size_t build_blobs(Ctx &ctx, lt_schedule *s, const ChainView &cv, ExecPlan &P,
                          const std::map<int, int> &sp_index, const std::vector<int> &ds_space) {
  StagedParams &H = P.sp;
  const int nl = s->n_loops, nt = s->n_tiles;
  // header layout
  int hp = 2 * H.n_sp;
  for (int j = 0; j < nl; ++j) {
    H.loop_pos[j] = hp;
    hp += 2 + (int)cv.loops[j].desc.size() + 4 * (int)P.loops[j].plan_map.size();
  }
  H.ds_pos = hp;
  hp += 2 * H.n_ds;
  H.base_pos = hp;  // per dataset (+ scratch): first double of its rows in smem
  hp += H.n_ds + 1;
  H.ld_pos = hp;  // per dataset: (count, position) of its load list (load == 2)
  hp += 2 * H.n_ds;
  H.prog_pos = hp++;
  H.dep_pos = hp;  // dataflow: (count, position) of the tile's dependency list
  hp += 2;
  H.hs = hp;
  // host copies of the per-tile ranges
  std::vector<std::vector<int32_t>> off(nl), cb(nl);
  std::vector<std::vector<std::vector<int32_t>>> gco(nl), uto(nl);
  for (int j = 0; j < nl; ++j) {
    to_host(ctx, s->lists[j].offsets, nt + 1, off[j]);
    if (P.loops[j].chunk_base.get()) to_host(ctx, P.loops[j].chunk_base, nt + 1, cb[j]);
    gco[j].resize(P.loops[j].inc.size());
    uto[j].resize(P.loops[j].inc.size());
    for (size_t p = 0; p < P.loops[j].inc.size(); ++p) {
      to_host(ctx, P.loops[j].inc[p].gc_off, P.loops[j].inc[p].gc_off.n, gco[j][p]);
      to_host(ctx, P.loops[j].inc[p].ut_off, P.loops[j].inc[p].ut_off.n, uto[j][p]);
    }
  }
  LT_CK(cudaStreamSynchronize(ctx.stream));
  std::vector<const Footprint *> fps(H.n_sp);
  for (auto &kv : sp_index) fps[kv.second] = &P.fp.at(kv.first);

  // sections in blob order
  std::vector<Section> secs;
  auto sec = [&](const void *src, bool u8) -> Section & {
    secs.emplace_back();
    secs.back().src = src;
    secs.back().u8 = u8;
    return secs.back();
  };
  std::vector<int32_t> hdr_host;
  std::vector<int32_t> blen(nt, 0), bfull(nt, 0);
  std::vector<int64_t> boff(nt, 0);
  size_t blob_max = 0;
  int64_t total = 0;
  // section indices are fixed per chain; create them once
  std::vector<int> s_sp(H.n_sp), s_wf(H.n_ds, -1);
  std::vector<std::vector<int>> s_slot(nl), s_plan(nl);
  const int s_hdr = (int)secs.size();
  sec(nullptr, false);
  for (int k = 0; k < H.n_sp; ++k) s_sp[k] = (int)secs.size(), sec(fps[k]->elem.get(), false);
  for (int j = 0; j < nl; ++j) {
    for (size_t d = 0; d < cv.loops[j].desc.size(); ++d)
      s_slot[j].push_back((int)secs.size()), sec(P.loops[j].slots[d].get(), false);
    for (size_t p = 0; p < P.loops[j].inc.size(); ++p) {
      s_plan[j].push_back((int)secs.size());
      sec(P.loops[j].inc[p].gc_off.get(), false);
      sec(P.loops[j].inc[p].utgt.get(), false);
      sec(P.loops[j].inc[p].ut_off.get(), false);
      sec(P.loops[j].inc[p].slots.get(), false);
    }
  }
  for (int k = 0; k < H.n_ds; ++k)
    if (P.wflags[k].get()) s_wf[k] = (int)secs.size(), sec(P.wlist[k].get(), false);
  std::vector<int> s_ld(H.n_ds, -1);
  for (int k = 0; k < H.n_ds; ++k)
    if (H.ds[k].load == 2) s_ld[k] = (int)secs.size(), sec(P.llist[k].get(), false);
  const int s_dep = P.dataflow ? (int)secs.size() : -1;
  if (P.dataflow) sec(P.nbr.get(), false);
  std::vector<int32_t> hdr(H.hs);
  int n_exec = 0;
  P.scratch_base_host.assign(nt, 0);
  for (int t = 0; t < nt; ++t) {
    if (s->region[t] == LT_NONEXEC) continue;
    ++n_exec;
    int64_t cur = H.hs;
    auto put = [&](int si, int64_t src_off, int32_t len, int32_t sub) -> int32_t {
      Section &S = secs[si];
      S.src_off.push_back(src_off);
      S.dst_off.push_back(total + cur);
      S.len.push_back(len);
      S.sub.push_back(sub);
      const int32_t at = (int32_t)cur;
      cur += len;
      return at;
    };
    std::fill(hdr.begin(), hdr.end(), -1);
    for (int k = 0; k < H.n_sp; ++k) {
      const int32_t o = fps[k]->off_host[t], n = fps[k]->off_host[t + 1] - o;
      hdr[2 * k] = n;
      hdr[2 * k + 1] = put(s_sp[k], o, n, 0);
    }
    for (int j = 0; j < nl; ++j) {
      const LoopPlan &LP = P.loops[j];
      int32_t *h = &hdr[H.loop_pos[j]];
      const int32_t o = off[j][t], n = off[j][t + 1] - o;
      h[0] = n;
      // elements per chunk of this tile (per-tile for staged deferred loops)
      h[1] = LP.tile_chunk_host.empty() ? LP.chunk : LP.tile_chunk_host[t];
      const int nd = (int)cv.loops[j].desc.size();
      for (int d = 0; d < nd; ++d) {
        // descriptors with the same map (or all direct ones) share one slot map
        int same = -1;
        for (int e = 0; e < d && same < 0; ++e)
          if (cv.loops[j].desc[e].map == cv.loops[j].desc[d].map) same = e;
        if (same >= 0) {
          h[2 + d] = h[2 + same];
          continue;
        }
        const int ar = cv.loops[j].desc[d].map < 0 ? 1 : cv.maps[cv.loops[j].desc[d].map].arity;
        h[2 + d] = put(s_slot[j][d], (int64_t)o * ar, n * ar, 0);
      }
      for (size_t p = 0; p < LP.inc.size(); ++p) {
        const int32_t g0 = cb[j][t], nch = cb[j][t + 1] - g0;
        const int32_t U0 = gco[j][p][g0], U1 = gco[j][p][g0 + nch];
        const int32_t S0 = uto[j][p][U0], S1 = uto[j][p][U1];
        const int si = s_plan[j][p];
        int32_t *q = &h[2 + nd + 4 * p];
        q[0] = put(si, g0, nch + 1, U0);
        q[1] = put(si + 1, U0, U1 - U0, 0);
        q[2] = put(si + 2, U0, U1 - U0 + 1, S0);
        q[3] = put(si + 3, S0, S1 - S0, 0);
      }
    }
    for (int k = 0; k < H.n_ds; ++k) {
      hdr[H.ds_pos + 2 * k] = 0;
      if (s_wf[k] < 0) continue;
      const int32_t o = P.wbeg[k][t], n = P.wbeg[k][t + 1] - o;
      hdr[H.ds_pos + 2 * k] = n;
      hdr[H.ds_pos + 2 * k + 1] = put(s_wf[k], o, n, 0);
    }
    for (int k = 0; k < H.n_ds; ++k) {
      hdr[H.ld_pos + 2 * k] = 0;
      if (s_ld[k] < 0) continue;
      const int32_t o = P.lbeg[k][t], n = P.lbeg[k][t + 1] - o;
      hdr[H.ld_pos + 2 * k] = n;
      hdr[H.ld_pos + 2 * k + 1] = put(s_ld[k], o, n, 0);
    }
    hdr[H.dep_pos] = 0;
    if (s_dep >= 0) {
      const int32_t o = P.nbr_off_host[t], n = P.nbr_off_host[t + 1] - o;
      hdr[H.dep_pos] = n;
      hdr[H.dep_pos + 1] = put(s_dep, o, n, 0);
    }
    cur = (cur + 3) / 4 * 4;  // 16-byte aligned programs
    hdr[H.prog_pos] = (int32_t)cur;
    {  // row bases: read-only datasets first (packed behind the program), then the others
      int64_t acc = cur / 2;
      for (int pass = 1; pass >= 0; --pass)
        for (int k = 0; k < H.n_ds; ++k) {
          if (H.ds[k].ro != pass) continue;
          acc += acc & H.ds[k].vec;  // 16-byte aligned rows for pair copies
          if (H.ds[k].tma) acc = (acc + 15) & ~int64_t(15);  // 128-byte aligned for TMA
          hdr[H.base_pos + k] = (int32_t)acc;
          const auto &oh = fps[H.ds[k].sp]->off_host;
          acc += ds_rows(oh[t + 1] - oh[t], H.ds[k].tma) * H.ds[k].stride;
        }
      hdr[H.base_pos + H.n_ds] = (int32_t)acc;
      P.scratch_base_host[t] = (int32_t)acc;
    }
    {  // header section
      Section &S = secs[s_hdr];
      S.src_off.push_back((int64_t)hdr_host.size());
      S.dst_off.push_back(total);
      S.len.push_back(H.hs);
      S.sub.push_back(0);
      hdr_host.insert(hdr_host.end(), hdr.begin(), hdr.end());
    }
    blob_max = std::max(blob_max, (size_t)cur * 4);
    blen[t] = (int32_t)cur;
    if (H.ro_packed) {  // room for the read-only rows behind the program (k_pack_ro)
      int64_t acc = cur / 2;
      for (int k = 0; k < H.n_ds; ++k) {
        if (!H.ds[k].ro) continue;
        acc += acc & H.ds[k].vec;
        if (H.ds[k].tma) acc = (acc + 15) & ~int64_t(15);
        const auto &oh = fps[H.ds[k].sp]->off_host;
        acc += ds_rows(oh[t + 1] - oh[t], H.ds[k].tma) * H.ds[k].stride;
      }
      cur = (2 * acc + 3) / 4 * 4;
    }
    bfull[t] = (int32_t)cur;
    boff[t] = total;
    total += cur;
  }
  P.blob_off_host = boff;
  P.blob_len_host = blen;
  P.blob_full_host = bfull;
  P.blob.alloc(std::max<int64_t>(total, 4), ctx.stream);
  P.blob_off.alloc(nt, ctx.stream);
  P.blob_len.alloc(nt, ctx.stream);
  LT_CK(cudaMemcpyAsync(P.blob_off.get(), boff.data(), 8 * nt, cudaMemcpyHostToDevice, ctx.stream));
  LT_CK(cudaMemcpyAsync(P.blob_len.get(), blen.data(), 4 * nt, cudaMemcpyHostToDevice, ctx.stream));
  DevBuf<int32_t> hdr_dev(std::max<int64_t>((int64_t)hdr_host.size(), 1), ctx.stream);
  if (!hdr_host.empty())
    LT_CK(cudaMemcpyAsync(hdr_dev.get(), hdr_host.data(), 4 * hdr_host.size(),
                          cudaMemcpyHostToDevice, ctx.stream));
  secs[s_hdr].src = hdr_dev.get();
  for (Section &S : secs) {
    const int n = (int)S.len.size();
    if (n == 0) continue;
    DevBuf<int64_t> so(n, ctx.stream), dof(n, ctx.stream);
    DevBuf<int32_t> ln(n, ctx.stream), sb(n, ctx.stream);
    LT_CK(cudaMemcpyAsync(so.get(), S.src_off.data(), 8 * n, cudaMemcpyHostToDevice, ctx.stream));
    LT_CK(cudaMemcpyAsync(dof.get(), S.dst_off.data(), 8 * n, cudaMemcpyHostToDevice, ctx.stream));
    LT_CK(cudaMemcpyAsync(ln.get(), S.len.data(), 4 * n, cudaMemcpyHostToDevice, ctx.stream));
    LT_CK(cudaMemcpyAsync(sb.get(), S.sub.data(), 4 * n, cudaMemcpyHostToDevice, ctx.stream));
    const int grid = std::min(n, 65535);
    if (S.u8)
      k_seg_copy_u8<<<grid, 128, 0, ctx.stream>>>((const uint8_t *)S.src, so.get(), ln.get(),
                                                  P.blob.get(), dof.get(), n);
    else
      k_seg_copy<<<grid, 128, 0, ctx.stream>>>((const int32_t *)S.src, so.get(), ln.get(), sb.get(),
                                               P.blob.get(), dof.get(), n);
    LT_CK_LAUNCH();
    LT_CK(cudaStreamSynchronize(ctx.stream));
  }
  (void)n_exec;
  (void)ds_space;
  P.tile_blob = blen;
  return blob_max;
}

// ---- same-colour write conflicts -----------------------------------------------------
// Equal-coloured tiles must not share an element one of them writes.  The
// inspector guarantees it for complete chains, but the reference algorithm can
// emit schedules that break it (e.g. FIG2's sub-chain [edge_inc, cell_inc]:
// reductions of the last loop split over equal-coloured tiles -- 43 violations
// of the reference's own legality oracle; its sequential executor masks them).
// Such tiles are ordered into sub-colours in tile-id order, the reference's
// sequential order, so results stay bitwise equal to execute_schedule.
__global__ void k_conflict_keys(const int32_t *elem, const uint32_t *tile, int64_t n,
                                uint64_t flag, uint64_t *keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) keys[i] = ((uint64_t)(uint32_t)elem[i] << 32) | ((uint64_t)tile[i] << 1) | flag;
}

__global__ void k_conflict_pairs(const uint64_t *keys, int64_t n, const int32_t *color,
                                 PairSet ps) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || !(keys[i] & 1)) return;
  const uint64_t e = keys[i] >> 32;
  const int ti = (int)((keys[i] >> 1) & 0x7fffffff);
  for (int64_t j = i - 1; j >= 0 && (keys[j] >> 32) == e; --j) {
    const int tj = (int)((keys[j] >> 1) & 0x7fffffff);
    if (tj != ti && color[tj] == color[ti]) pair_insert(ps, ti, tj);
  }
  for (int64_t j = i + 1; j < n && (keys[j] >> 32) == e; ++j) {
    const int tj = (int)((keys[j] >> 1) & 0x7fffffff);
    if (tj != ti && color[tj] == color[ti]) pair_insert(ps, ti, tj);
  }
}

static void build_ranks(Ctx &ctx, lt_schedule *s, const ChainView &cv, ExecPlan &P) {
  const int nt = s->n_tiles;
  DevBuf<int32_t> region(nt, ctx.stream), color(nt, ctx.stream);
  LT_CK(cudaMemcpyAsync(region.get(), s->region.data(), 4 * nt, cudaMemcpyHostToDevice, ctx.stream));
  LT_CK(cudaMemcpyAsync(color.get(), s->color.data(), 4 * nt, cudaMemcpyHostToDevice, ctx.stream));
  std::map<int, std::vector<FpSource>> all, wr;
  for (int j = 0; j < s->n_loops; ++j) {
    const LoopDesc &L = cv.loops[j];
    std::vector<int> seen;
    bool direct = false, direct_w = false;
    for (const lt_desc &d : L.desc) {
      const bool w = d.mode != LT_READ;
      if (d.map < 0) {
        direct = true;
        direct_w |= w;
      } else {
        if (std::find(seen.begin(), seen.end(), d.map) == seen.end()) {
          seen.push_back(d.map);
          all[cv.maps[d.map].target].push_back({j, d.map});
        }
        if (w) wr[cv.maps[d.map].target].push_back({j, d.map});
      }
    }
    if (direct) all[L.space].push_back({j, -1});
    if (direct_w) wr[L.space].push_back({j, -1});
  }
  PairTable pt(ctx, pow2_at_least(int64_t(nt) * 16));
  for (;;) {
    for (auto &kv : wr) {
      Footprint fa, fw;
      build_footprint(ctx, s, cv, all[kv.first], region, fa);
      build_footprint(ctx, s, cv, kv.second, region, fw);
      const int64_t n = fa.n + fw.n;
      if (fw.n == 0) continue;
      DevBuf<uint64_t> k(n, ctx.stream), ks(n, ctx.stream);
      if (fa.n)
        k_conflict_keys<<<grid_for(fa.n, 256), 256, 0, ctx.stream>>>(fa.elem.get(), fa.tile.get(),
                                                                    fa.n, 0, k.get());
      k_conflict_keys<<<grid_for(fw.n, 256), 256, 0, ctx.stream>>>(fw.elem.get(), fw.tile.get(),
                                                                  fw.n, 1, k.get() + fa.n);
      LT_CK_LAUNCH();
      size_t tmp = 0;
      LT_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k.get(), ks.get(), (int)n, 0, 64,
                                           ctx.stream));
      DevBuf<char> tb((int64_t)tmp, ctx.stream);
      LT_CK(cub::DeviceRadixSort::SortKeys(tb.get(), tmp, k.get(), ks.get(), (int)n, 0, 64,
                                           ctx.stream));
      k_conflict_pairs<<<grid_for(n, 256), 256, 0, ctx.stream>>>(ks.get(), n, color.get(),
                                                                 pt.view());
      LT_CK_LAUNCH();
    }
    if (pt.status().second) { pt.resize(pt.cap * 2); continue; }
    break;
  }
  std::vector<std::vector<int>> lower(nt);  // conflicting tiles with a smaller id
  for (unsigned long long key : pt.fetch()) {
    const int a = (int)(key >> 32), b = (int)(key & 0xffffffffu);
    lower[std::max(a, b)].push_back(std::min(a, b));
  }
  std::vector<int32_t> sub(nt, 0);
  int max_sub = 0;
  for (int t = 0; t < nt; ++t)
    for (int u : lower[t]) {
      sub[t] = std::max(sub[t], sub[u] + 1);
      max_sub = std::max(max_sub, (int)sub[t]);
    }
  P.max_subcolor = max_sub;
  P.rank.resize(nt);
  for (int t = 0; t < nt; ++t) P.rank[t] = s->color[t] * (max_sub + 1) + sub[t];
}

// Which executor: LT_EXEC=global (tiles read global memory, one launch per
// colour), staged (footprints in shared memory, one launch per colour) or
// dataflow (staged, one persistent launch with tile dependencies).  Default:
// dataflow when the largest tile footprint fits shared memory, else global.
static int exec_preference() {
  const char *e = getenv("LT_EXEC");
  if (!e) return 0;
  if (!strcmp(e, "global")) return -1;
  if (!strcmp(e, "staged")) return 1;
  if (!strcmp(e, "dataflow")) return 2;
  return 0;
}

// Shared-memory rows of a staged dataset: odd stride (conflict-free 64-bit
// accesses) for odd vpe; for even vpe with 16-byte aligned data, 16-byte pair
// copies need an even stride, kept = 2 (mod 4) so 64-bit accesses conflict at
// most 2-way.
static bool ds_vec(int v, const double *p) {
  return v % 2 == 0 && reinterpret_cast<uintptr_t>(p) % 16 == 0;
}
// TMA gather4 datasets: 16-byte rows (vec), at most 256 doubles wide (TMA box
// limit); their shared rows are dense (stride = vpe, the layout gather4 writes)
// and the footprint is padded to a multiple of four rows.  LT_NO_TMA=1: the
// round-1 layout (stride = 2 mod 4 doubles) and cp.async gathers.
// A gather4 writes its four rows densely at the box width into 128-byte aligned
// shared memory: TMA rows are padded to a multiple of four doubles (box wider
// than the tensor; the extra columns are zero-filled) and every TMA dataset's
// rows start 128-byte aligned.  Only rows of >= 12 doubles (P2-P3 DoF rows),
// where the padding is at most two doubles.  Opt-in (LT_TMA=1): measured 7 %
// slower than the 128-thread cp.async gathers at configs 3 and 4 (rows of
// 96-240 bytes; one warp issues the gather4s after the dependency wait, where
// every thread issues its cp.async copies in parallel).
static bool ds_tma(int v, const double *p) {
  static const bool on = LT_TMA_GATHER && getenv("LT_TMA") && atoi(getenv("LT_TMA")) > 0;
  return on && ds_vec(v, p) && v >= 12 && v <= 256;
}
static int ds_stride(int v, bool vec, bool tma = false) {
  return tma ? (v + 3) & ~3 : vec ? (v % 4 == 2 ? v : v + 2) : (v | 1);
}
static int64_t ds_rows(int64_t n, bool tma) { return tma ? (n + 3) & ~int64_t(3) : n; }

#if LT_TMA_GATHER
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    LT_CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p)
      fail(LT_E_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// [rows x vpe] float64 rows as a 2-D tensor with a one-row box (tile::gather4
// fetches four rows of it per instruction)
static void row_tensor_map(CUtensorMap *m, const double *data, int64_t rows, int vpe,
                           int box_width) {
  const cuuint64_t dims[2] = {(cuuint64_t)vpe, (cuuint64_t)std::max<int64_t>(rows, 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)vpe * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)box_width, 1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(
      m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(data), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(LT_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

#endif  // LT_TMA_GATHER

// Footprints, slot maps and written flags of the staged executor.  Returns
// false (and leaves the plan untouched) when a footprint exceeds shared memory.
static bool build_stage(Ctx &ctx, lt_schedule *s, const ChainView &cv, const lt_arg *args,
                        ExecPlan &P, std::vector<int> &ds_of, std::vector<int> &ds_space,
                        std::vector<int> &ds_vpe, std::vector<double *> &ds_ptr,
                        size_t &regions_max) {
  const int nl = s->n_loops;
  if (nl > LT_MAX_SLOOPS) return false;
  // distinct datasets by device pointer
  int a = 0;
  for (int j = 0; j < nl; ++j) {
    for (size_t d = 0; d < cv.loops[j].desc.size(); ++d, ++a) {
      const lt_desc &D = cv.loops[j].desc[d];
      const int space = D.map < 0 ? cv.loops[j].space : cv.maps[D.map].target;
      int found = -1;
      for (size_t k = 0; k < ds_ptr.size(); ++k)
        if (ds_ptr[k] == args[a].values) found = (int)k;
      if (found < 0) {
        if ((int)ds_ptr.size() >= LT_MAX_STAGED) return false;
        found = (int)ds_ptr.size();
        ds_ptr.push_back(args[a].values);
        ds_space.push_back(space);
        ds_vpe.push_back(args[a].vpe);
      }
      ds_of.push_back(found);
    }
  }
  P.region.alloc(s->n_tiles, ctx.stream);
  LT_CK(cudaMemcpyAsync(P.region.get(), s->region.data(), sizeof(int32_t) * s->n_tiles,
                        cudaMemcpyHostToDevice, ctx.stream));
  // footprints per space touched by a dataset
  std::map<int, std::vector<FpSource>> sources;
  for (int j = 0; j < nl; ++j) {
    std::vector<int> seen;
    bool direct = false;
    for (const lt_desc &D : cv.loops[j].desc) {
      if (D.map < 0) {
        direct = true;
      } else if (std::find(seen.begin(), seen.end(), D.map) == seen.end()) {
        seen.push_back(D.map);
        sources[cv.maps[D.map].target].push_back({j, D.map});
      }
    }
    if (direct) sources[cv.loops[j].space].push_back({j, -1});
  }
  if (sources.size() > LT_MAX_SPACES) return false;
  for (size_t k = 0; k < ds_ptr.size(); ++k)  // 32-bit row offsets in the gather/store-back
    if ((uint64_t)cv.total(ds_space[k]) * (uint64_t)ds_vpe[k] >= (1ull << 32)) return false;
  for (auto &kv : sources) build_footprint(ctx, s, cv, kv.second, P.region, P.fp[kv.first]);
  P.ds_bytes = 0;
  for (size_t k = 0; k < ds_ptr.size(); ++k)
    P.ds_bytes += (size_t)cv.total(ds_space[k]) * (size_t)ds_vpe[k] * sizeof(double);
  // shared-memory regions of the largest tile: footprint ids + dataset rows
  regions_max = 0;
  P.tile_rows.assign(s->n_tiles, 0);
  for (int t = 0; t < s->n_tiles; ++t) {
    if (s->region[t] == LT_NONEXEC) continue;
    size_t r = 0;
    for (size_t k = 0; k < ds_ptr.size(); ++k) {
      const auto &oh = P.fp[ds_space[k]].off_host;
      const bool tma = ds_tma(ds_vpe[k], ds_ptr[k]);
      r += (size_t)ds_rows(oh[t + 1] - oh[t], tma) *
               ds_stride(ds_vpe[k], ds_vec(ds_vpe[k], ds_ptr[k]), tma) + (tma ? 16 : 1);
    }
    regions_max = std::max(regions_max, r * sizeof(double));
    P.tile_rows[t] = r * sizeof(double);
  }
  P.data_max = regions_max;
  return regions_max + 16 * 1024 <= kSmemMax;
}

// LT_DEBUG_PLAN=1: shared-memory composition and per-tile size percentiles
static void print_plan_stats(const lt_schedule *s, const ExecPlan &P, size_t blob_max,
                             size_t scratch_max) {
  std::vector<size_t> rows, blob, tot;
  for (int t = 0; t < s->n_tiles; ++t) {
    if (s->region[t] == LT_NONEXEC) continue;
    rows.push_back(P.tile_rows[t]);
    blob.push_back(4 * (size_t)P.tile_blob[t]);
    tot.push_back(P.tile_rows[t] + 4 * (size_t)P.tile_blob[t]);
  }
  auto pct = [](std::vector<size_t> v, double q) -> size_t {
    if (v.empty()) return 0;
    std::sort(v.begin(), v.end());
    return v[std::min(v.size() - 1, (size_t)(q * (double)v.size()))];
  };
  fprintf(stderr, "[lt plan] tiles %zu smem %zu = blob_max %zu + rows_max %zu + scratch %zu\n",
          rows.size(), P.smem_bytes, blob_max, P.data_max, scratch_max);
  const char *nm[3] = {"rows", "blob", "rows+blob"};
  const std::vector<size_t> *vv[3] = {&rows, &blob, &tot};
  for (int i = 0; i < 3; ++i)
    fprintf(stderr, "[lt plan]   %-9s p50 %zu p90 %zu p99 %zu max %zu\n", nm[i], pct(*vv[i], 0.5),
            pct(*vv[i], 0.9), pct(*vv[i], 0.99), pct(*vv[i], 1.0));
  for (int j = 0; j < s->n_loops; ++j)
    fprintf(stderr, "[lt plan]   loop %d chunk %d scratch/pos %d deferred %d nobar %d\n", j,
            P.loops[j].chunk, P.loops[j].scratch_per_pos, (int)P.loops[j].deferred,
            (int)P.host_loops[j].nobar);
}

// Rows that need no gather: a dataset whose first access in the chain is a
// direct WRITE by a kernel that writes every component ("DF") gets, per tile,
// the list of its footprint rows that loop does *not* write; only those are
// gathered (load == 2).  DG: the volume loop writes ru, rs of the tile's
// cells, so only rows other tiles' cells contribute to are loaded.
__global__ void k_clear_slots(const int32_t *elements, const int32_t *sigma, int64_t n,
                              const int32_t *fp_off, const int32_t *slot, uint8_t *flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || slot[i] < 0) return;
  flag[fp_off[sigma[elements[i]]] + slot[i]] = 0;
}

static void build_load_lists(Ctx &ctx, lt_schedule *s, const ChainView &cv, ExecPlan &P,
                             const std::vector<int> &ds_of, const std::vector<int> &ds_space) {
  StagedParams &H = P.sp;
  const int nl = s->n_loops;
  P.llist.resize(H.n_ds);
  P.lbeg.resize(H.n_ds);
  for (int k = 0; k < H.n_ds; ++k) {
    if (H.ds[k].ro || getenv("LT_LOAD_ALL")) continue;
    int j0 = -1, d0 = -1, hits = 0;
    for (int j = 0, q = 0; j < nl && j0 < 0; ++j) {
      for (size_t d = 0; d < cv.loops[j].desc.size(); ++d)
        if (ds_of[q + d] == k) {
          ++hits;
          if (d0 < 0) d0 = (int)d;
        }
      if (hits) j0 = j;
      q += (int)cv.loops[j].desc.size();
    }
    if (j0 < 0 || hits != 1) continue;
    const lt_desc &D = cv.loops[j0].desc[d0];
    const char *tok = kSpecs[cv.loops[j0].kernel].sig + 3 * d0;
    if (D.map >= 0 || D.mode != LT_WRITE || tok[1] != 'F') continue;
    const Footprint &fp = P.fp.at(ds_space[k]);
    const int64_t n = fp.n;
    DevBuf<uint8_t> flag(std::max<int64_t>(n, 1), ctx.stream);
    LT_CK(cudaMemsetAsync(flag.get(), 1, std::max<int64_t>(n, 1), ctx.stream));
    const LoopLists &Lj = s->lists[j0];
    if (Lj.n)
      k_clear_slots<<<grid_for(Lj.n, 256), 256, 0, ctx.stream>>>(
          Lj.elements.get(), Lj.sigma.get(), Lj.n, fp.off.get(), P.loops[j0].slots[d0].get(),
          flag.get());
    LT_CK_LAUNCH();
    DevBuf<int32_t> f32(std::max<int64_t>(n, 1), ctx.stream), scan(n + 1, ctx.stream);
    int64_t cnt = 0;
    if (n) {
      k_u8_to_i32<<<grid_for(n, 256), 256, 0, ctx.stream>>>(flag.get(), n, f32.get());
      LT_CK_LAUNCH();
      exclusive_sum(ctx, f32.get(), scan.get(), n);
      cnt = last_plus(ctx, scan.get(), f32.get(), n);
    }
    k_set_int<<<1, 1, 0, ctx.stream>>>(scan.get() + n, (int32_t)cnt);
    LT_CK_LAUNCH();
    P.llist[k].alloc(std::max<int64_t>(cnt, 1), ctx.stream);
    if (n) {
      k_compact_written<<<grid_for(n, 256), 256, 0, ctx.stream>>>(
          flag.get(), scan.get(), fp.tile.get(), fp.off.get(), n, P.llist[k].get());
      LT_CK_LAUNCH();
    }
    DevBuf<int32_t> lb(s->n_tiles + 1, ctx.stream);
    k_gather_at<<<grid_for(s->n_tiles + 1, 256), 256, 0, ctx.stream>>>(scan.get(), fp.off.get(),
                                                                       s->n_tiles + 1, lb.get());
    LT_CK_LAUNCH();
    to_host(ctx, lb, s->n_tiles + 1, P.lbeg[k]);
    LT_CK(cudaStreamSynchronize(ctx.stream));
    H.ds[k].load = 2;
  }
}

// scratch_override > 0: record budget for the deferred (DG facet) loops, chunks
// not rounded to warps (second planning pass, see plan_with_occupancy)
static std::shared_ptr<ExecPlan> build_plan(Ctx &ctx, lt_schedule *s, const ChainView &cv,
                                            const lt_arg *args, int use_local,
                                            bool force_global = false,
                                            size_t scratch_override = 0,
                                            const std::vector<int64_t> *tile_budget = nullptr) {
  auto plan = std::make_shared<ExecPlan>();
  ExecPlan &P = *plan;
  const int nl = s->n_loops;
  P.loops.resize(nl);
  P.host_loops.resize(nl);
  build_ranks(ctx, s, cv, P);
  std::vector<int> ds_of, ds_space, ds_vpe;
  std::vector<double *> ds_ptr;
  size_t regions_max = 0;
  const int pref = force_global ? -1 : exec_preference();
  if (pref >= 0) {
    P.staged = build_stage(ctx, s, cv, args, P, ds_of, ds_space, ds_vpe, ds_ptr, regions_max);
    if (!P.staged && pref > 0)
      fail(LT_E_EXECUTION, "LT_EXEC=staged/dataflow: tile footprint rows " +
                               std::to_string(P.data_max) + " B exceed shared memory");
    if (!P.staged) P.fp.clear();
    P.dataflow = P.staged && pref != 1;
  }
  const int block = P.staged ? LT_SBLOCK : LT_BLOCK;
  const size_t budget = P.staged ? std::min<size_t>(scratch_override ? scratch_override
                                                                     : scratch_budget(),
                                                    kSmemMax - regions_max)
                                 : kSmemBudget;
  size_t scratch_max = 0;
  int a = 0;
  for (int j = 0; j < nl; ++j) {
    const LoopDesc &L = cv.loops[j];
    LoopPlan &LP = P.loops[j];
    DLoop &D = P.host_loops[j];
    fill_dloop(D, cv, j, args + a, ctx, use_local);
    if (P.staged && D.deferred) D.rec = dg_corr_size_staged(L.kernel - K_DG_FIRST);
    int spp = 0;
    for (int d = 0; d < D.n_desc; ++d) {
      if (L.desc[d].map < 0 || L.desc[d].mode == LT_READ) continue;
      D.a[d].inc_off = spp;  // scaled by chunk below
      spp += D.a[d].arity * D.a[d].vpe;
      LP.inc_desc.push_back(d);
    }
    // DG facet loops keep per-side correction records (5 NQ + 2 doubles)
    // instead of lifted increments (5 ND each)
    LP.deferred = D.deferred;
    if (D.deferred) spp = D.a[4].arity * D.rec;
    LP.scratch_per_pos = spp;
    // staged deferred loops: the whole budget (a chunk is one records phase
    // and one apply phase; fewer chunks, fewer phases per tile)
    LP.chunk = choose_chunk(spp, budget, block, !(P.staged && D.deferred && scratch_override));
    if (spp) {  // no larger than the longest tile list of the loop (scratch is per CTA)
      std::vector<int32_t> off(s->n_tiles + 1);
      LT_CK(cudaMemcpyAsync(off.data(), s->lists[j].offsets.get(), 4 * (s->n_tiles + 1),
                            cudaMemcpyDeviceToHost, ctx.stream));
      LT_CK(cudaStreamSynchronize(ctx.stream));
      int longest = 1;
      for (int t = 0; t < s->n_tiles; ++t) longest = std::max(longest, off[t + 1] - off[t]);
      LP.chunk = std::min(LP.chunk, longest);
    }
    for (int d : LP.inc_desc) D.a[d].inc_off *= LP.chunk;
    scratch_max = std::max(scratch_max, sizeof(double) * (size_t)LP.scratch_per_pos * LP.chunk);
    D.chunk = LP.chunk;
    const LoopLists &Lj = s->lists[j];
    D.offsets = Lj.offsets.get();
    D.elements = Lj.elements.get();
    if (use_local && !P.staged) {
      for (int d = 0; d < D.n_desc; ++d) {
        if (L.desc[d].map < 0) continue;
        auto it = s->local_maps.find(std::make_pair(j, (int)L.desc[d].map));
        if (it == s->local_maps.end()) fail(LT_E_EXECUTION, "schedule lacks local maps");
        D.a[d].lmap = it->second.get();
      }
    }
    if (P.staged) {
      LP.slots.resize(D.n_desc);
      for (int d = 0; d < D.n_desc; ++d) {
        const lt_desc &X = L.desc[d];
        const int ar = X.map < 0 ? 1 : cv.maps[X.map].arity;
        const int space = X.map < 0 ? L.space : cv.maps[X.map].target;
        const Footprint &fp = P.fp.at(space);
        LP.slots[d].alloc(std::max<int64_t>(Lj.n * ar, 1), ctx.stream);
        if (Lj.n)
          k_slots<<<grid_for(Lj.n * ar, 256), 256, 0, ctx.stream>>>(
              Lj.elements.get(), Lj.sigma.get(), X.map < 0 ? nullptr : cv.maps[X.map].values, ar,
              Lj.n, P.region.get(), fp.off.get(), fp.elem.get(), LP.slots[d].get());
        LT_CK_LAUNCH();
        D.a[d].slot = LP.slots[d].get();
        D.a[d].ds = ds_of[a + d];
        D.a[d].sstride = ds_stride(D.a[d].vpe, ds_vec(D.a[d].vpe, D.a[d].data),
                                   ds_tma(D.a[d].vpe, D.a[d].data));
      }
    }
    if (!LP.inc_desc.empty()) {
      std::vector<int32_t> off(s->n_tiles + 1);
      LT_CK(cudaMemcpyAsync(off.data(), Lj.offsets.get(), sizeof(int32_t) * (s->n_tiles + 1),
                            cudaMemcpyDeviceToHost, ctx.stream));
      LT_CK(cudaStreamSynchronize(ctx.stream));
      std::vector<int32_t> cb(s->n_tiles + 1, 0);
      if (P.staged && D.deferred && tile_budget) {
        // per-tile chunks: a tile's scratch starts right behind its own rows, so a
        // tile smaller than the largest one has room for longer chunks (fewer
        // records + apply phases); never shorter than the uniform chunk
        LP.tile_chunk_host.resize(s->n_tiles);
        for (int t = 0; t < s->n_tiles; ++t) {
          const int len = off[t + 1] - off[t];
          const int64_t fit = (*tile_budget)[t] / (int64_t)(sizeof(double) * LP.scratch_per_pos);
          LP.tile_chunk_host[t] =
              (int32_t)std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(fit, LP.chunk),
                                                            std::max(len, 1)));
        }
        LP.tile_chunk.alloc(s->n_tiles, ctx.stream);
        LT_CK(cudaMemcpyAsync(LP.tile_chunk.get(), LP.tile_chunk_host.data(),
                              sizeof(int32_t) * s->n_tiles, cudaMemcpyHostToDevice, ctx.stream));
      }
      for (int t = 0; t < s->n_tiles; ++t) {
        const int ch = LP.tile_chunk_host.empty() ? LP.chunk : LP.tile_chunk_host[t];
        cb[t + 1] = cb[t] + (off[t + 1] - off[t] + ch - 1) / ch;
      }
      LP.chunk_base.alloc(s->n_tiles + 1, ctx.stream);
      LT_CK(cudaMemcpyAsync(LP.chunk_base.get(), cb.data(), sizeof(int32_t) * cb.size(),
                            cudaMemcpyHostToDevice, ctx.stream));
      if (P.staged) {
        std::vector<int32_t> gct(std::max<int32_t>(cb.back(), 1), 0);
        for (int t = 0; t < s->n_tiles; ++t)
          for (int g = cb[t]; g < cb[t + 1]; ++g) gct[g] = t;
        LP.gc_tile.alloc((int64_t)gct.size(), ctx.stream);
        LT_CK(cudaMemcpyAsync(LP.gc_tile.get(), gct.data(), sizeof(int32_t) * gct.size(),
                              cudaMemcpyHostToDevice, ctx.stream));
      }
      D.chunk_base = LP.chunk_base.get();
      // one ordered-gather plan per distinct map (e.g. ru and rs through if2c share one)
      for (size_t i = 0; i < LP.inc_desc.size(); ++i) {
        const int m = L.desc[LP.inc_desc[i]].map;
        if (std::find(LP.plan_map.begin(), LP.plan_map.end(), m) == LP.plan_map.end())
          LP.plan_map.push_back(m);
      }
      LP.inc.resize(LP.plan_map.size());
      for (size_t p = 0; p < LP.plan_map.size(); ++p) {
        const lt_map &mp = cv.maps[LP.plan_map[p]];
        build_inc_plan(ctx, s, j, mp, LP.chunk, cb, LP.chunk_base, LP.inc[p],
                       P.staged ? &P.fp.at(mp.target) : nullptr,
                       P.staged ? &LP.gc_tile : nullptr, LP.tile_chunk.get());
      }
      for (size_t i = 0; i < LP.inc_desc.size(); ++i) {
        const int d = LP.inc_desc[i];
        const int p = (int)(std::find(LP.plan_map.begin(), LP.plan_map.end(), L.desc[d].map) -
                            LP.plan_map.begin());
        IncPlan &IP = D.inc[i];
        IP.desc = d;
        IP.plan = p;
        IP.gc_off = LP.inc[p].gc_off.get();
        IP.utgt = LP.inc[p].utgt.get();
        IP.ut_off = LP.inc[p].ut_off.get();
        IP.slots = LP.inc[p].slots.get();
      }
      D.n_inc = (int)LP.inc_desc.size();
      D.n_plans = (int)LP.plan_map.size();
    }
    a += D.n_desc;
  }
  if (P.staged) {
    // written flags per staged dataset; a dataset needs no load when its first
    // access in the chain is a direct WRITE over exactly the rows it writes
    StagedParams &H = P.sp;
    std::memset(&H, 0, sizeof(H));
    H.n_loops = nl;
    H.n_ds = (int)ds_ptr.size();
    std::map<int, int> sp_index;
    for (auto &kv : P.fp) {
      const int k = (int)sp_index.size();
      sp_index[kv.first] = k;
    }
    H.n_sp = (int)sp_index.size();
    P.wflags.resize(ds_ptr.size());
    for (size_t k = 0; k < ds_ptr.size(); ++k) {
      H.ds[k].data = ds_ptr[k];
      H.ds[k].vpe = ds_vpe[k];
      H.ds[k].vec = ds_vec(ds_vpe[k], ds_ptr[k]) ? 1 : 0;
      H.ds[k].tma = ds_tma(ds_vpe[k], ds_ptr[k]) ? 1 : 0;
      H.ds[k].stride = ds_stride(ds_vpe[k], H.ds[k].vec, H.ds[k].tma);
#if LT_TMA_GATHER
      if (H.ds[k].tma)
        row_tensor_map(&H.tmap[k], ds_ptr[k], cv.total(ds_space[k]), ds_vpe[k], H.ds[k].stride);
#endif
      const int unit = H.ds[k].vec ? ds_vpe[k] / 2 : ds_vpe[k];  // pairs or doubles per row
      H.ds[k].di = LT_SBLOCK / unit;
      H.ds[k].dc = LT_SBLOCK % unit;
      H.ds[k].magic = lt_magic(unit);
      H.ds[k].sp = sp_index.at(ds_space[k]);
      H.ds[k].load = 1;
      H.ds[k].ro = 1;
    }
    for (int j = 0, q = 0; j < nl; ++j)
      for (size_t d = 0; d < cv.loops[j].desc.size(); ++d, ++q)
        if (cv.loops[j].desc[d].mode != LT_READ) H.ds[ds_of[q]].ro = 0;
    // dataflow: blobs leave room for the read-only rows of every tile behind
    // its program; repeated executions pack them there (k_pack_ro, once per
    // call) so they arrive with the program in one bulk copy.  H.ro_packed
    // marks the plan packable; each launch sets it for its own parameters.
    H.ro_packed = 0;
    if (P.dataflow)
      for (int k = 0; k < H.n_ds; ++k) H.ro_packed |= H.ds[k].ro;
    a = 0;
    for (int j = 0; j < nl; ++j) {
      const LoopDesc &L = cv.loops[j];
      const LoopLists &Lj = s->lists[j];
      for (size_t d = 0; d < L.desc.size(); ++d) {
        const int k = ds_of[a + d];
        if (L.desc[d].mode == LT_READ) continue;
        if (!P.wflags[k].get()) {
          const Footprint &fp = P.fp.at(ds_space[k]);
          P.wflags[k].alloc(std::max<int64_t>(fp.off_host.back(), 1), ctx.stream);
          LT_CK(cudaMemsetAsync(P.wflags[k].get(), 0, P.wflags[k].n, ctx.stream));
          H.ds[k].written = 1;
        }
        const int ar = L.desc[d].map < 0 ? 1 : cv.maps[L.desc[d].map].arity;
        if (Lj.n)
          k_mark_written<<<grid_for(Lj.n * ar, 256), 256, 0, ctx.stream>>>(
              Lj.elements.get(), Lj.sigma.get(), ar, Lj.n, P.fp.at(ds_space[k]).off.get(),
              P.loops[j].slots[d].get(), P.wflags[k].get());
        LT_CK_LAUNCH();
      }
      a += (int)L.desc.size();
    }
    // written rows per dataset as compact tile-local lists (store-back work items)
    P.wlist.resize(ds_ptr.size());
    P.wbeg.resize(ds_ptr.size());
    for (size_t k = 0; k < ds_ptr.size(); ++k) {
      if (!P.wflags[k].get()) continue;
      const Footprint &fp = P.fp.at(ds_space[k]);
      const int64_t n = fp.n;
      DevBuf<int32_t> f32(std::max<int64_t>(n, 1), ctx.stream), scan(n + 1, ctx.stream);
      int64_t cnt = 0;
      if (n) {
        k_u8_to_i32<<<grid_for(n, 256), 256, 0, ctx.stream>>>(P.wflags[k].get(), n, f32.get());
        LT_CK_LAUNCH();
        exclusive_sum(ctx, f32.get(), scan.get(), n);
        cnt = last_plus(ctx, scan.get(), f32.get(), n);
      }
      k_set_int<<<1, 1, 0, ctx.stream>>>(scan.get() + n, (int32_t)cnt);
      LT_CK_LAUNCH();
      P.wlist[k].alloc(std::max<int64_t>(cnt, 1), ctx.stream);
      if (n) {
        k_compact_written<<<grid_for(n, 256), 256, 0, ctx.stream>>>(
            P.wflags[k].get(), scan.get(), fp.tile.get(), fp.off.get(), n, P.wlist[k].get());
        LT_CK_LAUNCH();
      }
      DevBuf<int32_t> wb(s->n_tiles + 1, ctx.stream);
      k_gather_at<<<grid_for(s->n_tiles + 1, 256), 256, 0, ctx.stream>>>(scan.get(), fp.off.get(),
                                                                         s->n_tiles + 1, wb.get());
      LT_CK_LAUNCH();
      to_host(ctx, wb, s->n_tiles + 1, P.wbeg[k]);
      LT_CK(cudaStreamSynchronize(ctx.stream));
    }
    build_load_lists(ctx, s, cv, P, ds_of, ds_space);
    H.n_gather = H.n_store = 0;
#if LT_TMA_GATHER
    H.n_tma = 0;
#endif
    for (int k = 0; k < H.n_ds; ++k) {
      if (!H.ds[k].ro && H.ds[k].load) H.gather_ds[H.n_gather++] = (int8_t)k;
      if (H.ds[k].written) H.store_ds[H.n_store++] = (int8_t)k;
#if LT_TMA_GATHER
      if (!H.ds[k].ro && H.ds[k].load == 1 && H.ds[k].tma) ++H.n_tma;
#endif
    }
    for (int j = 0; j + 1 < nl; ++j)
      P.host_loops[j].nobar = barrier_free_pair(ctx, s, cv, args, j);
    for (int j = 0; j < nl; ++j) H.loops[j] = P.host_loops[j];
    if (P.dataflow) build_dependencies(ctx, s, P);  // tile programs carry the lists
    const size_t blob_max = build_blobs(ctx, s, cv, P, sp_index, ds_space);
    H.blob = P.blob.get();
    H.blob_off = P.blob_off.get();
    H.blob_len = P.blob_len.get();
    if (blob_max + P.data_max + scratch_max + kAlignSlack > kSmemMax) {  // caller falls back
      g_last_fit = "tile program " + std::to_string(blob_max) + " B + rows " +
                   std::to_string(P.data_max) + " B + scratch " + std::to_string(scratch_max) +
                   " B > " + std::to_string(kSmemMax) + " B";
      return nullptr;
    }
    P.smem_bytes = blob_max + P.data_max + scratch_max + kAlignSlack;  // + lt_align128 slack
    P.scratch_bytes = scratch_max;
    if (tile_budget) {  // per-tile chunks: the largest (rows + own scratch) of any tile
      size_t need = 0;
      for (int t = 0; t < s->n_tiles; ++t) {
        if (s->region[t] == LT_NONEXEC) continue;
        size_t sc = 0;
        for (int j = 0; j < nl; ++j) {
          const LoopPlan &LP = P.loops[j];
          const int ch = LP.tile_chunk_host.empty() ? LP.chunk : LP.tile_chunk_host[t];
          sc = std::max(sc, sizeof(double) * (size_t)LP.scratch_per_pos * ch);
        }
        need = std::max(need, sizeof(double) * (size_t)P.scratch_base_host[t] + sc);
      }
      if (need + kAlignSlack > kSmemMax) return nullptr;
      P.smem_bytes = need + kAlignSlack;
    }
    if (const char *pad = getenv("LT_SMEM_PAD_KB"))  // diagnostics: force lower occupancy
      P.smem_bytes = std::min(kSmemMax, P.smem_bytes + 1024 * (size_t)atoi(pad));
    if (getenv("LT_DEBUG_PLAN")) print_plan_stats(s, P, blob_max, scratch_max);
  } else {
    P.smem_bytes = scratch_max;
  }
  P.dloops.alloc(nl, ctx.stream);
  LT_CK(cudaMemcpyAsync(P.dloops.get(), P.host_loops.data(), sizeof(DLoop) * nl,
                        cudaMemcpyHostToDevice, ctx.stream));
  // colour phases: core tiles by ascending colour, then boundary tiles
  for (int reg : {LT_CORE, LT_BOUNDARY}) {
    std::map<int, std::vector<int32_t>> by_color;
    for (int t = 0; t < s->n_tiles; ++t)
      if (s->region[t] == reg) by_color[P.rank[t]].push_back(t);
    for (auto &kv : by_color) {
      DevBuf<int32_t> ids((int64_t)kv.second.size(), ctx.stream);
      LT_CK(cudaMemcpyAsync(ids.get(), kv.second.data(), sizeof(int32_t) * kv.second.size(),
                            cudaMemcpyHostToDevice, ctx.stream));
      P.phases.emplace_back((int)kv.second.size(), std::move(ids));
      P.phase_region.push_back(reg);
      P.phase_color.push_back(kv.first);
    }
  }
  LT_CK(cudaStreamSynchronize(ctx.stream));
  return plan;
}

// Mirror the volume kernels' operator tables into the constant bank (field-lane
// volume items read them as instruction operands).  Device-to-device on the
// execution stream before every launch: in-place parameter updates and captured
// graphs see current values.  One mirror per degree and process: contexts that
// run the same degree with different tables must not execute concurrently.
static void refresh_const_tables(Ctx &ctx, const ExecPlan &P) {
  for (const DLoop &L : P.host_loops) {
    const int k = L.kernel - K_DG_FIRST;
    if (k < 0 || k % 5 != 0 || !L.params) continue;
    const int p = k / 5 + 1, nd = dg_nd(p);
    const size_t bytes = sizeof(double) * 2 * nd * nd;
    const void *sym = p == 1   ? (const void *)c_dg_vol_p1
                      : p == 2 ? (const void *)c_dg_vol_p2
                      : p == 3 ? (const void *)c_dg_vol_p3
                               : (const void *)c_dg_vol_p4;
    LT_CK(cudaMemcpyToSymbolAsync(sym, L.params, bytes, 0, cudaMemcpyDeviceToDevice,
                                  ctx.stream));
  }
}

typedef void (*StagedFn)(const StagedParams, const int32_t *);
static StagedFn staged_fn(int fam) {
  switch (fam) {
    case 0: return k_staged_tiles<0>;
    case 1: return k_staged_tiles<1>;
    case 2: return k_staged_tiles<2>;
    case 3: return k_staged_tiles<3>;
    case 4: return k_staged_tiles<4>;
    default: return k_staged_tiles<5>;
  }
}

typedef void (*DataflowFn)(const StagedParams, const DataflowArgs);
#ifndef LT_WIDE_MINB
// CTAs per SM of the wide build (128 registers at 128 threads): measured in
// round 2 against the 168-register <= 3 CTAs/SM build, 4 CTAs/SM at a smaller
// seed tile win (config 3 ts 16: 13.56 vs 13.94 ms at ts 24; config 4 cut
// ts 12: 44.6 vs 45.6 ms at ts 16)
#define LT_WIDE_MINB 4
#endif
#ifndef LT_NARROW_MINB
#define LT_NARROW_MINB 6  // CTAs per SM of the narrow (80-register at 128 threads) build
#endif
static DataflowFn dataflow_fn(int fam, bool wide = false) {
  if (wide) switch (fam) {
      case 1: return k_dataflow<1, LT_WIDE_MINB>;
      case 2: return k_dataflow<2, LT_WIDE_MINB>;
      case 3: return k_dataflow<3, LT_WIDE_MINB>;
      case 4: return k_dataflow<4, LT_WIDE_MINB>;
      default: break;
    }
  switch (fam) {
    case 0: return k_dataflow<0, LT_NARROW_MINB>;
    case 1: return k_dataflow<1, LT_NARROW_MINB>;
    case 2: return k_dataflow<2, LT_NARROW_MINB>;
    case 3: return k_dataflow<3, LT_NARROW_MINB>;
    case 4: return k_dataflow<4, LT_NARROW_MINB>;
    default: return k_dataflow<5, LT_NARROW_MINB>;
  }
}

#ifndef LT_PASS2_MIN
#define LT_PASS2_MIN 1024   // re-plan only for at least this much more record scratch
#endif
#ifndef LT_PASS2_SLACK
#define LT_PASS2_SLACK 1024  // left for the longer chunks' apply plans in the tile programs
#endif
// CTAs per SM of the dataflow build that would run a plan with this much
// shared memory (the wide build when <= LT_WIDE_MINB fit, as in execute_tiled)
static int dataflow_occupancy(int fam, size_t smem) {
  auto occ = [&](const void *fn) {
    int per_sm = 0;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess) {
      cudaGetLastError();  // beyond the kernel's limit (static shared memory included)
      return 0;
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, LT_SBLOCK, smem) !=
        cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return per_sm;
  };
  int per_sm = occ((const void *)dataflow_fn(fam, false));
  if (per_sm <= LT_WIDE_MINB && fam >= 1 && fam <= 4 && !getenv("LT_NARROW"))
    per_sm = occ((const void *)dataflow_fn(fam, true));
  return per_sm;
}

// Two planning passes for DG chains on the dataflow executor: the first with
// the default record budget fixes the CTAs per SM the tile programs allow;
// the second gives the facet loops' correction records all shared memory that
// keeps that occupancy (bigger chunks: fewer records + ordered-apply phases
// per tile).  Config 3: 14.66 -> ~14.1 ms; config 2: one chunk per tile.
static std::shared_ptr<ExecPlan> plan_with_occupancy(Ctx &ctx, lt_schedule *s,
                                                     const ChainView &cv, const lt_arg *args,
                                                     int use_local) {
  auto plan = build_plan(ctx, s, cv, args, use_local);
  if (!plan || !plan->dataflow || getenv("LT_SCRATCH_KB")) return plan;
  bool deferred = false;
  for (const LoopPlan &LP : plan->loops) deferred |= LP.deferred;
  if (!deferred) return plan;
  const int fam = chain_family(cv);
  const int occ = dataflow_occupancy(fam, plan->smem_bytes);
  const size_t fixed = plan->smem_bytes - plan->scratch_bytes;
  size_t best = plan->scratch_bytes;
  for (size_t sc = kSmemMax - 1024 - fixed; sc > plan->scratch_bytes + 512; sc -= 256)
    if (dataflow_occupancy(fam, fixed + sc) >= occ) {
      best = sc;
      break;
    }
  if (getenv("LT_UNIFORM_CHUNKS")) {  // round-1/2 behaviour: one chunk size for all tiles
    if (best < plan->scratch_bytes + LT_PASS2_MIN) return plan;
    // the blob grows slightly with longer chunks' plans: leave 1 KB of slack
    auto p2 = build_plan(ctx, s, cv, args, use_local, false, best - LT_PASS2_SLACK);
    if (p2 && p2->dataflow && dataflow_occupancy(fam, p2->smem_bytes) >= occ) return p2;
    return plan;
  }
  // per-tile chunks.  A tile's scratch begins behind its own program and rows,
  // so every tile smaller than the largest can hold longer chunks in the same
  // CTA allocation (half the tiles of a 2-timestep DG chain need under half the
  // shared memory of the largest); the largest tiles get what the uniform
  // second pass would have given them
  for (const LoopPlan &LP : plan->loops)
    if (LP.scratch_per_pos && !LP.deferred) return plan;  // uniform inc_off scaling
  const size_t target = fixed + best;
  std::vector<int64_t> tile_budget(s->n_tiles, 0);
  for (int t = 0; t < s->n_tiles; ++t)
    tile_budget[t] = (int64_t)target - (int64_t)kAlignSlack - 256 -
                     (int64_t)sizeof(double) * plan->scratch_base_host[t];
  auto p3 = build_plan(ctx, s, cv, args, use_local, false, plan->scratch_bytes, &tile_budget);
  if (p3 && p3->dataflow && dataflow_occupancy(fam, p3->smem_bytes) >= occ) return p3;
  return plan;
}

// dry: build the plan and queue items, report what a call would launch, and
// launch nothing (lt_prepare: plan building without touching the datasets)
static void execute_tiled(Ctx &ctx, lt_schedule *s, const ChainView &cv, const lt_arg *args,
                          int phases, int use_local, int repeats, lt_exec_info *info,
                          bool dry = false) {
  if ((int)cv.loops.size() != s->n_loops)
    fail(LT_E_STALE_SCHEDULE, "schedule loop count differs from chain");
  for (int j = 0; j < s->n_loops; ++j)
    if (s->loop_space[j] != cv.loops[j].space || s->lists[j].n != cv.total(cv.loops[j].space))
      fail(LT_E_STALE_SCHEDULE, "schedule was inspected for a different chain");
  if (repeats < 1) fail(LT_E_VALUE, "repeats must be >= 1");
  if (repeats > 1 && phases != (LT_PHASE_CORE | LT_PHASE_BOUNDARY))
    fail(LT_E_VALUE, "repeated execution needs both phases (no halo exchange in between)");
  validate_bindings(ctx, cv, args);
  const std::string key = plan_key(ctx, cv, args, use_local) + std::to_string(exec_preference());
  if (!s->plan || s->plan->key != key) {
    s->plan = plan_with_occupancy(ctx, s, cv, args, use_local);
    if (!s->plan) {  // tile programs do not fit shared memory
      if (exec_preference() > 0)
        fail(LT_E_EXECUTION, "LT_EXEC=staged/dataflow: " + g_last_fit);
      s->plan = build_plan(ctx, s, cv, args, use_local, true);
    }
    s->plan->key = key;
  }
  ExecPlan &P = *s->plan;
  const int fam = chain_family(cv);
  if (P.dataflow && P.grid == 0) {
    // register budget: the 80-register build reaches 6 CTAs per SM; when the
    // tile programs' shared memory allows at most 3, the 168-register build
    // costs no occupancy and spills nothing
    int per_sm = 0, sms = 0;
    const void *narrow = (const void *)dataflow_fn(fam, false);
    if (P.smem_bytes > 48 * 1024)
      LT_CK(cudaFuncSetAttribute(narrow, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)P.smem_bytes));
    LT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, narrow, LT_SBLOCK, P.smem_bytes));
    P.wide = per_sm <= LT_WIDE_MINB && fam >= 1 && fam <= 4 && !getenv("LT_NARROW");
    if (P.wide) {
      const void *w = (const void *)dataflow_fn(fam, true);
      if (P.smem_bytes > 48 * 1024)
        LT_CK(cudaFuncSetAttribute(w, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)P.smem_bytes));
      LT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, w, LT_SBLOCK, P.smem_bytes));
    }
    LT_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx.device));
    P.grid = std::max(1, per_sm) * sms;
    if (getenv("LT_DEBUG_PLAN"))
      fprintf(stderr, "[lt plan] dataflow %s build, %d CTAs/SM, grid %d\n",
              P.wide ? "wide" : "narrow", per_sm, P.grid);
  }
  const void *fn = P.dataflow  ? (const void *)dataflow_fn(fam, P.wide)
                   : P.staged ? (const void *)staged_fn(fam)
                              : (const void *)fused_fn(fam);
  if (P.smem_bytes > 48 * 1024)
    LT_CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)P.smem_bytes));
  int launches = 0, colors = 0;
  int64_t visits = 0;
  if (P.dataflow) {
    const bool core = phases & LT_PHASE_CORE, bnd = phases & LT_PHASE_BOUNDARY;
    DataflowArgs D;
    D.order = core && bnd ? P.order_all.get() : core ? P.order_core.get() : P.order_bnd.get();
    D.n_exec = core && bnd ? P.n_all : core ? P.n_core : P.n_bnd;
    D.n_items = D.n_exec * repeats;
    {
      const int kind = core && bnd ? 0 : core ? 1 : 2;
      if (!P.items.count({kind, repeats})) build_items(ctx, P, kind, repeats, P.ds_bytes);
      auto &its = P.items.at({kind, repeats});
      D.item_tk = its.tk.get();
      D.item_ol = its.ol.get();
      if (info) {
        info->wave_order = P.items_wave.at({kind, repeats});
        info->wide_build = P.wide ? 1 : 0;
      }
    }
    D.done = P.done.get();
    D.queue = P.queue.get();
    // a boundary-only call continues the counters of the core-only call that
    // must directly precede it (its core dependencies are complete); its own
    // tiles' counters restart at zero so overlapping boundary tiles still wait
    if (!core && !dry && P.last_call != 1)
      fail(LT_E_EXECUTION, "dataflow: a boundary-only execution must directly follow the "
                           "core-only execution of the same schedule");
    StagedParams sp = P.sp;
    sp.ro_packed = pack_for(P, repeats);
    if (dry) {
      launches = (D.n_items > 0) * (1 + (int)sp.ro_packed);
    } else {
    if (core)
      LT_CK(cudaMemsetAsync(P.done.get(), 0, 4 * P.done.n, ctx.stream));
    else if (P.n_bnd > 0) {
      k_zero_at<<<grid_for(P.n_bnd, 256), 256, 0, ctx.stream>>>(P.done.get(), P.order_bnd.get(),
                                                               P.n_bnd);
      LT_CK_LAUNCH();
    }
    P.last_call = core && bnd ? 0 : core ? 1 : 2;
    LT_CK(cudaMemsetAsync(P.queue.get(), 0, 4, ctx.stream));
    // packing costs one pass over the read-only rows: it pays when every tile
    // runs more than once in this call
    if (D.n_items > 0 && sp.ro_packed) {
      k_pack_ro<<<std::min(D.n_exec, 16 * 148), 256, 0, ctx.stream>>>(sp, D.order, D.n_exec);
      LT_CK_LAUNCH();
      ++launches;
    }
    if (D.n_items > 0) {
      refresh_const_tables(ctx, P);
      dataflow_fn(fam, P.wide)<<<std::min(P.grid, D.n_items), LT_SBLOCK, P.smem_bytes, ctx.stream>>>(
          sp, D);
      LT_CK_LAUNCH();
      ++launches;
    }
    }
    colors = (int)P.phases.size();
  } else {
    if (P.staged && !dry) refresh_const_tables(ctx, P);
    for (int r = 0; r < repeats; ++r) {
      for (size_t ph = 0; ph < P.phases.size(); ++ph) {
        const int reg = P.phase_region[ph];
        if (!((reg == LT_CORE && (phases & LT_PHASE_CORE)) ||
              (reg == LT_BOUNDARY && (phases & LT_PHASE_BOUNDARY))))
          continue;
        if (dry)
          ;
        else if (P.staged)
          staged_fn(fam)<<<P.phases[ph].first, LT_SBLOCK, P.smem_bytes, ctx.stream>>>(
              P.sp, P.phases[ph].second.get());
        else
          fused_fn(fam)<<<P.phases[ph].first, LT_BLOCK, P.smem_bytes, ctx.stream>>>(
              P.dloops.get(), s->n_loops, P.phases[ph].second.get());
        if (!dry) LT_CK_LAUNCH();
        ++launches;
        if (r == 0) ++colors;
      }
    }
  }
  for (int j = 0; j < s->n_loops; ++j) visits += cv.exec_size(cv.loops[j].space) * repeats;
  if (info) {
    info->launches = launches;
    info->n_colors = colors;
    info->elements = visits;
    info->staged = P.dataflow ? 2 : P.staged ? 1 : 0;
    info->smem_bytes = (int32_t)P.smem_bytes;
  }
}

// inverse maps for the untiled executor, cached per device map buffer
struct InvKey {
  const int32_t *values;
  int64_t n_source, n_target;
  int arity;
  bool operator<(const InvKey &o) const {
    return std::tie(values, n_source, n_target, arity) <
           std::tie(o.values, o.n_source, o.n_target, o.arity);
  }
};
struct InvVal {
  DevBuf<int32_t> off, flat;
};
static std::map<std::pair<Ctx *, InvKey>, InvVal> g_inverse_cache;

static InvVal &cached_inverse(Ctx &ctx, const lt_map &mp, int64_t ns, int64_t nt) {
  auto key = std::make_pair(&ctx, InvKey{mp.values, ns, nt, mp.arity});
  auto it = g_inverse_cache.find(key);
  if (it != g_inverse_cache.end()) return it->second;
  InvVal v;
  v.off.alloc(nt + 1, ctx.stream);
  v.flat.alloc(ns * mp.arity, ctx.stream);
  invert_flat(ctx, mp.values, ns, mp.arity, nt, v.off.get(), v.flat.get());
  return g_inverse_cache.emplace(key, std::move(v)).first->second;
}

void forget_map(Ctx *ctx, const int32_t *values) {
  for (auto it = g_inverse_cache.begin(); it != g_inverse_cache.end();) {
    if ((ctx == nullptr || it->first.first == ctx) && it->first.second.values == values)
      it = g_inverse_cache.erase(it);
    else
      ++it;
  }
}

void forget_ctx(Ctx *ctx) {
  for (auto it = g_inverse_cache.begin(); it != g_inverse_cache.end();)
    it = (it->first.first == ctx) ? g_inverse_cache.erase(it) : std::next(it);
}

static void execute_untiled(Ctx &ctx, const ChainView &cv, const lt_arg *args,
                            lt_exec_info *info) {
  validate_bindings(ctx, cv, args);
  int a = 0, launches = 0;
  int64_t visits = 0;
  std::vector<DevBuf<double>> scratch;
  DevBuf<DLoop> dl((int64_t)cv.loops.size(), ctx.stream);
  std::vector<DLoop> host(cv.loops.size());
  for (size_t j = 0; j < cv.loops.size(); ++j) {
    const LoopDesc &L = cv.loops[j];
    DLoop &D = host[j];
    fill_dloop(D, cv, (int)j, args + a, ctx, 0);
    const int64_t n = cv.exec_size(L.space);
    if (D.deferred) {  // one correction record per (element, k)
      scratch.emplace_back(std::max<int64_t>(n * D.a[4].arity * D.rec, 1), ctx.stream);
      D.a[4].scr = scratch.back().get();
    } else {
      for (int d = 0; d < D.n_desc; ++d) {
        if (L.desc[d].map < 0 || L.desc[d].mode == LT_READ) continue;
        scratch.emplace_back(std::max<int64_t>(n * D.a[d].arity * D.a[d].vpe, 1), ctx.stream);
        D.a[d].scr = scratch.back().get();
      }
    }
    a += D.n_desc;
  }
  LT_CK(cudaMemcpyAsync(dl.get(), host.data(), sizeof(DLoop) * host.size(),
                        cudaMemcpyHostToDevice, ctx.stream));
  UntiledFn ufn = untiled_fn(chain_family(cv));
  for (size_t j = 0; j < cv.loops.size(); ++j) {
    const LoopDesc &L = cv.loops[j];
    const int64_t n = cv.exec_size(L.space);
    visits += n;
    if (n == 0) continue;
    ufn<<<grid_for(n * host[j].lanes, 256), 256, 0, ctx.stream>>>(dl.get() + j, (int)n);
    LT_CK_LAUNCH();
    ++launches;
    if (host[j].deferred) {
      const lt_map &mp = cv.maps[L.desc[4].map];
      const int64_t nt = cv.total(mp.target);
      InvVal &inv = cached_inverse(ctx, mp, cv.total(mp.source), nt);
      const int64_t work = nt * (host[j].a[4].vpe >> 1);
      if (work) {
        untiled_deferred_fn(chain_family(cv))<<<grid_for(work, 256), 256, 0, ctx.stream>>>(
            dl.get() + j, inv.off.get(), inv.flat.get(), nt, (int)n);
        LT_CK_LAUNCH();
        ++launches;
      }
      continue;
    }
    for (int d = 0; d < (int)L.desc.size(); ++d) {
      if (L.desc[d].map < 0 || L.desc[d].mode == LT_READ) continue;
      const lt_map &mp = cv.maps[L.desc[d].map];
      const int64_t nt = cv.total(mp.target);
      InvVal &inv = cached_inverse(ctx, mp, cv.total(mp.source), nt);
      const int64_t work = nt * host[j].a[d].vpe;
      if (work == 0) continue;
      k_untiled_apply<<<grid_for(work, 256), 256, 0, ctx.stream>>>(
          dl.get() + j, d, inv.off.get(), inv.flat.get(), nt, (int)n);
      LT_CK_LAUNCH();
      ++launches;
    }
  }
  if (info) {
    info->launches = launches;
    info->n_colors = 0;
    info->elements = visits;
  }
}

}  // namespace lt

using namespace lt;

lt_schedule::~lt_schedule() {}

extern "C" int lt_kernel_lookup(const char *name, int32_t *kernel_id, int32_t *nargs) {
  LT_API_BEGIN
  if (!name) fail(LT_E_VALUE, "null name");
  for (int i = 0; i < kNumKernels; ++i) {
    if (std::strcmp(kSpecs[i].name, name) == 0) {
      if (kernel_id) *kernel_id = i;
      if (nargs) *nargs = sig_count(kSpecs[i].sig);
      return LT_OK;
    }
  }
  fail(LT_E_EXECUTION, std::string("kernel '") + name + "' is not a native kernel");
  LT_API_END
}

extern "C" int lt_kernel_count(void) { return kNumKernels; }

#ifdef LT_PHASE_TIMING
extern "C" int lt_phase_cycles(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 64);
  if (reset) {
    static unsigned long long zero[64] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, zero, sizeof(zero));
  }
  return 0;
}
#endif

extern "C" const char *lt_kernel_name(int32_t id) {
  return (id >= 0 && id < kNumKernels) ? kSpecs[id].name : nullptr;
}

extern "C" int lt_execute(lt_ctx *ctx, lt_schedule *s, const lt_chain *chain, const lt_arg *args,
                          int32_t phases, int32_t use_local_maps, lt_exec_info *info) {
  LT_API_BEGIN
  if (!ctx || !s || !chain || !args) fail(LT_E_VALUE, "null argument");
  ChainView cv(chain);
  execute_tiled(*ctx, s, cv, args, phases, use_local_maps ? 1 : 0, 1, info);
  LT_API_END
}

extern "C" int lt_execute_repeat(lt_ctx *ctx, lt_schedule *s, const lt_chain *chain,
                                 const lt_arg *args, int32_t repeats, int32_t use_local_maps,
                                 lt_exec_info *info) {
  LT_API_BEGIN
  if (!ctx || !s || !chain || !args) fail(LT_E_VALUE, "null argument");
  ChainView cv(chain);
  execute_tiled(*ctx, s, cv, args, LT_PHASE_CORE | LT_PHASE_BOUNDARY, use_local_maps ? 1 : 0,
                repeats, info);
  LT_API_END
}

extern "C" int lt_prepare(lt_ctx *ctx, lt_schedule *s, const lt_chain *chain,
                          const lt_arg *args, int32_t phases, int32_t repeats,
                          int32_t use_local_maps, lt_exec_info *info) {
  LT_API_BEGIN
  if (!ctx || !s || !chain || !args) fail(LT_E_VALUE, "null argument");
  ChainView cv(chain);
  execute_tiled(*ctx, s, cv, args, phases, use_local_maps ? 1 : 0, repeats, info, true);
  LT_API_END
}

extern "C" int lt_execute_untiled(lt_ctx *ctx, const lt_chain *chain, const lt_arg *args,
                                  lt_exec_info *info) {
  LT_API_BEGIN
  if (!ctx || !chain || !args) fail(LT_E_VALUE, "null argument");
  ChainView cv(chain);
  execute_untiled(*ctx, cv, args, info);
  LT_API_END
}
