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

#include <algorithm>
#include <cstring>
#include <tuple>

#include "lt_dg.cuh"
#include "lt_kernels.cuh"

namespace lt {

// ---- kernel table -------------------------------------------------------------
// signature tokens per descriptor: D* direct any, DR direct read, DW direct
// write/rw, MR mapped read, MI mapped inc (or write)
struct KernelSpec {
  const char *name;
  const char *sig;
};

static const KernelSpec kSpecs[] = {
    {"edge_inc", "D*,MI"},  {"cell_inc", "D*,MI"},  {"edge_read", "DW,MR"},
    {"cell_read", "DW,MR"}, {"toy_k1", "D*,MI"},    {"toy_k2", "DW,MR"},
    {"toy_k3", "DW,MR"},
#define LT_DG_SPEC(P)                                                                  \
  {"dg_vol_p" #P, "DR,DR,DR,DR,DW,DW"}, {"dg_iflux_p" #P, "DR,MR,MR,MR,MI,MI"},        \
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
};

struct FlatCtx {  // untiled: element ids, global scratch
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
};

// FAM selects which DG degree is compiled into an instantiation (0: scalar
// kernels only, 1..4: scalar + DG P, 5: everything) so a P1 chain does not
// pay the register footprint of P4 bodies.
template <int FAM, class C>
__device__ __forceinline__ void dispatch(int kernel, C &c) {
  switch (kernel) {
    case K_EDGE_INC: body_edge_inc(c); break;
    case K_CELL_INC: body_edge_inc(c); break;  // same body: every target += own value
    case K_EDGE_READ: body_sum_read(c); break;
    case K_CELL_READ: body_sum_read(c); break;
    case K_TOY_K1: body_toy_k1(c); break;
    case K_TOY_K2: body_toy_k2(c); break;
    case K_TOY_K3: body_toy_k3(c); break;
    default:
      if (FAM > 0) dg_dispatch<FAM>(kernel - K_DG_FIRST, c);
      break;
  }
}

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
      const int lp = threadIdx.x;
      if (lp < CH && c0 + lp < n) {
        const int gpos = beg + c0 + lp;
        TileCtx cx{L, L.elements[gpos], gpos, lp, smem};
        dispatch<FAM>(L.kernel, cx);
      }
      if (L.n_inc) {
        __syncthreads();
        const int gc = L.chunk_base[t] + c0 / CH;
        for (int i = 0; i < L.n_inc; ++i) apply_chunk(L, L.inc[i], gc, smem);
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

// ---- untiled executor --------------------------------------------------------------
template <int FAM>
__global__ void __launch_bounds__(256) k_untiled_body(const DLoop *__restrict__ Lp, int n) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const DLoop &L = *Lp;
  FlatCtx cx{L, e};
  dispatch<FAM>(L.kernel, cx);
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

// ---- plan building -------------------------------------------------------------------
__global__ void k_inc_keys(const int32_t *elements, const int32_t *sigma, const int32_t *offsets,
                           const int32_t *chunk_base, const int32_t *map, int arity, int CH,
                           int64_t n, uint64_t *keys, int32_t *vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * arity) return;
  const int64_t p = i / arity;
  const int k = (int)(i - p * arity);
  const int e = elements[p];
  const int t = sigma[e];
  const int pos = (int)(p - offsets[t]);
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
};

struct LoopPlan {
  int chunk = LT_BLOCK;
  int scratch_per_pos = 0;  // doubles
  DevBuf<int32_t> chunk_base;
  std::vector<IncBuffers> inc;
  std::vector<int> inc_desc;
};

struct ExecPlan {
  std::string key;
  std::vector<LoopPlan> loops;
  std::vector<std::pair<int, DevBuf<int32_t>>> phases;  // (#tiles, tile ids) per colour phase
  std::vector<int> phase_region;
  std::vector<int> phase_color;
  DevBuf<DLoop> dloops;
  std::vector<DLoop> host_loops;
  size_t smem_bytes = 0;
};

static int choose_chunk(int scratch_per_pos, size_t smem_budget) {
  if (scratch_per_pos == 0) return LT_BLOCK;
  int ch = (int)(smem_budget / (sizeof(double) * (size_t)scratch_per_pos));
  ch = std::min(ch, LT_BLOCK);
  if (ch >= 32) ch -= ch % 32;
  if (ch < 1) fail(LT_E_EXECUTION, "loop contributions exceed shared memory");
  return ch;
}

static void build_inc_plan(Ctx &ctx, const lt_schedule *s, int j, const lt_map &mp, int CH,
                           const std::vector<int32_t> &chunk_base_host,
                           const DevBuf<int32_t> &chunk_base, IncBuffers &out) {
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
      CH, n, kin.get(), vin.get());
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
  DevBuf<uint32_t> run_gc(R, ctx.stream);
  k_run_fill<<<grid_for(nnz, 256), 256, 0, ctx.stream>>>(kout.get(), heads.get(), run_idx.get(),
                                                         nnz, out.utgt.get(), out.ut_off.get(),
                                                         run_gc.get());
  LT_CK_LAUNCH();
  k_set_int<<<1, 1, 0, ctx.stream>>>(out.ut_off.get() + R, (int32_t)nnz);
  LT_CK_LAUNCH();
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
      if (p[1] == 'W' && D.mode != LT_WRITE && D.mode != LT_RW)
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

static std::string plan_key(const ChainView &cv, const lt_arg *args, int use_local) {
  std::string k = std::to_string(use_local) + "|";
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

static std::shared_ptr<ExecPlan> build_plan(Ctx &ctx, lt_schedule *s, const ChainView &cv,
                                            const lt_arg *args, int use_local) {
  auto plan = std::make_shared<ExecPlan>();
  const int nl = s->n_loops;
  plan->loops.resize(nl);
  plan->host_loops.resize(nl);
  int a = 0;
  for (int j = 0; j < nl; ++j) {
    const LoopDesc &L = cv.loops[j];
    LoopPlan &P = plan->loops[j];
    DLoop &D = plan->host_loops[j];
    fill_dloop(D, cv, j, args + a, ctx, use_local);
    int spp = 0;
    for (int d = 0; d < D.n_desc; ++d) {
      if (L.desc[d].map < 0 || L.desc[d].mode == LT_READ) continue;
      D.a[d].inc_off = spp;  // scaled by chunk below
      spp += D.a[d].arity * D.a[d].vpe;
      P.inc_desc.push_back(d);
    }
    P.scratch_per_pos = spp;
    P.chunk = choose_chunk(spp, kSmemBudget);
    for (int d : P.inc_desc) D.a[d].inc_off *= P.chunk;
    plan->smem_bytes = std::max(plan->smem_bytes, sizeof(double) * (size_t)spp * P.chunk);
    D.chunk = P.chunk;
    D.offsets = s->lists[j].offsets.get();
    D.elements = s->lists[j].elements.get();
    if (use_local) {
      for (int d = 0; d < D.n_desc; ++d) {
        if (L.desc[d].map < 0) continue;
        auto it = s->local_maps.find(std::make_pair(j, (int)L.desc[d].map));
        if (it == s->local_maps.end()) fail(LT_E_EXECUTION, "schedule lacks local maps");
        D.a[d].lmap = it->second.get();
      }
    }
    if (!P.inc_desc.empty()) {
      std::vector<int32_t> off(s->n_tiles + 1);
      LT_CK(cudaMemcpyAsync(off.data(), s->lists[j].offsets.get(),
                            sizeof(int32_t) * (s->n_tiles + 1), cudaMemcpyDeviceToHost,
                            ctx.stream));
      LT_CK(cudaStreamSynchronize(ctx.stream));
      std::vector<int32_t> cb(s->n_tiles + 1, 0);
      for (int t = 0; t < s->n_tiles; ++t)
        cb[t + 1] = cb[t] + (off[t + 1] - off[t] + P.chunk - 1) / P.chunk;
      P.chunk_base.alloc(s->n_tiles + 1, ctx.stream);
      LT_CK(cudaMemcpyAsync(P.chunk_base.get(), cb.data(), sizeof(int32_t) * cb.size(),
                            cudaMemcpyHostToDevice, ctx.stream));
      D.chunk_base = P.chunk_base.get();
      P.inc.resize(P.inc_desc.size());
      for (size_t i = 0; i < P.inc_desc.size(); ++i) {
        const int d = P.inc_desc[i];
        build_inc_plan(ctx, s, j, cv.maps[L.desc[d].map], P.chunk, cb, P.chunk_base, P.inc[i]);
        IncPlan &IP = D.inc[i];
        IP.desc = d;
        IP.gc_off = P.inc[i].gc_off.get();
        IP.utgt = P.inc[i].utgt.get();
        IP.ut_off = P.inc[i].ut_off.get();
        IP.slots = P.inc[i].slots.get();
      }
      D.n_inc = (int)P.inc_desc.size();
    }
    a += D.n_desc;
  }
  plan->dloops.alloc(nl, ctx.stream);
  LT_CK(cudaMemcpyAsync(plan->dloops.get(), plan->host_loops.data(), sizeof(DLoop) * nl,
                        cudaMemcpyHostToDevice, ctx.stream));
  // colour phases: core tiles by ascending colour, then boundary tiles
  for (int reg : {LT_CORE, LT_BOUNDARY}) {
    std::map<int, std::vector<int32_t>> by_color;
    for (int t = 0; t < s->n_tiles; ++t)
      if (s->region[t] == reg) by_color[s->color[t]].push_back(t);
    for (auto &kv : by_color) {
      DevBuf<int32_t> ids((int64_t)kv.second.size(), ctx.stream);
      LT_CK(cudaMemcpyAsync(ids.get(), kv.second.data(), sizeof(int32_t) * kv.second.size(),
                            cudaMemcpyHostToDevice, ctx.stream));
      plan->phases.emplace_back((int)kv.second.size(), std::move(ids));
      plan->phase_region.push_back(reg);
      plan->phase_color.push_back(kv.first);
    }
  }
  LT_CK(cudaStreamSynchronize(ctx.stream));
  return plan;
}

static void execute_tiled(Ctx &ctx, lt_schedule *s, const ChainView &cv, const lt_arg *args,
                          int phases, int use_local, lt_exec_info *info) {
  if ((int)cv.loops.size() != s->n_loops)
    fail(LT_E_STALE_SCHEDULE, "schedule loop count differs from chain");
  for (int j = 0; j < s->n_loops; ++j)
    if (s->loop_space[j] != cv.loops[j].space || s->lists[j].n != cv.total(cv.loops[j].space))
      fail(LT_E_STALE_SCHEDULE, "schedule was inspected for a different chain");
  validate_bindings(ctx, cv, args);
  const std::string key = plan_key(cv, args, use_local);
  if (!s->plan || s->plan->key != key) {
    s->plan = build_plan(ctx, s, cv, args, use_local);
    s->plan->key = key;
  }
  ExecPlan &P = *s->plan;
  FusedFn fn = fused_fn(chain_family(cv));
  if (P.smem_bytes > 48 * 1024)
    LT_CK(cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)P.smem_bytes));
  int launches = 0, colors = 0;
  int64_t visits = 0;
  for (size_t ph = 0; ph < P.phases.size(); ++ph) {
    const int reg = P.phase_region[ph];
    if (!((reg == LT_CORE && (phases & LT_PHASE_CORE)) ||
          (reg == LT_BOUNDARY && (phases & LT_PHASE_BOUNDARY))))
      continue;
    fn<<<P.phases[ph].first, LT_BLOCK, P.smem_bytes, ctx.stream>>>(
        P.dloops.get(), s->n_loops, P.phases[ph].second.get());
    LT_CK_LAUNCH();
    ++launches;
    ++colors;
  }
  for (int j = 0; j < s->n_loops; ++j) visits += cv.exec_size(cv.loops[j].space);
  if (info) {
    info->launches = launches;
    info->n_colors = colors;
    info->elements = visits;
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
    for (int d = 0; d < D.n_desc; ++d) {
      if (L.desc[d].map < 0 || L.desc[d].mode == LT_READ) continue;
      scratch.emplace_back(std::max<int64_t>(n * D.a[d].arity * D.a[d].vpe, 1), ctx.stream);
      D.a[d].scr = scratch.back().get();
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
    ufn<<<grid_for(n, 256), 256, 0, ctx.stream>>>(dl.get() + j, (int)n);
    LT_CK_LAUNCH();
    ++launches;
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

extern "C" const char *lt_kernel_name(int32_t id) {
  return (id >= 0 && id < kNumKernels) ? kSpecs[id].name : nullptr;
}

extern "C" int lt_execute(lt_ctx *ctx, lt_schedule *s, const lt_chain *chain, const lt_arg *args,
                          int32_t phases, int32_t use_local_maps, lt_exec_info *info) {
  LT_API_BEGIN
  if (!ctx || !s || !chain || !args) fail(LT_E_VALUE, "null argument");
  ChainView cv(chain);
  execute_tiled(*ctx, s, cv, args, phases, use_local_maps ? 1 : 0, info);
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
