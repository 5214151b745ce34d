// lt_legality.cu — GPU restatement of the reference's brute-force legality
// oracle (pkg/tests/legality.py:15-151), for schedules of any size.
//
// Reference rule (legality.py check_legality):
//  * cross-loop pairs: for loops x < y and elements e_x, e_y touching the same
//    (space, element) key -- flow (x writes, y reads), anti (x reads, y
//    writes) or output (both write), increments counted as writes, and not
//    both accesses direct (legality.py:44-63) -- the tile running e_y must be
//    the tile running e_x or have a strictly higher colour;
//  * reductions: two distinct elements of one loop incrementing the same key
//    through a map may not run in distinct tiles of equal colour.
// Pairs involving the non-exec tile (or no tile) are skipped; only
// executable elements are visited (legality.py:35-41).
//
// GPU formulation: one record per (loop, executable element, descriptor,
// arity slot) keyed by (target space, target element, loop, direct), radix
// sorted; one thread per target key walks its records (O(run^2), runs are a
// few dozen long) and appends every violating pair to a bounded buffer; the
// host de-duplicates pairs (the reference counts a set of pairs).
#include <cub/cub.cuh>

#include <set>
#include <tuple>

#include "lt_internal.cuh"

namespace lt {

namespace {

constexpr int kSpaceBits = 4, kElemBits = 31, kLoopBits = 7;
constexpr int kKeyLo = 1 + kLoopBits;  // direct bit + loop below the target

struct LegLoop {
  const int32_t *sigma;  // tile of each element of the loop's space
  int64_t exec;          // executable elements
  int space;
};

struct LegDesc {
  const int32_t *map;  // nullptr: direct
  int loop, arity, target_space, mode;
  int64_t base;        // first record of this descriptor
};

__global__ void k_leg_records(const LegDesc *ds, int n_desc, const LegLoop *loops,
                              int64_t total, uint64_t *keys, uint64_t *vals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < total;
       r += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = n_desc - 1;  // descriptor of record r (bases ascending)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ds[mid].base <= r) lo = mid; else hi = mid - 1;
    }
    const LegDesc &D = ds[lo];
    const int64_t off = r - D.base;
    const int64_t e = off / D.arity;
    const int k = (int)(off % D.arity);
    const int64_t tgt = D.map ? D.map[e * D.arity + k] : e;
    const int space = D.map ? D.target_space : loops[D.loop].space;
    keys[r] = ((uint64_t)space << (kElemBits + kKeyLo)) | ((uint64_t)tgt << kKeyLo) |
              ((uint64_t)D.loop << 1) | (D.map ? 0u : 1u);
    const unsigned rd = D.mode == LT_READ, wr = !rd, inc = D.map && D.mode == LT_INC;
    vals[r] = ((uint64_t)e << 3) | (rd << 0) | (wr << 1) | (inc << 2);
  }
}

__global__ void k_leg_heads(const uint64_t *keys, int64_t n, int32_t *heads) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) heads[i] = (i == 0 || (keys[i] >> kKeyLo) != (keys[i - 1] >> kKeyLo)) ? 1 : 0;
}

__global__ void k_leg_starts(const int32_t *heads, const int32_t *idx, int64_t n, int64_t *start) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && heads[i]) start[idx[i]] = i;
}

struct Viol {
  int32_t kind, x, ex, y, ey;  // kind 0: cross-loop pair; 1: reduction (x = loop, ex < ey)
};

__global__ void k_leg_scan(const uint64_t *keys, const uint64_t *vals, const int64_t *start,
                           int64_t n_runs, int64_t n, const LegLoop *loops, const int32_t *color,
                           int tne, Viol *out, int cap, unsigned long long *count) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_runs;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = start[g], b = g + 1 < n_runs ? start[g + 1] : n;
    for (int64_t j = a; j < b; ++j) {
      const int ly = (int)((keys[j] >> 1) & ((1u << kLoopBits) - 1));
      const bool dy = keys[j] & 1;
      const int ey = (int)(vals[j] >> 3);
      const unsigned fy = (unsigned)(vals[j] & 7);
      const int ty = loops[ly].sigma[ey];
      if (ty < 0 || ty == tne) continue;
      for (int64_t i = a; i < j; ++i) {
        const int lx = (int)((keys[i] >> 1) & ((1u << kLoopBits) - 1));
        const bool dx = keys[i] & 1;
        const int ex = (int)(vals[i] >> 3);
        const unsigned fx = (unsigned)(vals[i] & 7);
        const int tx = loops[lx].sigma[ex];
        if (tx < 0 || tx == tne) continue;
        if (lx < ly) {
          const bool dep = ((fx & 2) && (fy & 1)) || ((fx & 1) && (fy & 2)) ||
                           ((fx & 2) && (fy & 2));
          if (!dep || (dx && dy)) continue;
          if (tx == ty || color[ty] > color[tx]) continue;
          const unsigned long long at = atomicAdd(count, 1ull);
          if (at < (unsigned long long)cap) out[at] = Viol{0, lx, ex, ly, ey};
        } else if (lx == ly && (fx & 4) && (fy & 4) && ex != ey && tx != ty &&
                   color[tx] == color[ty]) {
          const unsigned long long at = atomicAdd(count, 1ull);
          if (at < (unsigned long long)cap)
            out[at] = Viol{1, lx, ex < ey ? ex : ey, lx, ex < ey ? ey : ex};
        }
      }
    }
  }
}

}  // namespace

}  // namespace lt

using namespace lt;

extern "C" int lt_check_legality(lt_ctx *ctx, const lt_schedule *s, const lt_chain *chain,
                                 int64_t *n_pairs, int64_t *n_reductions, int32_t *overflow) {
  LT_API_BEGIN
  if (!ctx || !s || !chain || !n_pairs || !n_reductions) fail(LT_E_VALUE, "null argument");
  ChainView cv(chain);
  if ((int)cv.loops.size() != s->n_loops)
    fail(LT_E_STALE_SCHEDULE, "schedule loop count differs from chain");
  if ((int)cv.loops.size() >= (1 << kLoopBits) || (int)cv.spaces.size() >= (1 << kSpaceBits))
    fail(LT_E_VALUE, "legality check: too many loops or spaces");
  std::vector<LegLoop> hl(cv.loops.size());
  std::vector<LegDesc> hd;
  int64_t total = 0;
  for (size_t j = 0; j < cv.loops.size(); ++j) {
    const LoopDesc &L = cv.loops[j];
    if (cv.total(L.space) >= (1ll << kElemBits)) fail(LT_E_VALUE, "legality check: space too large");
    hl[j] = LegLoop{s->lists[j].sigma.get(), cv.exec_size(L.space), L.space};
    for (const lt_desc &d : L.desc) {
      LegDesc D{};
      D.map = d.map < 0 ? nullptr : cv.maps[d.map].values;
      D.loop = (int)j;
      D.arity = d.map < 0 ? 1 : cv.maps[d.map].arity;
      D.target_space = d.map < 0 ? L.space : cv.maps[d.map].target;
      D.mode = d.mode;
      D.base = total;
      total += hl[j].exec * D.arity;
      if (hl[j].exec > 0) hd.push_back(D);
    }
  }
  *n_pairs = *n_reductions = 0;
  if (overflow) *overflow = 0;
  if (total == 0) return LT_OK;
  if (total >= (1ll << 31)) fail(LT_E_VALUE, "legality check: too many accesses");
  cudaStream_t st = ctx->stream;
  DevBuf<LegLoop> dl((int64_t)hl.size(), st);
  DevBuf<LegDesc> dd((int64_t)hd.size(), st);
  DevBuf<int32_t> dcolor(s->n_tiles, st);
  LT_CK(cudaMemcpyAsync(dl.get(), hl.data(), sizeof(LegLoop) * hl.size(), cudaMemcpyHostToDevice, st));
  LT_CK(cudaMemcpyAsync(dd.get(), hd.data(), sizeof(LegDesc) * hd.size(), cudaMemcpyHostToDevice, st));
  LT_CK(cudaMemcpyAsync(dcolor.get(), s->color.data(), 4 * s->n_tiles, cudaMemcpyHostToDevice, st));
  DevBuf<uint64_t> k0(total, st), v0(total, st), k1(total, st), v1(total, st);
  k_leg_records<<<std::min<int64_t>(grid_for(total, 256), 148 * 32), 256, 0, st>>>(
      dd.get(), (int)hd.size(), dl.get(), total, k0.get(), v0.get());
  LT_CK_LAUNCH();
  const int end_bit = kSpaceBits + kElemBits + kKeyLo;
  size_t tmp = 0;
  LT_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0.get(), k1.get(), v0.get(), v1.get(),
                                        (int)total, 0, end_bit, st));
  {
    DevBuf<char> tb((int64_t)tmp, st);
    LT_CK(cub::DeviceRadixSort::SortPairs(tb.get(), tmp, k0.get(), k1.get(), v0.get(), v1.get(),
                                          (int)total, 0, end_bit, st));
  }
  k0.release();
  v0.release();
  DevBuf<int32_t> heads(total, st), idx(total, st);
  k_leg_heads<<<grid_for(total, 256), 256, 0, st>>>(k1.get(), total, heads.get());
  LT_CK_LAUNCH();
  tmp = 0;
  LT_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, heads.get(), idx.get(), (int)total, st));
  {
    DevBuf<char> tb((int64_t)tmp, st);
    LT_CK(cub::DeviceScan::ExclusiveSum(tb.get(), tmp, heads.get(), idx.get(), (int)total, st));
  }
  int32_t a = 0, b = 0;
  LT_CK(cudaMemcpyAsync(&a, idx.get() + total - 1, 4, cudaMemcpyDeviceToHost, st));
  LT_CK(cudaMemcpyAsync(&b, heads.get() + total - 1, 4, cudaMemcpyDeviceToHost, st));
  LT_CK(cudaStreamSynchronize(st));
  const int64_t runs = (int64_t)a + b;
  DevBuf<int64_t> start(runs, st);
  k_leg_starts<<<grid_for(total, 256), 256, 0, st>>>(heads.get(), idx.get(), total, start.get());
  LT_CK_LAUNCH();
  const int cap = 1 << 20;
  DevBuf<Viol> out(cap, st);
  DevBuf<unsigned long long> count(1, st);
  LT_CK(cudaMemsetAsync(count.get(), 0, 8, st));
  k_leg_scan<<<std::min<int64_t>(grid_for(runs, 128), 148 * 64), 128, 0, st>>>(
      k1.get(), v1.get(), start.get(), runs, total, dl.get(), dcolor.get(), s->n_tiles - 1,
      out.get(), cap, count.get());
  LT_CK_LAUNCH();
  unsigned long long hc = 0;
  LT_CK(cudaMemcpyAsync(&hc, count.get(), 8, cudaMemcpyDeviceToHost, st));
  LT_CK(cudaStreamSynchronize(st));
  const int64_t got = (int64_t)std::min<unsigned long long>(hc, cap);
  std::vector<Viol> hv(got);
  if (got)
    LT_CK(cudaMemcpyAsync(hv.data(), out.get(), sizeof(Viol) * got, cudaMemcpyDeviceToHost, st));
  LT_CK(cudaStreamSynchronize(st));
  std::set<std::tuple<int, int, int, int>> pairs, red;
  for (const Viol &v : hv) {
    if (v.kind == 0) pairs.insert({v.x, v.ex, v.y, v.ey});
    else red.insert({v.x, v.ex, v.ey, 0});
  }
  *n_pairs = (int64_t)pairs.size();
  *n_reductions = (int64_t)red.size();
  if (overflow) *overflow = hc > (unsigned long long)cap ? 1 : 0;
  LT_API_END
}
