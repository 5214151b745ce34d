// lt_pairs.cuh -- device hash set of tile pairs (a < b), shared by the
// inspector (ConflictMatrix, inspector.py:66-77) and the execution planner.
#pragma once

#include <algorithm>

#include "lt_internal.cuh"

namespace lt {

// ---- tile-pair hash set (ConflictMatrix, inspector.py:66-77) -----------------
static constexpr unsigned long long kEmpty = ~0ull;

struct PairSet {
  unsigned long long *keys;
  unsigned int *count;
  int *overflow;
  unsigned int mask;
};

__device__ __forceinline__ unsigned int mix64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return (unsigned int)k;
}

__device__ __forceinline__ void pair_insert(const PairSet &s, int a, int b) {
  if (a == b) return;
  if (a > b) { int t = a; a = b; b = t; }
  unsigned long long key = ((unsigned long long)(unsigned)a << 32) | (unsigned)b;
  unsigned int h = mix64(key) & s.mask;
  for (unsigned int probe = 0; probe <= s.mask; ++probe) {
    unsigned long long cur = *((volatile unsigned long long *)&s.keys[h]);
    if (cur == key) return;
    if (cur == kEmpty) {
      unsigned long long prev = atomicCAS(&s.keys[h], kEmpty, key);
      if (prev == kEmpty) {
        unsigned int c = atomicAdd(s.count, 1u);
        if (c > (s.mask >> 1)) *s.overflow = 1;
        return;
      }
      if (prev == key) return;
    }
    h = (h + 1) & s.mask;
  }
  *s.overflow = 1;
}

static __global__ void k_pairs_compact(const unsigned long long *keys, unsigned int cap,
                                unsigned long long *out, unsigned int *n_out) {
  unsigned int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap) return;
  unsigned long long k = keys[i];
  if (k != kEmpty) out[atomicAdd(n_out, 1u)] = k;
}

struct PairTable {
  Ctx &ctx;
  unsigned int cap = 0;
  DevBuf<unsigned long long> keys;
  DevBuf<unsigned int> counters;  // [0]=count, [1]=overflow, [2]=compact count
  explicit PairTable(Ctx &c, unsigned int capacity) : ctx(c) { resize(capacity); }
  void resize(unsigned int capacity) {
    cap = capacity;
    keys.alloc(cap, ctx.stream);
    counters.alloc(4, ctx.stream);
    clear();
  }
  void clear() {
    LT_CK(cudaMemsetAsync(keys.get(), 0xff, sizeof(unsigned long long) * cap, ctx.stream));
    LT_CK(cudaMemsetAsync(counters.get(), 0, sizeof(unsigned int) * 4, ctx.stream));
  }
  PairSet view() {
    return PairSet{keys.get(), counters.get(), (int *)(counters.get() + 1), cap - 1};
  }
  // synchronous: (count, overflow)
  std::pair<unsigned int, bool> status() {
    unsigned int h[2];
    LT_CK(cudaMemcpyAsync(h, counters.get(), sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
    LT_CK(cudaStreamSynchronize(ctx.stream));
    return {h[0], h[1] != 0};
  }
  std::vector<unsigned long long> fetch() {
    unsigned int n = status().first;
    DevBuf<unsigned long long> out(std::max<unsigned int>(n, 1), ctx.stream);
    LT_CK(cudaMemsetAsync(counters.get() + 2, 0, sizeof(unsigned int), ctx.stream));
    k_pairs_compact<<<grid_for(cap, 256), 256, 0, ctx.stream>>>(keys.get(), cap, out.get(),
                                                                counters.get() + 2);
    LT_CK_LAUNCH();
    std::vector<unsigned long long> h(n);
    if (n)
      LT_CK(cudaMemcpyAsync(h.data(), out.get(), sizeof(unsigned long long) * n,
                            cudaMemcpyDeviceToHost, ctx.stream));
    LT_CK(cudaStreamSynchronize(ctx.stream));
    std::sort(h.begin(), h.end());
    return h;
  }
};

inline unsigned int pow2_at_least(int64_t v) {
  unsigned int c = 1u << 16;
  while ((int64_t)c < v && c < (1u << 30)) c <<= 1;
  return c;
}

}  // namespace lt
