// lt_inspect.cu — GPU inspector: seed partition, assignment, inverse maps,
// projection (Alg. 3), tiling (Alg. 4), conflict detection and the recolouring
// loop of Alg. 1.  Restates reference pkg/src/looptile/inspector.py:185-495 for
// sm_100a: every per-element loop of the reference is one thread per element;
// conflict pairs go into a device hash set (exact set semantics); greedy tile
// colouring (tiles << elements) runs on the host in C++.
#include <cub/cub.cuh>

#include <algorithm>
#include <set>

#include "lt_internal.cuh"
#include "lt_pairs.cuh"

namespace lt {

int bits_for(int64_t max_value) {
  int b = 1;
  while (b < 63 && (int64_t(1) << b) <= max_value) ++b;
  return b;
}

// ---- radix sort / scan wrappers (CUB, header-only, compiled into this .so) --
void sort_pairs_u32(Ctx &ctx, const uint32_t *kin, const int32_t *vin, int64_t n, int end_bit,
                    uint32_t *kout, int32_t *vout) {
  if (n == 0) return;
  size_t tmp = 0;
  LT_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0, end_bit,
                                        ctx.stream));
  DevBuf<char> t((int64_t)tmp, ctx.stream);
  LT_CK(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kin, kout, vin, vout, (int)n, 0, end_bit,
                                        ctx.stream));
}

void sort_pairs_u64(Ctx &ctx, const uint64_t *kin, const int32_t *vin, int64_t n, int end_bit,
                    uint64_t *kout, int32_t *vout) {
  if (n == 0) return;
  size_t tmp = 0;
  LT_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0, end_bit,
                                        ctx.stream));
  DevBuf<char> t((int64_t)tmp, ctx.stream);
  LT_CK(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kin, kout, vin, vout, (int)n, 0, end_bit,
                                        ctx.stream));
}

__global__ void k_iota(int32_t *out, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int32_t)i;
}

// offsets[t] = first index i with keys[i] >= t  (t in [0, n_bins])
__global__ void k_lower_bound(const uint32_t *keys, int64_t n, int64_t n_bins, int32_t *offsets) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > n_bins) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int64_t)keys[mid] < t) lo = mid + 1; else hi = mid;
  }
  offsets[t] = (int32_t)lo;
}

void lower_bound_u32(Ctx &ctx, const uint32_t *keys, int64_t n, int64_t n_bins, int32_t *offsets) {
  k_lower_bound<<<grid_for(n_bins + 1, 256), 256, 0, ctx.stream>>>(keys, n, n_bins, offsets);
  LT_CK_LAUNCH();
}

// invert_map (chain.py:118-135): stable sort of the flat map by target keeps
// flat (source, k) order inside each segment -> segments ascending by source.
void invert_flat(Ctx &ctx, const int32_t *values, int64_t n_source, int arity, int64_t n_target,
                 int32_t *offsets, int32_t *flat_sorted) {
  int64_t nnz = n_source * arity;
  DevBuf<int32_t> iota(nnz, ctx.stream);
  DevBuf<uint32_t> ksorted(nnz, ctx.stream);
  if (nnz) {
    k_iota<<<grid_for(nnz, 256), 256, 0, ctx.stream>>>(iota.get(), nnz);
    LT_CK_LAUNCH();
    sort_pairs_u32(ctx, (const uint32_t *)values, iota.get(), nnz, bits_for(n_target), ksorted.get(),
                   flat_sorted);
  }
  k_lower_bound<<<grid_for(n_target + 1, 256), 256, 0, ctx.stream>>>(ksorted.get(), nnz, n_target,
                                                                     offsets);
  LT_CK_LAUNCH();
}

// assign (inspector.py:385-391): stable argsort by tile -> per-tile ascending lists
void assign_lists(Ctx &ctx, const int32_t *sigma, int64_t n, int n_tiles, LoopLists &out) {
  out.offsets.alloc(n_tiles + 1, ctx.stream);
  out.elements.alloc(n, ctx.stream);
  DevBuf<int32_t> iota(n, ctx.stream);
  DevBuf<uint32_t> ks(n, ctx.stream);
  if (n) {
    k_iota<<<grid_for(n, 256), 256, 0, ctx.stream>>>(iota.get(), n);
    LT_CK_LAUNCH();
    sort_pairs_u32(ctx, (const uint32_t *)sigma, iota.get(), n, bits_for(n_tiles), ks.get(),
                   out.elements.get());
  }
  k_lower_bound<<<grid_for(n_tiles + 1, 256), 256, 0, ctx.stream>>>(ks.get(), n, n_tiles,
                                                                    out.offsets.get());
  LT_CK_LAUNCH();
}

__global__ void k_gather_rows(const int32_t *map, int arity, const int32_t *elements, int64_t n,
                              int32_t *out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * arity) return;
  int64_t p = i / arity;
  int k = (int)(i - p * arity);
  out[i] = map[(int64_t)elements[p] * arity + k];
}

void gather_rows(Ctx &ctx, const int32_t *map, int arity, const int32_t *elements, int64_t n,
                 int32_t *out) {
  if (n == 0) return;
  k_gather_rows<<<grid_for(n * arity, 256), 256, 0, ctx.stream>>>(map, arity, elements, n, out);
  LT_CK_LAUNCH();
}


// ---- inspection kernels ------------------------------------------------------

// partition_seed (inspector.py:185-205)
__global__ void k_partition_seed(int32_t *sigma, int64_t core, int64_t boundary, int64_t total,
                                 int64_t ts, int32_t m, int32_t k) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  int32_t t;
  if (e < core) t = (int32_t)(e / ts);
  else if (e < core + boundary) t = m + (int32_t)((e - core) / ts);
  else t = m + k;
  sigma[e] = t;
}

// _seed_adjacency (inspector.py:208-225): tiles sharing a seed-map target
__global__ void k_seed_adjacency(const int32_t *inv_off, const int32_t *inv_flat, int arity,
                                 const int32_t *sigma0, int64_t n_target, PairSet ps) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= n_target) return;
  int b = inv_off[g], e = inv_off[g + 1];
  for (int i = b; i < e; ++i) {
    int ti = sigma0[inv_flat[i] / arity];
    if (ti < 0) continue;  // element in no seed list
    for (int j = i + 1; j < e; ++j) {
      int tj = sigma0[inv_flat[j] / arity];
      if (tj >= 0 && ti != tj) pair_insert(ps, ti, tj);
    }
  }
}

// project, mapped descriptor (inspector.py:287-315): per target element, start
// from the old projection, scan the ascending inverse segment; the first
// strictly-higher colour wins; a second distinct tile of an already-seen colour
// is a conflict with the first tile seen with that colour.
__global__ void k_project_mapped(const int32_t *inv_off, const int32_t *inv_flat, int arity,
                                 const int32_t *sigma, const int32_t *colors,
                                 const int32_t *old_phi, int32_t *new_phi, int64_t n_target,
                                 PairSet ps) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_target) return;
  int best = -1, best_color = -1;
  int old_best = -1, old_color = -1;
  if (old_phi != nullptr && old_phi[e] >= 0) {
    old_best = old_phi[e];
    old_color = colors[old_best];
    best = old_best;
    best_color = old_color;
  }
  int b = inv_off[e], end = inv_off[e + 1];
  for (int i = b; i < end; ++i) {
    int t = sigma[inv_flat[i] / arity];
    int c = colors[t];
    int prior = -1;
    if (old_best >= 0 && old_color == c) {
      prior = old_best;
    } else {
      for (int j = b; j < i; ++j) {
        int tj = sigma[inv_flat[j] / arity];
        if (colors[tj] == c) { prior = tj; break; }
      }
    }
    if (prior >= 0 && prior != t) pair_insert(ps, prior, t);
    if (c > best_color) { best = t; best_color = c; }
  }
  new_phi[e] = best;
}

// project, direct descriptor (inspector.py:278-286): clash pairs old vs new
__global__ void k_project_direct(const int32_t *old_phi, const int32_t *sigma,
                                 const int32_t *colors, int64_t n, PairSet ps) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  int o = old_phi[e], s = sigma[e];
  if (o >= 0 && s >= 0 && o != s && colors[o] == colors[s]) pair_insert(ps, o, s);
}

struct Candidates {
  const int32_t *proj[LT_MAX_DESC];
  const int32_t *map[LT_MAX_DESC];  // nullptr for direct
  int arity[LT_MAX_DESC];
  int n;
};

// tile_loop (inspector.py:319-382) fused with the T_ne forcing of :480
__global__ void k_tile_loop(Candidates cand, const int32_t *colors, int64_t total,
                            int64_t exec_size, int32_t tne, int32_t *sigma_out,
                            int *first_missing, PairSet ps) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  int held = -1, held_color = -1;
  for (int d = 0; d < cand.n; ++d) {
    const int32_t *pa = cand.proj[d];
    const int32_t *mp = cand.map[d];
    int a = cand.arity[d];
    for (int k = 0; k < a; ++k) {
      int c = mp ? pa[mp[e * a + k]] : pa[e];
      if (c < 0) continue;
      int col = colors[c];
      if (col > held_color) { held = c; held_color = col; }
    }
  }
  if (e < exec_size) {
    if (held < 0) {
      atomicMin(first_missing, (int)e);
    } else if (ps.keys) {  // second sweep only when conflicts are collected
      for (int d = 0; d < cand.n; ++d) {
        const int32_t *pa = cand.proj[d];
        const int32_t *mp = cand.map[d];
        int a = cand.arity[d];
        for (int k = 0; k < a; ++k) {
          int c = mp ? pa[mp[e * a + k]] : pa[e];
          if (c >= 0 && c != held && colors[c] == held_color) pair_insert(ps, held, c);
        }
      }
    }
    sigma_out[e] = held;
  } else {
    sigma_out[e] = tne >= 0 ? tne : held;
  }
}

__global__ void k_scatter_sigma(const int32_t *offsets, const int32_t *elements, int n_tiles,
                                int32_t *sigma) {
  int t = blockIdx.x;
  if (t >= n_tiles) return;
  for (int i = offsets[t] + threadIdx.x; i < offsets[t + 1]; i += blockDim.x) sigma[elements[i]] = t;
}

// ---- host colouring (color_tiles, inspector.py:228-263) ---------------------
static void color_tiles_host(int mode, const std::vector<int32_t> &region,
                             const std::vector<std::vector<int>> &adj, std::vector<int32_t> &color) {
  int n = (int)region.size();
  if (mode != LT_SHARED) {
    for (int t = 0; t < n; ++t) color[t] = t;
    return;
  }
  std::vector<int> stamp(n + 2, -1);
  std::vector<char> assigned(n, 0);
  int floor = 0;
  for (int reg : {LT_CORE, LT_BOUNDARY}) {
    std::fill(assigned.begin(), assigned.end(), 0);
    int maxc = -1;
    bool any = false;
    for (int t = 0; t < n; ++t) {
      if (region[t] != reg) continue;
      for (int nb : adj[t])
        if (assigned[nb]) stamp[color[nb]] = t;
      int c = floor;
      while (c < (int)stamp.size() && stamp[c] == t) ++c;
      color[t] = c;
      assigned[t] = 1;
      maxc = std::max(maxc, c);
      any = true;
    }
    if (any) floor = maxc + 1;
  }
  color[n - 1] = floor;  // non-exec tile above everything
}

void build_local_maps(lt_schedule *s, const ChainView &cv) {
  Ctx &ctx = *s->ctx;
  s->local_maps.clear();
  for (int j = 0; j < s->n_loops; ++j) {
    for (int m : s->loop_maps[j]) {
      const lt_map &mp = cv.maps[m];
      DevBuf<int32_t> out(s->lists[j].n * mp.arity, ctx.stream);
      gather_rows(ctx, mp.values, mp.arity, s->lists[j].elements.get(), s->lists[j].n, out.get());
      s->local_maps.emplace(std::make_pair(j, m), std::move(out));
    }
  }
}

static void fill_loop_maps(lt_schedule *s, const ChainView &cv) {
  s->loop_space.clear();
  s->loop_maps.assign(cv.loops.size(), {});
  for (size_t j = 0; j < cv.loops.size(); ++j) {
    s->loop_space.push_back(cv.loops[j].space);
    for (const lt_desc &d : cv.loops[j].desc) {
      if (d.map < 0) continue;
      auto &v = s->loop_maps[j];
      if (std::find(v.begin(), v.end(), d.map) == v.end()) v.push_back(d.map);
    }
  }
}

static void finish_info(lt_schedule *s) {
  std::set<int> colors(s->color.begin(), s->color.end());
  s->info.mode = s->mode;
  s->info.n_loops = s->n_loops;
  s->info.n_tiles = s->n_tiles;
  s->info.n_core_tiles = s->n_core;
  s->info.n_boundary_tiles = s->n_boundary;
  s->info.rounds = s->rounds;
  s->info.n_colors = (int)colors.size();
}

// ---- inspect_chain (inspector.py:433-495) ------------------------------------
static lt_schedule *inspect(Ctx &ctx, const ChainView &cv, int64_t ts, int mode) {
  if (ts < 1) fail(LT_E_VALUE, "tile size must be >= 1, got " + std::to_string(ts));
  if (cv.loops.empty()) fail(LT_E_INVALID_CHAIN, "a loop chain needs at least one loop");
  double t_start = now_s();
  auto sched = std::make_unique<lt_schedule>();
  lt_schedule *s = sched.get();
  s->ctx = static_cast<lt_ctx *>(&ctx);
  s->mode = mode;
  s->n_loops = (int)cv.loops.size();
  fill_loop_maps(s, cv);
  s->lists.resize(s->n_loops);

  // -- seed partition + assign + seed map
  double t0 = now_s();
  const int seed_space = cv.loops[0].space;
  const lt_space &S0 = cv.spaces[seed_space];
  int64_t m64 = (S0.core + ts - 1) / ts, k64 = (S0.boundary + ts - 1) / ts;
  if (m64 + k64 + 1 >= (int64_t(1) << 30)) fail(LT_E_VALUE, "too many tiles");
  const int m = (int)m64, k = (int)k64, n_tiles = m + k + 1, tne = m + k;
  s->n_tiles = n_tiles;
  s->n_core = m;
  s->n_boundary = k;
  s->region.assign(n_tiles, LT_CORE);
  for (int t = m; t < m + k; ++t) s->region[t] = LT_BOUNDARY;
  s->region[tne] = LT_NONEXEC;
  s->color.assign(n_tiles, -1);
  LoopLists &L0 = s->lists[0];
  L0.n = cv.total(seed_space);
  L0.sigma.alloc(L0.n, ctx.stream);
  if (L0.n)
    k_partition_seed<<<grid_for(L0.n, 256), 256, 0, ctx.stream>>>(
        L0.sigma.get(), S0.core, S0.boundary, L0.n, ts, m, k);
  LT_CK_LAUNCH();
  assign_lists(ctx, L0.sigma.get(), L0.n, n_tiles, L0);
  // find_seed_map (inspector.py:421-430)
  int seed_map = -1;
  for (const lt_desc &d : cv.loops[0].desc)
    if (d.map >= 0 && cv.maps[d.map].source == seed_space) { seed_map = d.map; break; }
  if (seed_map < 0)
    for (size_t i = 0; i < cv.maps.size(); ++i)
      if (cv.maps[i].source == seed_space) { seed_map = (int)i; break; }
  LT_CK(cudaStreamSynchronize(ctx.stream));
  s->info.partition_s += now_s() - t0;

  // inverse maps, built once per inspection (inspector.py:289-291)
  std::map<int, std::pair<DevBuf<int32_t>, DevBuf<int32_t>>> inverse;
  auto inverse_of = [&](int mi) -> std::pair<DevBuf<int32_t>, DevBuf<int32_t>> & {
    auto it = inverse.find(mi);
    if (it != inverse.end()) return it->second;
    const lt_map &mp = cv.maps[mi];
    int64_t ns = cv.total(mp.source), nt = cv.total(mp.target);
    DevBuf<int32_t> off(nt + 1, ctx.stream), flat(ns * mp.arity, ctx.stream);
    invert_flat(ctx, mp.values, ns, mp.arity, nt, off.get(), flat.get());
    return inverse.emplace(mi, std::make_pair(std::move(off), std::move(flat))).first->second;
  };

  PairTable pairs(ctx, pow2_at_least(int64_t(n_tiles) * 64));

  // -- seed adjacency (shared mode only)
  t0 = now_s();
  std::vector<std::vector<int>> adj(n_tiles);
  if (mode == LT_SHARED && seed_map >= 0) {
    for (;;) {
      auto &inv = inverse_of(seed_map);
      const lt_map &mp = cv.maps[seed_map];
      int64_t nt = cv.total(mp.target);
      if (nt)
        k_seed_adjacency<<<grid_for(nt, 256), 256, 0, ctx.stream>>>(
            inv.first.get(), inv.second.get(), mp.arity, L0.sigma.get(), nt, pairs.view());
      LT_CK_LAUNCH();
      if (pairs.status().second) { pairs.resize(pairs.cap * 2); continue; }
      break;
    }
    for (unsigned long long key : pairs.fetch()) {
      int a = (int)(key >> 32), b = (int)(key & 0xffffffffu);
      adj[a].push_back(b);
      adj[b].push_back(a);
    }
  }
  s->info.coloring_s += now_s() - t0;

  // projection buffers per space
  const int n_spaces = (int)cv.spaces.size();
  std::vector<DevBuf<int32_t>> phi(n_spaces), phi_tmp(n_spaces);
  std::vector<char> present(n_spaces, 0);
  for (int sp = 0; sp < n_spaces; ++sp) {
    phi[sp].alloc(cv.total(sp), ctx.stream);
    phi_tmp[sp].alloc(cv.total(sp), ctx.stream);
  }
  for (int j = 1; j < s->n_loops; ++j) {
    s->lists[j].n = cv.total(cv.loops[j].space);
    s->lists[j].sigma.alloc(s->lists[j].n, ctx.stream);
  }
  DevBuf<int32_t> colors_dev(n_tiles, ctx.stream);
  DevBuf<int> missing(1, ctx.stream);
  std::set<unsigned long long> fake;
  const int64_t max_rounds = 10 * (int64_t)n_tiles;
  int rounds = 0;

  for (;;) {
    ++rounds;
    if (rounds > max_rounds)
      fail(LT_E_COLORING_LIMIT,
           "recoloring did not converge after " + std::to_string(max_rounds) + " rounds");
    t0 = now_s();
    color_tiles_host(mode, s->region, adj, s->color);
    LT_CK(cudaMemcpyAsync(colors_dev.get(), s->color.data(), sizeof(int32_t) * n_tiles,
                          cudaMemcpyHostToDevice, ctx.stream));
    s->info.coloring_s += now_s() - t0;

    t0 = now_s();
    pairs.clear();
    std::fill(present.begin(), present.end(), 0);
    const int32_t *sigma = L0.sigma.get();
    for (int j = 1; j < s->n_loops; ++j) {
      // project loop j-1 (inspector.py:266-316), descriptors in order
      const LoopDesc &prev = cv.loops[j - 1];
      for (const lt_desc &d : prev.desc) {
        if (d.map < 0) {
          int sp = prev.space;
          int64_t n = cv.total(sp);
          if (present[sp] && n)
            k_project_direct<<<grid_for(n, 256), 256, 0, ctx.stream>>>(
                phi[sp].get(), sigma, colors_dev.get(), n, pairs.view());
          LT_CK_LAUNCH();
          if (n)
            LT_CK(cudaMemcpyAsync(phi[sp].get(), sigma, sizeof(int32_t) * n,
                                  cudaMemcpyDeviceToDevice, ctx.stream));
          present[sp] = 1;
        } else {
          const lt_map &mp = cv.maps[d.map];
          auto &inv = inverse_of(d.map);
          int sp = mp.target;
          int64_t n = cv.total(sp);
          if (n)
            k_project_mapped<<<grid_for(n, 256), 256, 0, ctx.stream>>>(
                inv.first.get(), inv.second.get(), mp.arity, sigma, colors_dev.get(),
                present[sp] ? phi[sp].get() : nullptr, phi_tmp[sp].get(), n, pairs.view());
          LT_CK_LAUNCH();
          std::swap(phi[sp], phi_tmp[sp]);
          present[sp] = 1;
        }
      }
      // tile loop j (inspector.py:319-382)
      const LoopDesc &cur = cv.loops[j];
      Candidates cand{};
      for (const lt_desc &d : cur.desc) {
        int sp = d.map < 0 ? cur.space : cv.maps[d.map].target;
        if (!present[sp]) continue;
        if (cand.n >= LT_MAX_DESC) fail(LT_E_INSPECTION, "too many descriptors");
        cand.proj[cand.n] = phi[sp].get();
        cand.map[cand.n] = d.map < 0 ? nullptr : cv.maps[d.map].values;
        cand.arity[cand.n] = d.map < 0 ? 1 : cv.maps[d.map].arity;
        cand.n++;
      }
      if (cand.n == 0)
        fail(LT_E_INSPECTION, "loop " + std::to_string(j) + " over space " +
                                  std::to_string(cur.space) +
                                  ": no projection covers any accessed space");
      int big = 0x7fffffff;
      LT_CK(cudaMemcpyAsync(missing.get(), &big, sizeof(int), cudaMemcpyHostToDevice, ctx.stream));
      LoopLists &Lj = s->lists[j];
      if (Lj.n)
        k_tile_loop<<<grid_for(Lj.n, 256), 256, 0, ctx.stream>>>(
            cand, colors_dev.get(), Lj.n, cv.exec_size(cur.space), tne, Lj.sigma.get(),
            missing.get(), pairs.view());
      LT_CK_LAUNCH();
      int miss = big;
      LT_CK(cudaMemcpyAsync(&miss, missing.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
      LT_CK(cudaStreamSynchronize(ctx.stream));
      if (miss != big)
        fail(LT_E_INSPECTION, "loop " + std::to_string(j) + ": element " + std::to_string(miss) +
                                  " of space " + std::to_string(cur.space) +
                                  " is not reachable through any projection");
      assign_lists(ctx, Lj.sigma.get(), Lj.n, n_tiles, Lj);
      sigma = Lj.sigma.get();
    }
    auto st = pairs.status();
    s->info.projection_tiling_s += now_s() - t0;
    if (st.second) {  // hash set overflow: enlarge and replay this round
      pairs.resize(pairs.cap * 2);
      --rounds;
      continue;
    }
    if (st.first) {
      for (unsigned long long key : pairs.fetch()) {
        if (fake.insert(key).second) {
          int a = (int)(key >> 32), b = (int)(key & 0xffffffffu);
          adj[a].push_back(b);
          adj[b].push_back(a);
        }
      }
      continue;
    }
    break;
  }
  s->rounds = rounds;

  t0 = now_s();
  build_local_maps(s, cv);
  LT_CK(cudaStreamSynchronize(ctx.stream));
  s->info.local_maps_s += now_s() - t0;
  s->info.total_s = now_s() - t_start;
  finish_info(s);
  return sched.release();
}

static lt_schedule *import_schedule(Ctx &ctx, const ChainView &cv, int mode, int n_tiles,
                                    const int32_t *colors, const int32_t *regions, int rounds,
                                    const int32_t *const *offsets,
                                    const int32_t *const *elements) {
  auto sched = std::make_unique<lt_schedule>();
  lt_schedule *s = sched.get();
  s->ctx = static_cast<lt_ctx *>(&ctx);
  s->mode = mode;
  s->n_loops = (int)cv.loops.size();
  s->n_tiles = n_tiles;
  s->rounds = rounds;
  s->color.assign(colors, colors + n_tiles);
  s->region.assign(regions, regions + n_tiles);
  for (int t = 0; t < n_tiles; ++t) {
    if (s->region[t] == LT_CORE) s->n_core++;
    if (s->region[t] == LT_BOUNDARY) s->n_boundary++;
  }
  if (n_tiles < 1 || s->region[n_tiles - 1] != LT_NONEXEC)
    fail(LT_E_VALUE, "the last tile must be the non-exec tile");
  fill_loop_maps(s, cv);
  s->lists.resize(s->n_loops);
  for (int j = 0; j < s->n_loops; ++j) {
    LoopLists &L = s->lists[j];
    L.n = cv.total(cv.loops[j].space);
    if (offsets[j][0] != 0 || offsets[j][n_tiles] != L.n)
      fail(LT_E_VALUE, "iteration lists of loop " + std::to_string(j) +
                           " do not partition the space");
    L.offsets.alloc(n_tiles + 1, ctx.stream);
    L.elements.alloc(L.n, ctx.stream);
    L.sigma.alloc(L.n, ctx.stream);
    LT_CK(cudaMemcpyAsync(L.offsets.get(), offsets[j], sizeof(int32_t) * (n_tiles + 1),
                          cudaMemcpyHostToDevice, ctx.stream));
    if (L.n) {
      LT_CK(cudaMemcpyAsync(L.elements.get(), elements[j], sizeof(int32_t) * L.n,
                            cudaMemcpyHostToDevice, ctx.stream));
      LT_CK(cudaMemsetAsync(L.sigma.get(), 0xff, sizeof(int32_t) * L.n, ctx.stream));
      k_scatter_sigma<<<n_tiles, 256, 0, ctx.stream>>>(L.offsets.get(), L.elements.get(), n_tiles,
                                                       L.sigma.get());
      LT_CK_LAUNCH();
    }
  }
  build_local_maps(s, cv);
  LT_CK(cudaStreamSynchronize(ctx.stream));
  finish_info(s);
  return sched.release();
}

}  // namespace lt

using namespace lt;

__global__ void k_div_inplace(int32_t *v, int64_t n, int a) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] /= a;
}

extern "C" int lt_invert_map(lt_ctx *ctx, const int32_t *values, int64_t n_source, int32_t arity,
                             int64_t n_target, int32_t *offsets, int32_t *sources) {
  LT_API_BEGIN
  if (!ctx) fail(LT_E_VALUE, "null context");
  invert_flat(*ctx, values, n_source, arity, n_target, offsets, sources);
  // flat (source*arity + k) -> source id
  if (n_source * arity > 0) {
    k_div_inplace<<<grid_for(n_source * arity, 256), 256, 0, ctx->stream>>>(sources,
                                                                            n_source * arity, arity);
    LT_CK_LAUNCH();
  }
  LT_CK(cudaStreamSynchronize(ctx->stream));
  LT_API_END
}

extern "C" int lt_inspect(lt_ctx *ctx, const lt_chain *chain, int64_t tile_size, int32_t mode,
                          lt_schedule **out) {
  LT_API_BEGIN
  if (!ctx || !chain || !out) fail(LT_E_VALUE, "null argument");
  ChainView cv(chain);
  *out = inspect(*ctx, cv, tile_size, mode);
  LT_API_END
}

extern "C" int lt_schedule_import(lt_ctx *ctx, const lt_chain *chain, int32_t mode,
                                  int32_t n_tiles, const int32_t *colors, const int32_t *regions,
                                  int32_t rounds, const int32_t *const *offsets,
                                  const int32_t *const *elements, lt_schedule **out) {
  LT_API_BEGIN
  if (!ctx || !chain || !out) fail(LT_E_VALUE, "null argument");
  ChainView cv(chain);
  *out = import_schedule(*ctx, cv, mode, n_tiles, colors, regions, rounds, offsets, elements);
  LT_API_END
}

extern "C" int lt_schedule_info_get(const lt_schedule *s, lt_schedule_info *info) {
  LT_API_BEGIN
  if (!s || !info) fail(LT_E_VALUE, "null argument");
  *info = s->info;
  LT_API_END
}

extern "C" int lt_schedule_tiles(const lt_schedule *s, int32_t *colors, int32_t *regions) {
  LT_API_BEGIN
  if (!s) fail(LT_E_VALUE, "null schedule");
  if (colors) std::copy(s->color.begin(), s->color.end(), colors);
  if (regions) std::copy(s->region.begin(), s->region.end(), regions);
  LT_API_END
}

extern "C" int lt_schedule_lists(const lt_schedule *s, int32_t loop, int32_t *offsets,
                                 int32_t *elements) {
  LT_API_BEGIN
  if (!s || loop < 0 || loop >= s->n_loops) fail(LT_E_VALUE, "bad loop index");
  const LoopLists &L = s->lists[loop];
  cudaStream_t st = s->ctx->stream;
  if (offsets)
    LT_CK(cudaMemcpyAsync(offsets, L.offsets.get(), sizeof(int32_t) * (s->n_tiles + 1),
                          cudaMemcpyDeviceToHost, st));
  if (elements && L.n)
    LT_CK(cudaMemcpyAsync(elements, L.elements.get(), sizeof(int32_t) * L.n,
                          cudaMemcpyDeviceToHost, st));
  LT_CK(cudaStreamSynchronize(st));
  LT_API_END
}

extern "C" int lt_schedule_tile_of(const lt_schedule *s, int32_t loop, const int32_t **sigma,
                                   int64_t *n) {
  LT_API_BEGIN
  if (!s || loop < 0 || loop >= s->n_loops) fail(LT_E_VALUE, "bad loop index");
  *sigma = s->lists[loop].sigma.get();
  *n = s->lists[loop].n;
  LT_API_END
}

extern "C" int lt_schedule_local_map(const lt_schedule *s, int32_t loop, int32_t map,
                                     int32_t *out) {
  LT_API_BEGIN
  if (!s) fail(LT_E_VALUE, "null schedule");
  auto it = s->local_maps.find(std::make_pair((int)loop, (int)map));
  if (it == s->local_maps.end()) fail(LT_E_VALUE, "loop has no local map for that map");
  if (it->second.n)
    LT_CK(cudaMemcpyAsync(out, it->second.get(), sizeof(int32_t) * it->second.n,
                          cudaMemcpyDeviceToHost, s->ctx->stream));
  LT_CK(cudaStreamSynchronize(s->ctx->stream));
  LT_API_END
}

extern "C" int lt_schedule_destroy(lt_schedule *s) {
  LT_API_BEGIN
  delete s;
  LT_API_END
}

// ---- step-level inspector API (reference inspector.py public functions) -------

namespace lt {

static void copy_pairs(PairTable &pt, int64_t *pairs, int64_t cap, int64_t *n_pairs) {
  std::vector<unsigned long long> v = pt.fetch();
  *n_pairs = (int64_t)v.size();
  if (pairs)
    for (int64_t i = 0; i < (int64_t)v.size() && i < cap; ++i) pairs[i] = (int64_t)v[i];
}

static unsigned int pair_capacity(int n_tiles) {
  return pow2_at_least(int64_t(std::max(n_tiles, 1)) * 64);
}

}  // namespace lt

extern "C" int lt_partition_seed(lt_ctx *ctx, const lt_space *sp, int64_t ts, int32_t *sigma,
                                 int32_t *n_core_tiles, int32_t *n_boundary_tiles) {
  LT_API_BEGIN
  if (!ctx || !sp) fail(LT_E_VALUE, "null argument");
  if (ts < 1) fail(LT_E_VALUE, "tile size must be >= 1, got " + std::to_string(ts));
  const int64_t m = (sp->core + ts - 1) / ts, k = (sp->boundary + ts - 1) / ts;
  const int64_t total = sp->core + sp->boundary + sp->nonexec;
  if (total)
    k_partition_seed<<<grid_for(total, 256), 256, 0, ctx->stream>>>(sigma, sp->core, sp->boundary,
                                                                     total, ts, (int)m, (int)k);
  LT_CK_LAUNCH();
  LT_CK(cudaStreamSynchronize(ctx->stream));
  *n_core_tiles = (int32_t)m;
  *n_boundary_tiles = (int32_t)k;
  LT_API_END
}

extern "C" int lt_assign(lt_ctx *ctx, const int32_t *sigma, int64_t n, int32_t n_tiles,
                         int32_t *offsets, int32_t *elements) {
  LT_API_BEGIN
  if (!ctx) fail(LT_E_VALUE, "null context");
  LoopLists L;
  assign_lists(*ctx, sigma, n, n_tiles, L);
  LT_CK(cudaMemcpyAsync(offsets, L.offsets.get(), 4 * (n_tiles + 1), cudaMemcpyDeviceToDevice,
                        ctx->stream));
  if (n)
    LT_CK(cudaMemcpyAsync(elements, L.elements.get(), 4 * n, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  LT_CK(cudaStreamSynchronize(ctx->stream));
  LT_API_END
}

extern "C" int lt_seed_adjacency(lt_ctx *ctx, const int32_t *values, int64_t n_source,
                                 int32_t arity, int64_t n_target, const int32_t *sigma,
                                 int32_t n_tiles, int64_t *pairs, int64_t capacity,
                                 int64_t *n_pairs) {
  LT_API_BEGIN
  if (!ctx) fail(LT_E_VALUE, "null context");
  DevBuf<int32_t> off(n_target + 1, ctx->stream), flat(n_source * arity, ctx->stream);
  invert_flat(*ctx, values, n_source, arity, n_target, off.get(), flat.get());
  PairTable pt(*ctx, pair_capacity(n_tiles));
  for (;;) {
    if (n_target)
      k_seed_adjacency<<<grid_for(n_target, 256), 256, 0, ctx->stream>>>(
          off.get(), flat.get(), arity, sigma, n_target, pt.view());
    LT_CK_LAUNCH();
    if (pt.status().second) { pt.resize(pt.cap * 2); continue; }
    break;
  }
  copy_pairs(pt, pairs, capacity, n_pairs);
  LT_API_END
}

extern "C" int lt_color_tiles(int32_t n_tiles, const int32_t *regions, int32_t mode,
                              const int64_t *pairs, int64_t n_pairs, int32_t *colors) {
  LT_API_BEGIN
  if (n_tiles < 1) fail(LT_E_VALUE, "no tiles");
  std::vector<int32_t> region(regions, regions + n_tiles), color(n_tiles, -1);
  std::vector<std::vector<int>> adj(n_tiles);
  for (int64_t i = 0; i < n_pairs; ++i) {
    const int a = (int)(pairs[i] >> 32), b = (int)(pairs[i] & 0xffffffff);
    if (a < 0 || b < 0 || a >= n_tiles || b >= n_tiles) fail(LT_E_VALUE, "pair outside tiles");
    adj[a].push_back(b);
    adj[b].push_back(a);
  }
  color_tiles_host(mode, region, adj, color);
  std::copy(color.begin(), color.end(), colors);
  LT_API_END
}

extern "C" int lt_project(lt_ctx *ctx, const lt_chain *chain, int32_t loop, const int32_t *sigma,
                          const int32_t *colors, int32_t n_tiles, int32_t *const *phi,
                          int32_t *present, int64_t *pairs, int64_t capacity, int64_t *n_pairs) {
  LT_API_BEGIN
  if (!ctx || !chain || !phi || !present) fail(LT_E_VALUE, "null argument");
  ChainView cv(chain);
  if (loop < 0 || loop >= (int)cv.loops.size()) fail(LT_E_VALUE, "bad loop index");
  const LoopDesc &L = cv.loops[loop];
  PairTable pt(*ctx, pair_capacity(n_tiles));
  std::vector<int32_t> pres(present, present + cv.spaces.size());
  for (;;) {
    // replay from the caller's projections each attempt (inputs stay untouched)
    std::map<int, DevBuf<int32_t>> cur;
    std::vector<char> have(cv.spaces.size());
    for (size_t sp = 0; sp < cv.spaces.size(); ++sp) have[sp] = pres[sp] != 0;
    auto view = [&](int sp) -> const int32_t * {
      auto it = cur.find(sp);
      return it != cur.end() ? it->second.get() : phi[sp];
    };
    for (const lt_desc &d : L.desc) {
      if (d.map < 0) {
        const int sp = L.space;
        const int64_t n = cv.total(sp);
        if (have[sp] && n)
          k_project_direct<<<grid_for(n, 256), 256, 0, ctx->stream>>>(view(sp), sigma, colors, n,
                                                                      pt.view());
        LT_CK_LAUNCH();
        DevBuf<int32_t> nb(n, ctx->stream);
        if (n)
          LT_CK(cudaMemcpyAsync(nb.get(), sigma, 4 * n, cudaMemcpyDeviceToDevice, ctx->stream));
        cur[sp] = std::move(nb);
        have[sp] = 1;
      } else {
        const lt_map &mp = cv.maps[d.map];
        const int sp = mp.target;
        const int64_t ns = cv.total(mp.source), nt = cv.total(sp);
        DevBuf<int32_t> off(nt + 1, ctx->stream), flat(ns * mp.arity, ctx->stream), nb(nt, ctx->stream);
        invert_flat(*ctx, mp.values, ns, mp.arity, nt, off.get(), flat.get());
        if (nt)
          k_project_mapped<<<grid_for(nt, 256), 256, 0, ctx->stream>>>(
              off.get(), flat.get(), mp.arity, sigma, colors, have[sp] ? view(sp) : nullptr,
              nb.get(), nt, pt.view());
        LT_CK_LAUNCH();
        cur[sp] = std::move(nb);
        have[sp] = 1;
      }
    }
    if (pt.status().second) { pt.resize(pt.cap * 2); continue; }
    for (auto &kv : cur) {
      const int64_t n = cv.total(kv.first);
      if (n)
        LT_CK(cudaMemcpyAsync(phi[kv.first], kv.second.get(), 4 * n, cudaMemcpyDeviceToDevice,
                              ctx->stream));
      present[kv.first] = 1;
    }
    break;
  }
  copy_pairs(pt, pairs, capacity, n_pairs);
  LT_API_END
}

extern "C" int lt_tile_loop(lt_ctx *ctx, const lt_chain *chain, int32_t loop,
                            int32_t *const *phi, const int32_t *present, const int32_t *colors,
                            int32_t n_tiles, int32_t tne, int32_t *sigma_out, int32_t detect,
                            int64_t *pairs, int64_t capacity, int64_t *n_pairs) {
  LT_API_BEGIN
  if (!ctx || !chain || !phi || !present) fail(LT_E_VALUE, "null argument");
  ChainView cv(chain);
  if (loop < 0 || loop >= (int)cv.loops.size()) fail(LT_E_VALUE, "bad loop index");
  const LoopDesc &L = cv.loops[loop];
  Candidates cand{};
  for (const lt_desc &d : L.desc) {
    const int sp = d.map < 0 ? L.space : cv.maps[d.map].target;
    if (!present[sp]) continue;
    if (cand.n >= LT_MAX_DESC) fail(LT_E_INSPECTION, "too many descriptors");
    cand.proj[cand.n] = phi[sp];
    cand.map[cand.n] = d.map < 0 ? nullptr : cv.maps[d.map].values;
    cand.arity[cand.n] = d.map < 0 ? 1 : cv.maps[d.map].arity;
    cand.n++;
  }
  if (cand.n == 0)
    fail(LT_E_INSPECTION, "loop " + std::to_string(loop) + " over space " +
                              std::to_string(L.space) + ": no projection covers any accessed space");
  const int64_t n = cv.total(L.space);
  PairTable pt(*ctx, pair_capacity(n_tiles));
  DevBuf<int> missing(1, ctx->stream);
  for (;;) {
    const int big = 0x7fffffff;
    LT_CK(cudaMemcpyAsync(missing.get(), &big, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    PairSet ps = pt.view();
    if (!detect) ps.keys = nullptr;
    if (n)
      k_tile_loop<<<grid_for(n, 256), 256, 0, ctx->stream>>>(cand, colors, n, cv.exec_size(L.space),
                                                             tne, sigma_out, missing.get(), ps);
    LT_CK_LAUNCH();
    int miss = big;
    LT_CK(cudaMemcpyAsync(&miss, missing.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    LT_CK(cudaStreamSynchronize(ctx->stream));
    if (miss != big)
      fail(LT_E_INSPECTION, "loop " + std::to_string(loop) + ": element " + std::to_string(miss) +
                                " of space " + std::to_string(L.space) +
                                " is not reachable through any projection");
    if (detect && pt.status().second) { pt.resize(pt.cap * 2); continue; }
    break;
  }
  if (detect) copy_pairs(pt, pairs, capacity, n_pairs);
  else *n_pairs = 0;
  LT_API_END
}

extern "C" int lt_gather_rows(lt_ctx *ctx, const int32_t *map_values, int32_t arity,
                              const int32_t *elements, int64_t n, int32_t *out) {
  LT_API_BEGIN
  if (!ctx) fail(LT_E_VALUE, "null context");
  gather_rows(*ctx, map_values, arity, elements, n, out);
  LT_CK(cudaStreamSynchronize(ctx->stream));
  LT_API_END
}
