// lt_internal.cuh — shared internals of libltcuda.so (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/looptile_cuda.h"

#define LT_MAX_DESC 8     // descriptors per loop
#define LT_MAX_INC 4      // indirect INC/WRITE descriptors per loop
#define LT_BLOCK 256      // threads per CTA of the fused tile executor

namespace lt {

// ---- error plumbing --------------------------------------------------------
struct Error {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string &msg) { throw Error{code, msg}; }

void set_last_error(const std::string &msg);

// a failed call's error is also the thread's "last error": clear it (a
// non-sticky error such as an out-of-memory allocation must not resurface in
// the caller's next unrelated CUDA call) before turning it into a status code
#define LT_CK(call)                                                               \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess) {                                                      \
      (void)cudaGetLastError();                                                   \
      ::lt::fail(LT_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    }                                                                             \
  } while (0)

#define LT_CK_LAUNCH() LT_CK(cudaGetLastError())

#define LT_API_BEGIN try {
#define LT_API_END                                        \
  }                                                       \
  catch (const ::lt::Error &e) {                          \
    ::lt::set_last_error(e.msg);                          \
    return e.code;                                        \
  }                                                       \
  catch (const std::bad_alloc &) {                        \
    ::lt::set_last_error("host out of memory");           \
    return LT_E_CUDA;                                     \
  }                                                       \
  catch (const std::exception &e) {                       \
    ::lt::set_last_error(e.what());                       \
    return LT_E_EXECUTION;                                \
  }                                                       \
  return LT_OK;

inline double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  return (int)(g < 1 ? 1 : g);
}

// ---- stream-ordered device buffer -----------------------------------------
template <class T>
struct DevBuf {
  T *p = nullptr;
  int64_t n = 0;
  cudaStream_t st = 0;
  DevBuf() = default;
  DevBuf(int64_t count, cudaStream_t s) { alloc(count, s); }
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n), st(o.st) { o.p = nullptr; o.n = 0; }
  DevBuf &operator=(DevBuf &&o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; st = o.st; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(int64_t count, cudaStream_t s) {
    release();
    st = s;
    n = count;
    if (count > 0) LT_CK(cudaMallocAsync((void **)&p, sizeof(T) * (size_t)count, s));
  }
  void release() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    n = 0;
  }
  T *get() const { return p; }
};

// ---- context ----------------------------------------------------------------
struct Ctx {
  int device = 0;
  cudaStream_t stream = 0;
  std::map<int, DevBuf<double>> params;  // per native kernel id
  uint64_t params_gen = 0;                // bumped when a parameter block is reallocated
};

// ---- host copy of an lt_chain ----------------------------------------------
struct LoopDesc {
  int space, kernel;
  std::vector<lt_desc> desc;
};
struct ChainView {
  std::vector<lt_space> spaces;
  std::vector<lt_map> maps;
  std::vector<LoopDesc> loops;
  int depth = 1;
  explicit ChainView(const lt_chain *c);
  int64_t total(int s) const { return spaces[s].core + spaces[s].boundary + spaces[s].nonexec; }
  int64_t exec_size(int s) const { return spaces[s].core + spaces[s].boundary; }
};

// ---- schedule ------------------------------------------------------------------
struct LoopLists {
  int64_t n = 0;            // space total
  DevBuf<int32_t> sigma;    // tile of each element
  DevBuf<int32_t> offsets;  // n_tiles + 1
  DevBuf<int32_t> elements; // tile-major, ascending within a tile
};

struct ExecPlan;  // lt_exec.cu

}  // namespace lt

struct lt_ctx : lt::Ctx {};

struct lt_schedule {
  lt_ctx *ctx = nullptr;
  int mode = 0, n_loops = 0, n_tiles = 0, n_core = 0, n_boundary = 0, rounds = 0;
  std::vector<int32_t> color, region;
  std::vector<int32_t> loop_space;
  std::vector<std::vector<int32_t>> loop_maps;  // distinct maps per loop (local-map keys)
  std::vector<lt::LoopLists> lists;
  std::map<std::pair<int, int>, lt::DevBuf<int32_t>> local_maps;
  lt_schedule_info info{};
  std::shared_ptr<lt::ExecPlan> plan;
  ~lt_schedule();
};

namespace lt {
// shared helpers implemented in lt_inspect.cu
void sort_pairs_u32(Ctx &ctx, const uint32_t *keys_in, const int32_t *vals_in, int64_t n,
                    int end_bit, uint32_t *keys_out, int32_t *vals_out);
void sort_pairs_u64(Ctx &ctx, const uint64_t *keys_in, const int32_t *vals_in, int64_t n,
                    int end_bit, uint64_t *keys_out, int32_t *vals_out);
void invert_flat(Ctx &ctx, const int32_t *values, int64_t n_source, int arity, int64_t n_target,
                 int32_t *offsets, int32_t *flat_sorted);
void gather_rows(Ctx &ctx, const int32_t *map, int arity, const int32_t *elements, int64_t n,
                 int32_t *out);
void lower_bound_u32(Ctx &ctx, const uint32_t *keys, int64_t n, int64_t n_bins, int32_t *offsets);
void forget_map(Ctx *ctx, const int32_t *values);
void forget_ctx(Ctx *ctx);
void assign_lists(Ctx &ctx, const int32_t *sigma, int64_t n, int n_tiles, LoopLists &out);
void build_local_maps(lt_schedule *s, const ChainView &cv);
int bits_for(int64_t max_value);
}  // namespace lt
