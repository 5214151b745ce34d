// lt_api.cu — context, error state, kernel parameters, halo packing and the
// host-side RCM data-layout pass of libltcuda.so.
#include <algorithm>
#include <deque>

#include "lt_internal.cuh"

namespace lt {

static thread_local std::string g_last_error;

void set_last_error(const std::string &msg) { g_last_error = msg; }

ChainView::ChainView(const lt_chain *c) {
  if (c->n_spaces < 0 || c->n_maps < 0 || c->n_loops < 0)
    fail(LT_E_INVALID_CHAIN, "negative chain sizes");
  spaces.assign(c->spaces, c->spaces + c->n_spaces);
  maps.assign(c->maps, c->maps + c->n_maps);
  depth = c->depth;
  for (const lt_space &s : spaces) {
    if (s.core < 0 || s.boundary < 0 || s.nonexec < 0)
      fail(LT_E_INVALID_CHAIN, "negative region size");
    if (s.core + s.boundary + s.nonexec >= (int64_t(1) << 31))
      fail(LT_E_INVALID_CHAIN, "space exceeds the int32 index range");
  }
  for (const lt_map &m : maps) {
    if (m.source < 0 || m.source >= c->n_spaces || m.target < 0 || m.target >= c->n_spaces)
      fail(LT_E_INVALID_CHAIN, "map references a space outside the chain");
    if (m.arity < 1) fail(LT_E_INVALID_CHAIN, "map arity < 1");
    if (!m.values && total(m.source) > 0) fail(LT_E_INVALID_CHAIN, "map without device values");
  }
  for (int j = 0; j < c->n_loops; ++j) {
    const lt_loop &l = c->loops[j];
    if (l.space < 0 || l.space >= c->n_spaces)
      fail(LT_E_INVALID_CHAIN, "loop iterates an unknown space");
    if (l.n_desc < 1) fail(LT_E_INVALID_CHAIN, "loop has no descriptors");
    LoopDesc d;
    d.space = l.space;
    d.kernel = l.kernel;
    d.desc.assign(l.desc, l.desc + l.n_desc);
    for (const lt_desc &x : d.desc) {
      if (x.map >= c->n_maps) fail(LT_E_INVALID_CHAIN, "descriptor uses an undeclared map");
      if (x.map >= 0 && maps[x.map].source != l.space)
        fail(LT_E_INVALID_CHAIN, "descriptor map not sourced on the loop's space");
      if (x.mode < LT_READ || x.mode > LT_RW) fail(LT_E_INVALID_CHAIN, "bad access mode");
    }
    loops.push_back(std::move(d));
  }
}

__global__ void k_pack(const double *values, int vpe, const int32_t *rows, int64_t n, double *out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * vpe) return;
  int64_t r = i / vpe;
  int c = (int)(i - r * vpe);
  out[i] = values[(int64_t)rows[r] * vpe + c];
}

__global__ void k_unpack(double *values, int vpe, const int32_t *rows, int64_t n, const double *in) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * vpe) return;
  int64_t r = i / vpe;
  int c = (int)(i - r * vpe);
  values[(int64_t)rows[r] * vpe + c] = in[i];
}

}  // namespace lt

using namespace lt;

extern "C" int lt_abi_version(void) { return LT_ABI_VERSION; }

extern "C" const char *lt_last_error(void) { return g_last_error.c_str(); }

extern "C" int lt_ctx_create(int device, lt_ctx **out) {
  LT_API_BEGIN
  if (!out) fail(LT_E_VALUE, "null output");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    fail(LT_E_CUDA, std::string("no CUDA device available (") + cudaGetErrorString(e) +
                        "); the looptile executor has no CPU fallback");
  if (device < 0 || device >= n) fail(LT_E_VALUE, "device index out of range");
  LT_CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  LT_CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    fail(LT_E_CUDA, std::string("device ") + prop.name + " is not sm_100 (B200); built for sm_100a");
  auto *c = new lt_ctx();
  c->device = device;
  c->stream = 0;
  *out = c;
  LT_API_END
}

extern "C" int lt_ctx_destroy(lt_ctx *ctx) {
  LT_API_BEGIN
  if (ctx) {
    forget_ctx(ctx);
    cudaStreamSynchronize(ctx->stream);
    delete ctx;
  }
  LT_API_END
}

extern "C" int lt_ctx_set_stream(lt_ctx *ctx, void *stream) {
  LT_API_BEGIN
  if (!ctx) fail(LT_E_VALUE, "null context");
  ctx->stream = (cudaStream_t)stream;
  LT_API_END
}

extern "C" int lt_ctx_synchronize(lt_ctx *ctx) {
  LT_API_BEGIN
  if (!ctx) fail(LT_E_VALUE, "null context");
  LT_CK(cudaStreamSynchronize(ctx->stream));
  LT_API_END
}

extern "C" int lt_ctx_forget_map(lt_ctx *ctx, const int32_t *values) {
  LT_API_BEGIN
  forget_map(ctx, values);
  LT_API_END
}

extern "C" int lt_ctx_set_kernel_params(lt_ctx *ctx, int32_t kernel_id, const double *host,
                                        int64_t n) {
  LT_API_BEGIN
  if (!ctx) fail(LT_E_VALUE, "null context");
  if (kernel_id < 0 || kernel_id >= lt_kernel_count()) fail(LT_E_EXECUTION, "unknown kernel id");
  // Update in place when the block fits: cached execution plans and captured
  // CUDA graphs hold the device pointer, so they see the new values.  A block
  // that must grow is reallocated and the generation bump invalidates every
  // cached plan (graphs captured before that must be re-captured).
  auto it = ctx->params.find(kernel_id);
  if (it == ctx->params.end() || it->second.n < std::max<int64_t>(n, 1)) {
    DevBuf<double> buf(std::max<int64_t>(n, 1), ctx->stream);
    ctx->params[kernel_id] = std::move(buf);
    ++ctx->params_gen;
  }
  if (n > 0)
    LT_CK(cudaMemcpyAsync(ctx->params[kernel_id].get(), host, sizeof(double) * n,
                          cudaMemcpyHostToDevice, ctx->stream));
  LT_CK(cudaStreamSynchronize(ctx->stream));
  LT_API_END
}

extern "C" int lt_halo_pack(lt_ctx *ctx, const double *values, int32_t vpe, const int32_t *rows,
                            int64_t n_rows, double *out) {
  LT_API_BEGIN
  if (!ctx) fail(LT_E_VALUE, "null context");
  if (n_rows * vpe > 0) {
    k_pack<<<grid_for(n_rows * vpe, 256), 256, 0, ctx->stream>>>(values, vpe, rows, n_rows, out);
    LT_CK_LAUNCH();
  }
  LT_API_END
}

extern "C" int lt_halo_unpack(lt_ctx *ctx, double *values, int32_t vpe, const int32_t *rows,
                              int64_t n_rows, const double *in) {
  LT_API_BEGIN
  if (!ctx) fail(LT_E_VALUE, "null context");
  if (n_rows * vpe > 0) {
    k_unpack<<<grid_for(n_rows * vpe, 256), 256, 0, ctx->stream>>>(values, vpe, rows, n_rows, in);
    LT_CK_LAUNCH();
  }
  LT_API_END
}

// Reverse Cuthill-McKee (mesh.py:123-145): start at the lowest-id vertex of
// minimum degree, visit neighbours by (degree, id), reverse the BFS order.
extern "C" int lt_rcm_order(int64_t n, const int64_t *offsets, const int64_t *nbrs,
                            int64_t *order_out) {
  LT_API_BEGIN
  if (n <= 0) fail(LT_E_VALUE, "empty graph");
  std::vector<int64_t> degree(n);
  int64_t start = 0;
  for (int64_t v = 0; v < n; ++v) {
    degree[v] = offsets[v + 1] - offsets[v];
    if (degree[v] < degree[start]) start = v;
  }
  std::vector<char> seen(n, 0);
  std::vector<int64_t> order;
  order.reserve(n);
  std::vector<int64_t> buf;
  size_t head = 0;
  order.push_back(start);
  seen[start] = 1;
  while (head < order.size()) {
    int64_t v = order[head++];
    buf.assign(nbrs + offsets[v], nbrs + offsets[v + 1]);
    std::sort(buf.begin(), buf.end(), [&](int64_t a, int64_t b) {
      return degree[a] != degree[b] ? degree[a] < degree[b] : a < b;
    });
    for (int64_t w : buf)
      if (!seen[w]) {
        seen[w] = 1;
        order.push_back(w);
      }
  }
  if ((int64_t)order.size() != n) fail(LT_E_VALUE, "graph is disconnected; renumbering unsupported");
  for (int64_t k = 0; k < n; ++k) order_out[k] = order[n - 1 - k];
  LT_API_END
}
