// lt_dg.cuh — elastic-wave DG kernels (placeholder until implemented)
#pragma once
#include "lt_kernels.cuh"

namespace lt {
template <class C>
__device__ __forceinline__ void dg_dispatch(int, C &) {}
inline void dg_validate(int, size_t j, const ChainView &, const LoopDesc &, const lt_arg *) {
  fail(LT_E_EXECUTION, "loop " + std::to_string(j) + ": DG kernels not built yet");
}
}  // namespace lt
