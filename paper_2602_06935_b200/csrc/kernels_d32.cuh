// Fast path placeholder (filled in by the specialised head_dim kernels).
#pragma once
#include "common.cuh"

namespace cotten {

template <typename T>
inline bool fast_fwd_supported(const OpParams&) {
  return false;
}
template <typename T>
inline bool fast_bwd_supported(const OpParams&) {
  return false;
}
template <typename T>
inline int launch_fast_fwd(const OpParams&, cudaStream_t) {
  return 0;
}
template <typename T>
inline int launch_fast_bwd(const OpParams&, cudaStream_t) {
  return 0;
}

}  // namespace cotten
