// Shared definitions for the cosine-attention kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cotten {

// Everything a forward or backward launch needs for the whole batch.  Units
// are (sequence b, head h) pairs, unit = b*H + h; element (b,h,i,j) lives at
// base[b*sb + h*sh + i*sn + j] (see include/cotten.h).
struct OpParams {
  const void* q;
  const void* k;
  const void* v;
  const void* dout;
  void* out;
  void* dq;
  void* dk;
  void* dv;
  const uint8_t* valid;  // [B][msb] bytes or nullptr
  void* saved_S;         // [B*H][D][D] accumulation type or nullptr
  void* saved_norms;     // [B*H][2][N] accumulation type or nullptr
  double* dm_unit;       // [B*H] or nullptr
  int* status;           // sticky per-device status word (COTTEN_STATUS_*)
  void* workspace;       // kernel-specific global scratch (generic bwd: G per unit)
  double* dm_total;      // tcgen05 bwd: fixed-order sum of dm_unit, written by the last CTA
  unsigned* grid_done;   // tcgen05 bwd: zeroed CTA-completion counter (dm_total)
  unsigned long long* tstamp;  // profiling (cotten_profile_begin): [0] min start, [1] max end (ns)
  int64_t B, H, N, D;
  int64_t sb, sh, sn, msb;
  double m, eps;
  const double* m_dev;    // device-resident m (cotten_*_mdev): read by the kernels instead of m
  int l2_ahead;           // tcgen05 producers: L2 prefetch distance in items (0 = off)
};

// The exponent m of s = exp(-m ln true_n): the host value, or the device-resident
// one (a learnable parameter updated on the device, encoder.cu) when given.
__device__ __forceinline__ double op_m(const OpParams& p) { return p.m_dev ? *p.m_dev : p.m; }

// Kernel time stamps from %globaltimer (ns) for the launch-duration profile
// (cotten_profile_begin): the first CTA start (after its programmatic
// dependency resolved) and the last warp exit, by atomics on a caller buffer
// that is baked into a CUDA graph like every other launch parameter.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct KernelStamp {
  unsigned long long* ts;
  __device__ explicit KernelStamp(const OpParams& p) : ts(p.tstamp) {
    if (ts && threadIdx.x == 0) atomicMin(ts, global_ns());
  }
  __device__ ~KernelStamp() {
    if (ts && (threadIdx.x & 31) == 0) atomicMax(ts + 1, global_ns());
  }
};

template <typename T>
struct AccOf {
  using type = float;
};
template <>
struct AccOf<double> {
  using type = double;
};

__device__ __forceinline__ float ld_acc(const float* p) { return *p; }
__device__ __forceinline__ double ld_acc(const double* p) { return *p; }
__device__ __forceinline__ float ld_acc(const __nv_bfloat16* p) { return __bfloat162float(*p); }

__device__ __forceinline__ void st_from(float* p, float x) { *p = x; }
__device__ __forceinline__ void st_from(double* p, double x) { *p = x; }
__device__ __forceinline__ void st_from(__nv_bfloat16* p, float x) { *p = __float2bfloat16_rn(x); }

template <typename A>
__device__ __forceinline__ A rsqrt_acc(A x);
template <>
__device__ __forceinline__ float rsqrt_acc<float>(float x) {
  return 1.0f / sqrtf(x);  // IEEE sqrt + div: within 1 ulp of the fp64 reference
}
template <>
__device__ __forceinline__ double rsqrt_acc<double>(double x) {
  return 1.0 / sqrt(x);
}

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

template <typename A>
__device__ __forceinline__ A warp_sum(A x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Count of valid rows of sequence b (attention.cpp:26-33), computed by the
// whole block; all threads get the result.
__device__ __forceinline__ int64_t block_true_count(const OpParams& p, int64_t b, int* s_cnt) {
  if (threadIdx.x == 0) *s_cnt = 0;
  __syncthreads();
  if (p.valid == nullptr) return p.N;
  int c = 0;
  const uint8_t* row = p.valid + b * p.msb;
  for (int64_t i = threadIdx.x; i < p.N; i += blockDim.x) c += row[i] != 0;
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(s_cnt, c);
  __syncthreads();
  return *s_cnt;
}

}  // namespace cotten
