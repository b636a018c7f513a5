// Device-resident Cotten4Rec encoder step around the cosine-attention
// operator: the SURVEY §8(f) rows (include/cotten_encoder.h).
//
//   f1  multi-head attention (attention.cpp:487-565): one QKV GEMM against the
//       per-head w_q/w_k/w_v packed side by side, the operator run IN PLACE on
//       the [B*n][3d] projection output (strides (n*3d, d_h, 3d): no
//       per-head copies, attention.cpp:506-508 / :518-523), W_o on the
//       operator's output read at the same stride; backward mirrors :539-561
//       (d_concat written at the operator's stride, one dQKV GEMM pair).
//   f2  post-norm block (encoder.cpp:183-257): fused (bias +) dropout +
//       residual + layer_norm kernels (:97-128), bias + GELU, their
//       backwards (layer_norm_backward :130-154, gelu_prime matrix.cpp:196-201),
//       deterministic column sums for the bias / gain gradients.
//   f3  query-slot gather (encoder.cpp:313-318), prediction_scores (:259-264)
//       and nll_loss (training.cpp:58-87) as one row-per-CTA softmax kernel.
//   f4  batch assembly (data.cpp:193-199 fit_sequence, training.cpp:15-56
//       mask_sequence, encoder.cpp:268-272 mask_for_ids) on the device.
//   plus clip_gradients + adam_step (training.cpp:89-143) on the flat buffer.
//
// GEMMs are cuBLAS SGEMM in plain FP32 (the projections are library GEMMs;
// K = d = 64 makes them HBM-bound); every other op is a kernel below.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cotten.h"
#include "../../include/cotten_encoder.h"

namespace cotten {
void set_last_error(const std::string& msg);  // cotten_capi.cu
int* status_word_for_current_device();         // cotten_capi.cu
}  // namespace cotten

namespace {

using cotten::set_last_error;

struct EncError {
  int code;
  std::string msg;
};
[[noreturn]] void enc_usage(const std::string& m) { throw EncError{COTTEN_ERR_USAGE, m}; }

#define ENC_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw EncError{COTTEN_ERR_INTERNAL, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)
#define ENC_BLAS(call)                                                                   \
  do {                                                                                   \
    cublasStatus_t s_ = (call);                                                          \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                     \
      throw EncError{COTTEN_ERR_INTERNAL, std::string(#call) + ": cublas status " +      \
                                              std::to_string((int)s_)};                  \
  } while (0)
#define ENC_OP(call)                                                                     \
  do {                                                                                   \
    int rc_ = (call);                                                                    \
    if (rc_ != COTTEN_OK) throw EncError{rc_, cotten_last_error()};                      \
  } while (0)

template <typename F>
int enc_guarded(F&& fn) {
  try {
    fn();
    return COTTEN_OK;
  } catch (const EncError& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return COTTEN_ERR_INTERNAL;
  }
}

// status bits of the encoder kernels (cotten_device_status)
constexpr int kStatusBadId = 2;         // embed: id outside [0, vocab+1] (DataError, encoder.cpp:88-90)
constexpr int kStatusNoRealItem = 4;    // assemble: a sequence without real items (training.cpp:21)
constexpr int kStatusQueryOverflow = 8; // assemble: K > max_queries

// ---- counter-based draws (dropout masks, the training mask) ----------------

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
// U[0, 1) with 53 random bits from (seed, stream, index).
__device__ __forceinline__ double u01(uint64_t seed, uint64_t stream, uint64_t idx) {
  const uint64_t x = splitmix64(splitmix64(seed ^ splitmix64(stream)) + idx);
  return (double)(x >> 11) * 0x1.0p-53;
}

// ---- small kernels ---------------------------------------------------------

// w_q[h], w_k[h], w_v[h] (3H consecutive d x d_h blocks, the reference's
// for_each_matrix order) <-> Wcat [d][3d], block blk at columns blk*d_h.
__global__ void pack_qkv_kernel(const float* __restrict__ w, float* __restrict__ wcat, int d,
                                int dh, int nblk, int unpack) {
  const int64_t total = (int64_t)nblk * d * dh;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int blk = (int)(e / ((int64_t)d * dh));
    const int rem = (int)(e - (int64_t)blk * d * dh);
    const int i = rem / dh, j = rem - i * dh;
    const int64_t c = (int64_t)i * nblk * dh + blk * dh + j;
    if (unpack)
      wcat[e] = w[c];  // (here w = dWcat, wcat = the gradient blocks)
    else
      wcat[c] = w[e];
  }
}

// E_t = item[id_t] + pos[t] (encoder.cpp:80-95), times the embedding dropout
// mask; valid = id != 0 (mask_for_ids, :268-272).
__global__ void embed_kernel(const int32_t* __restrict__ ids, int64_t R, int n, int d,
                             int64_t id_count, const float* __restrict__ item,
                             const float* __restrict__ pos, const float* __restrict__ mask,
                             float* __restrict__ x, uint8_t* __restrict__ valid, int* status) {
  const int64_t total = R * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d;
    const int j = (int)(e - r * d);
    const int t = (int)(r % n);
    const int32_t id = ids[r];
    float v;
    if (id < 0 || id >= id_count) {
      v = __int_as_float(0x7fc00000);
      if (j == 0) atomicOr(status, kStatusBadId);
    } else {
      v = item[(int64_t)id * d + j] + pos[(int64_t)t * d + j];
    }
    if (mask) v *= mask[e];
    x[e] = v;
    if (j == 0) valid[r] = id != 0;
  }
}

// Inverted-dropout masks {0, 1/(1-p)} (encoder.cpp:159-165), one float each.
__global__ void dropout_mask_kernel(float* __restrict__ mask, int64_t count, double p,
                                    uint64_t seed, uint64_t stream) {
  const float keep = (float)(1.0 / (1.0 - p));
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    mask[e] = u01(seed, stream, (uint64_t)e) < p ? 0.0f : keep;
}

__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sumd(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kLnMaxPerLane = 16;  // d <= 512

// s = (y + bias) * mask + x, then layer_norm (encoder.cpp:97-128): one warp
// per row, two-pass mean / variance like the reference.
__global__ void residual_ln_kernel(const float* __restrict__ y, int ldy,
                                   const float* __restrict__ bias, const float* __restrict__ mask,
                                   const float* __restrict__ x, const float* __restrict__ gain,
                                   const float* __restrict__ beta, float eps, int64_t R, int d,
                                   float* __restrict__ out, float* __restrict__ xhat,
                                   float* __restrict__ inv_std) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  float s[kLnMaxPerLane];
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < kLnMaxPerLane; ++k) {
    const int j = lane + 32 * k;
    s[k] = 0.f;
    if (j < d) {
      float v = y[r * ldy + j];
      if (bias) v += bias[j];
      if (mask) v *= mask[r * d + j];
      v += x[r * d + j];
      s[k] = v;
      sum += v;
    }
  }
  const float mean = warp_sumf(sum) / (float)d;
  float var = 0.f;
#pragma unroll
  for (int k = 0; k < kLnMaxPerLane; ++k) {
    const int j = lane + 32 * k;
    if (j < d) {
      const float c = s[k] - mean;
      var += c * c;
    }
  }
  var = warp_sumf(var) / (float)d;
  const float inv = 1.0f / sqrtf(var + eps);
#pragma unroll
  for (int k = 0; k < kLnMaxPerLane; ++k) {
    const int j = lane + 32 * k;
    if (j < d) {
      const float xh = (s[k] - mean) * inv;
      xhat[r * d + j] = xh;
      out[r * d + j] = gain[j] * xh + beta[j];
    }
  }
  if (lane == 0) inv_std[r] = inv;
}

// layer_norm_backward's dx (encoder.cpp:130-154) for one row per warp;
// optionally dx_masked = dx * mask (the dropout of the branch below).
__global__ void ln_bwd_kernel(const float* __restrict__ go, const float* __restrict__ xhat,
                              const float* __restrict__ inv_std, const float* __restrict__ gain,
                              int64_t R, int d, float* __restrict__ dx,
                              const float* __restrict__ mask, float* __restrict__ dx_masked,
                              int ld_masked) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  float dxh[kLnMaxPerLane], xh[kLnMaxPerLane];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int k = 0; k < kLnMaxPerLane; ++k) {
    const int j = lane + 32 * k;
    dxh[k] = 0.f;
    xh[k] = 0.f;
    if (j < d) {
      dxh[k] = go[r * d + j] * gain[j];
      xh[k] = xhat[r * d + j];
      s1 += dxh[k];
      s2 += dxh[k] * xh[k];
    }
  }
  s1 = warp_sumf(s1) / (float)d;
  s2 = warp_sumf(s2) / (float)d;
  const float inv = inv_std[r];
#pragma unroll
  for (int k = 0; k < kLnMaxPerLane; ++k) {
    const int j = lane + 32 * k;
    if (j < d) {
      const float v = inv * (dxh[k] - s1 - xh[k] * s2);
      dx[r * d + j] = v;
      if (dx_masked) dx_masked[r * ld_masked + j] = mask ? v * mask[r * d + j] : v;
    }
  }
}

__device__ __forceinline__ float gelu_f(float x) {  // matrix.cpp:191-194
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanhf(u));
}
__device__ __forceinline__ float gelu_prime_f(float x) {  // matrix.cpp:196-201
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  const float t = tanhf(u);
  const float du = 0.7978845608028654f * (1.0f + 3.0f * 0.044715f * x * x);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * du;
}

// z1 += b1 (kept for gelu_prime), a1 = gelu(z1)  (encoder.cpp:198-201)
__global__ void bias_gelu_kernel(float* __restrict__ z, const float* __restrict__ b,
                                 float* __restrict__ a, int64_t R, int c) {
  const int64_t total = R * c;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float v = z[e] + b[e % c];
    z[e] = v;
    a[e] = gelu_f(v);
  }
}
// da1 *= gelu_prime(z1)  (encoder.cpp:237)
__global__ void gelu_bwd_kernel(float* __restrict__ da, const float* __restrict__ z, int64_t total) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    da[e] *= gelu_prime_f(z[e]);
}
// Column sums over rows (bias / gain gradients, colsum_into encoder.cpp:167-172),
// deterministic: stage 1 writes per-(row-slab) partials in a fixed order,
// stage 2 adds them in slab order.  With b != nullptr it sums a * b.
constexpr int kColSlabs = 512;  // max row slabs (partials buffer: kColSlabs x C)
__global__ void colsum_stage1(const float* __restrict__ a, int lda, const float* __restrict__ b,
                              int ldb, int64_t R, int C, int slabs, float* __restrict__ part) {
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int w = threadIdx.x >> 5;  // 8 warps
  const int slab = blockIdx.y;
  const int64_t per = (R + slabs - 1) / slabs;
  const int64_t r0 = slab * per, r1 = min(R, r0 + per);
  // four independent accumulators (rows r, r + 8, r + 16, r + 24 of the warp's
  // stride-8 sequence) keep four loads in flight; fixed order, deterministic
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (c < C) {
    int64_t r = r0 + w;
    for (; r + 24 < r1; r += 32)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t rr = r + 8 * u;
        acc[u] += b ? a[rr * lda + c] * b[rr * ldb + c] : a[rr * lda + c];
      }
    for (; r < r1; r += 8) acc[0] += b ? a[r * lda + c] * b[r * ldb + c] : a[r * lda + c];
  }
  __shared__ float sh[8][32];
  sh[w][threadIdx.x & 31] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  __syncthreads();
  if (w == 0 && c < C) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += sh[k][threadIdx.x & 31];
    part[(int64_t)slab * C + c] = t;
  }
}
__global__ void colsum_stage2(const float* __restrict__ part, int C, int slabs, float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float t = 0.f;
  for (int s = 0; s < slabs; ++s) t += part[(int64_t)s * C + c];
  out[c] = t;
}

// gathered[k] = h[rows[k]] (encoder.cpp:313-318); rows < 0 are inactive (zeros)
__global__ void gather_rows_kernel(const float* __restrict__ h, const int32_t* __restrict__ rows,
                                   int64_t K, int d, float* __restrict__ out) {
  const int64_t total = K * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / d;
    const int j = (int)(e - k * d);
    const int32_t r = rows[k];
    out[e] = r >= 0 ? h[(int64_t)r * d + j] : 0.f;
  }
}
// dh[rows[k]] += dg[k] (encoder.cpp:343-347); the query slots of a sequence
// are distinct, so every target row is written by one k (dh zeroed first).
__global__ void scatter_rows_kernel(const float* __restrict__ dg, const int32_t* __restrict__ rows,
                                    int64_t K, int d, float* __restrict__ dh) {
  const int64_t total = K * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / d;
    const int j = (int)(e - k * d);
    const int32_t r = rows[k];
    if (r >= 0) dh[(int64_t)r * d + j] += dg[e];
  }
}

// logits += head_b (add_row_bias, encoder.cpp:262); rows of inactive slots zeroed.
__global__ void head_bias_kernel(float* __restrict__ logits, const float* __restrict__ b,
                                 const int32_t* __restrict__ rows, int64_t K, int C) {
  const int64_t total = K * (int64_t)C;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / C;
    logits[e] = rows[k] >= 0 ? logits[e] + b[e - k * C] : 0.f;
  }
}

// Number of active query rows (rows >= 0), one block.
__global__ void count_active_kernel(const int32_t* __restrict__ rows, int64_t K, int* out) {
  __shared__ int sh[32];
  int c = 0;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) c += rows[k] >= 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    *out = t;
  }
}

// nll_loss (training.cpp:58-87), one CTA per logits row: max and partition
// function over the item columns 1..V only, the row's loss into loss_rows,
// d_logits = softmax / K written over the logits (pad / mask columns 0).
constexpr int kNllThreads = 256;
__global__ void nll_kernel(float* __restrict__ logits, const int32_t* __restrict__ targets,
                           const int32_t* __restrict__ rows, const int* __restrict__ k_active,
                           int64_t V, double* __restrict__ loss_rows, int* status) {
  const int64_t k = blockIdx.x;
  const int64_t C = V + 2;
  float* row = logits + k * C;
  __shared__ float shf[32];
  __shared__ double shd[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (rows[k] < 0) {
    if (threadIdx.x == 0) loss_rows[k] = 0.0;
    return;
  }
  const int32_t t = targets[k];
  if (t < 1 || t > V) {  // UsageError in the reference (:69-70)
    if (threadIdx.x == 0) {
      loss_rows[k] = __longlong_as_double(0x7ff8000000000000ll);
      atomicOr(status, kStatusBadId);
    }
    return;
  }
  float mx = -INFINITY;
  for (int64_t j = 1 + threadIdx.x; j <= V; j += blockDim.x) mx = fmaxf(mx, row[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) shf[w] = mx;
  __syncthreads();
  mx = shf[0];
  for (int i = 1; i < nw; ++i) mx = fmaxf(mx, shf[i]);
  double z = 0.0;
  for (int64_t j = 1 + threadIdx.x; j <= V; j += blockDim.x) z += (double)expf(row[j] - mx);
  z = warp_sumd(z);
  if (lane == 0) shd[w] = z;
  __syncthreads();
  z = 0.0;
  for (int i = 0; i < nw; ++i) z += shd[i];  // fixed order
  const float xt = row[t];
  __syncthreads();
  const double inv_k = 1.0 / (double)*k_active;
  const float iz = (float)(1.0 / z);
  for (int64_t j = threadIdx.x; j < C; j += blockDim.x) {
    float g = 0.f;
    if (j >= 1 && j <= V) g = (float)((double)(expf(row[j] - mx) * iz) * inv_k);
    if (j == t) g -= (float)inv_k;
    row[j] = g;
  }
  if (threadIdx.x == 0) loss_rows[k] = -((double)xt - (double)mx - log(z));
}
// loss = sum(loss_rows) / K in a fixed order (one block)
__global__ void loss_reduce_kernel(const double* __restrict__ loss_rows, int64_t K,
                                   const int* __restrict__ k_active, double* loss) {
  __shared__ double sh[32];
  double t = 0.0;
  const int64_t per = (K + blockDim.x - 1) / blockDim.x;
  const int64_t lo = threadIdx.x * per, hi = min(K, lo + per);
  for (int64_t k = lo; k < hi; ++k) t += loss_rows[k];
  t = warp_sumd(t);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    *loss = s / (double)*k_active;
  }
}

// Embedding backward (encoder.cpp:363-373): item rows by atomics (ids repeat
// across sequences), position rows as deterministic sums over the batch.
__global__ void embed_bwd_item_kernel(const float* __restrict__ dh, const float* __restrict__ mask,
                                      const int32_t* __restrict__ ids, int64_t R, int d,
                                      int64_t id_count, float* __restrict__ d_item) {
  const int64_t total = R * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d;
    const int j = (int)(e - r * d);
    const int32_t id = ids[r];
    if (id < 0 || id >= id_count) continue;
    const float g = mask ? dh[e] * mask[e] : dh[e];
    atomicAdd(d_item + (int64_t)id * d + j, g);
  }
}
__global__ void embed_bwd_pos_kernel(const float* __restrict__ dh, const float* __restrict__ mask,
                                     int64_t B, int n, int d, float* __restrict__ d_pos) {
  const int64_t total = (int64_t)n * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    float t = 0.f;
    for (int64_t b = 0; b < B; ++b) {
      const int64_t i = b * total + e;
      t += mask ? dh[i] * mask[i] : dh[i];
    }
    d_pos[e] = t;
  }
}

// ---- clip_gradients + adam_step (training.cpp:89-143) ----------------------
constexpr int kNormBlocks = 296;
__global__ void sumsq_stage1(const float* __restrict__ g, int64_t count, double* __restrict__ part) {
  __shared__ double sh[32];
  double t = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    t += (double)g[e] * (double)g[e];
  t = warp_sumd(t);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    part[blockIdx.x] = s;
  }
}
// norm = sqrt(sum of partials + sum of the m grads^2); scale = max/norm when
// norm > max * (1 + 1e-12)  (training.cpp:89-102)
__global__ void clip_scale_kernel(const double* __restrict__ part, int nparts,
                                  const double* __restrict__ gm, int L, double max_norm,
                                  double* __restrict__ scale_out, double* __restrict__ norm_out) {
  if (threadIdx.x != 0) return;
  double sq = 0.0;
  for (int i = 0; i < nparts; ++i) sq += part[i];
  for (int l = 0; l < L; ++l) sq += gm[l] * gm[l];
  const double norm = sqrt(sq);
  *scale_out = norm <= max_norm * (1.0 + 1e-12) ? 1.0 : max_norm / norm;
  if (norm_out) *norm_out = norm;
}
// adam_update (training.cpp:111-119) with the clip scale applied to the
// gradient (clip_gradients rescales the gradients in place first)
__global__ void adam_kernel(float* __restrict__ p, float* __restrict__ g, float* __restrict__ m1,
                            float* __restrict__ m2, int64_t count, const double* __restrict__ scale,
                            float lr, float wd, float b1, float b2, float eps, float bc1, float bc2) {
  const float sc = (float)*scale;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float gr = g[e] * sc;
    g[e] = gr;
    float w = p[e];
    w -= lr * wd * w;
    const float a = b1 * m1[e] + (1.f - b1) * gr;
    const float v = b2 * m2[e] + (1.f - b2) * gr * gr;
    m1[e] = a;
    m2[e] = v;
    w -= lr * (a / bc1) / (sqrtf(v / bc2) + eps);
    p[e] = w;
  }
}
__global__ void adam_m_kernel(double* __restrict__ p, double* __restrict__ g, double* __restrict__ m1,
                              double* __restrict__ m2, int L, const double* __restrict__ scale,
                              double lr, double wd, double b1, double b2, double eps, double bc1,
                              double bc2) {
  const int l = threadIdx.x;
  if (l >= L) return;
  const double gr = g[l] * *scale;
  g[l] = gr;
  double w = p[l];
  w -= lr * wd * w;
  m1[l] = b1 * m1[l] + (1.0 - b1) * gr;
  m2[l] = b2 * m2[l] + (1.0 - b2) * gr * gr;
  w -= lr * (m1[l] / bc1) / (sqrt(m2[l] / bc2) + eps);
  p[l] = w;
}

// ---- batch assembly (f4) -----------------------------------------------------
// One warp per sequence.  fit_sequence (data.cpp:193-199): the last
// min(len, n) items, left-padded with 0.  mask_sequence (training.cpp:15-56):
// eval masks the last real slot; train draws every real slot with
// probability p_mask, redrawing the whole pass until one is drawn, and
// (bert) corrupts a drawn slot to the mask token (80 %), a random item
// (10 %) or keeps it (10 %).  Phase 0 counts the slots, phase 1 writes them
// at the sequence's offset.
__device__ __forceinline__ bool draw_slot(uint64_t seed, int64_t b, int i, int round, double p) {
  return u01(seed, 0xA000000000ull + (uint64_t)round, (uint64_t)b * 0x100000000ull + (uint64_t)i) < p;
}
__global__ void assemble_kernel(const int32_t* __restrict__ items, const int64_t* __restrict__ offs,
                                int64_t B, int n, int train, double p_mask, int bert,
                                uint64_t seed, int64_t vocab, int phase,
                                int32_t* __restrict__ counts, const int32_t* __restrict__ starts,
                                int32_t* __restrict__ ids, uint8_t* __restrict__ valid,
                                int32_t* __restrict__ qrows, int32_t* __restrict__ targets,
                                int64_t max_q, int* status) {
  const int lane = threadIdx.x & 31;
  const int64_t b = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const int64_t o0 = offs[b], len = offs[b + 1] - o0;
  const int64_t take = len < n ? len : n;
  const int pad = (int)(n - take);
  auto orig = [&](int i) -> int32_t {
    return i < pad ? 0 : items[o0 + len - take + (i - pad)];
  };
  // the round whose draws select >= 1 slot (eval: round -1 = the last real slot)
  int round = -1, last = -1;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const unsigned bal = __ballot_sync(0xffffffffu, i < n && orig(i) != 0);
    if (bal) last = i0 + 31 - __clz(bal);
  }
  if (last < 0) {  // DataError: no real items (training.cpp:21)
    if (phase == 0 && lane == 0) {
      atomicOr(status, kStatusNoRealItem);
      counts[b] = 0;
    }
    if (phase == 1)
      for (int i = lane; i < n; i += 32) {
        ids[b * n + i] = 0;
        valid[b * n + i] = 0;
      }
    return;
  }
  if (train) {
    for (round = 0;; ++round) {
      bool any = false;
      for (int i0 = 0; i0 < n && !any; i0 += 32) {
        const int i = i0 + lane;
        const bool hit = i < n && orig(i) != 0 && draw_slot(seed, b, i, round, p_mask);
        any = __any_sync(0xffffffffu, hit);
      }
      if (any) break;
    }
  }
  int base = phase == 1 ? starts[b] : 0, cnt = 0;
  const int32_t mask_token = (int32_t)(vocab + 1);
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    int32_t id = i < n ? orig(i) : 0;
    const bool hit = i < n && id != 0 &&
                     (train ? draw_slot(seed, b, i, round, p_mask) : i == last);
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (phase == 1 && i < n) {
      valid[b * n + i] = id != 0;
      int32_t out_id = id;
      if (hit) {
        const int k = base + cnt + __popc(bal & ((1u << lane) - 1u));
        if (k < max_q) {
          qrows[k] = (int32_t)(b * n + i);
          targets[k] = id;
        }
        out_id = mask_token;
        if (train && bert) {
          const double roll = u01(seed, 0xB000000000ull + (uint64_t)round,
                                  (uint64_t)b * 0x100000000ull + (uint64_t)i);
          if (roll >= 0.9)
            out_id = id;
          else if (roll >= 0.8)
            out_id = 1 + (int32_t)(splitmix64(seed ^ ((uint64_t)b << 32) ^ (uint64_t)i ^
                                              0xC000000000ull) % (uint64_t)vocab);
        }
      }
      ids[b * n + i] = out_id;
    }
    cnt += __popc(bal);
  }
  if (phase == 0 && lane == 0) counts[b] = cnt;
}
// exclusive scan of the per-sequence counts (one block), K total, overflow bit
__global__ void scan_counts_kernel(const int32_t* __restrict__ counts, int64_t B,
                                   int32_t* __restrict__ starts, int32_t* __restrict__ k_total,
                                   int64_t max_q, int* status) {
  __shared__ int32_t sh[1024];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < B; c0 += blockDim.x) {
    const int64_t i = c0 + threadIdx.x;
    const int32_t v = i < B ? counts[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {
      const int32_t t = threadIdx.x >= (unsigned)o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < B) starts[i] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += sh[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *k_total = carry;
    if (carry > max_q) atomicOr(status, kStatusQueryOverflow);
  }
}
// query rows [K, max_q) of an assembled batch: inactive
__global__ void fill_inactive_kernel(int32_t* __restrict__ qrows, const int32_t* __restrict__ k_total,
                                     int64_t max_q) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < max_q;
       k += (int64_t)gridDim.x * blockDim.x)
    if (k >= *k_total) qrows[k] = -1;
}

inline unsigned grid_for(int64_t total, int threads = 256) {
  int64_t g = (total + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

// ---- the encoder object -------------------------------------------------------

struct cotten_encoder {
  cotten_enc_config cfg{};
  int64_t max_batch = 0, max_q = 0;
  int64_t d = 0, dh = 0, H = 0, L = 0, C = 0, id_count = 0;
  // flat layout (for_each_matrix order)
  std::vector<int64_t> off, rows, cols;
  int64_t count = 0;
  // per-layer tensor indices
  struct LayerIdx {
    int wq, wo, w1, b1, w2, b2, g1, be1, g2, be2;
  };
  std::vector<LayerIdx> li;
  int t_item = 0, t_pos = 1, t_head_w = 0, t_head_b = 0;
  float *params = nullptr, *grads = nullptr, *adam1 = nullptr, *adam2 = nullptr;
  double *m = nullptr, *gm = nullptr, *m1m = nullptr, *m2m = nullptr;
  long adam_step = 0;
  cublasHandle_t blas = nullptr;
  // activations (sized for max_batch * max_seq rows)
  struct Layer {
    float *x, *qkv, *o3, *S, *xhat1, *inv1, *h1, *z1, *a1, *xhat2, *inv2;
  };
  std::vector<Layer> act;
  float* x_final = nullptr;  // output of the last block
  float *wcat = nullptr, *dwcat = nullptr;  // [L][d][3d]
  float* masks = nullptr;    // [(1 + 2L)][R][d]
  uint8_t* valid = nullptr;
  const int32_t* ids = nullptr;  // the last forward's ids (embedding backward)
  float *tmp_d = nullptr, *tmp_d2 = nullptr, *dgrad = nullptr, *d4 = nullptr, *do3 = nullptr,
        *dqkv = nullptr;
  float *gathered = nullptr, *logits = nullptr, *dgath = nullptr;
  double* loss_rows = nullptr;
  int* k_active = nullptr;
  float* col_part = nullptr;
  double *norm_part = nullptr, *clip_scale = nullptr;
  int32_t *asm_counts = nullptr, *asm_starts = nullptr;
  std::vector<void*> allocs;
  // the last forward
  int64_t B = 0, n = 0, K = 0;
  const int32_t* qrows = nullptr;
  bool train = false, have_fwd = false;
  const float* mask_src = nullptr;  // masks used by the last forward (nullptr = none)

  float* P(int t) { return params + off[t]; }
  float* G(int t) { return grads + off[t]; }
  template <typename T>
  T* alloc(size_t elems) {
    void* p = nullptr;
    ENC_CUDA(cudaMalloc(&p, elems * sizeof(T) + 16));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  ~cotten_encoder() {
    for (void* p : allocs) cudaFree(p);
    if (blas) cublasDestroy(blas);
  }
};

namespace {

// Row-major GEMM: C[M,N] (ldc) = op(A)[M,K] op(B)[K,N] + beta C.
void gemm_rm(cublasHandle_t h, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A,
             int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, float beta = 0.f) {
  const float one = 1.f;
  ENC_BLAS(cublasSgemm(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, (int)N,
                       (int)M, (int)K, &one, B, (int)ldb, A, (int)lda, &beta, C, (int)ldc));
}

void colsum(cotten_encoder* e, const float* a, int64_t lda, const float* b, int64_t ldb, int64_t R,
            int64_t C, float* out, cudaStream_t st) {
  // ~4 CTAs per SM over (column groups x row slabs), >= 64 rows per slab
  const int cg = (int)((C + 31) / 32);
  const int slabs = (int)std::max<int64_t>(1, std::min<int64_t>({kColSlabs, 592 / cg, (R + 63) / 64}));
  dim3 g1((unsigned)cg, (unsigned)slabs);
  colsum_stage1<<<g1, 256, 0, st>>>(a, (int)lda, b, (int)ldb, R, (int)C, slabs, e->col_part);
  colsum_stage2<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(e->col_part, (int)C, slabs, out);
}

cotten_desc op_desc(const cotten_encoder* e, int64_t B, int64_t n) {
  cotten_desc d{};
  d.batch = B;
  d.heads = e->H;
  d.seq_len = n;
  d.head_dim = e->dh;
  d.dtype = COTTEN_F32;
  d.eps = e->cfg.attn_eps;
  d.stride_b = n * 3 * e->d;  // the [B*n][3d] projection output, in place
  d.stride_h = e->dh;
  d.stride_n = 3 * e->d;
  d.mask_stride_b = n;
  return d;
}

}  // namespace

extern "C" {

int cotten_enc_create(const cotten_enc_config* cfg, int64_t max_batch, int64_t max_queries,
                      cotten_encoder** out) {
  return enc_guarded([&] {
    if (!cfg || !out) enc_usage("cotten_enc_create: null argument");
    if (cfg->vocab < 1) enc_usage("init_encoder: vocab must be >= 1");
    if (cfg->layers < 1) enc_usage("init_encoder: layers must be >= 1");
    if (cfg->dim < 1 || cfg->heads < 1 || cfg->dim % cfg->heads != 0)
      enc_usage("init_encoder: dim must be a positive multiple of heads (shape)");
    if (cfg->dim > 32 * kLnMaxPerLane) enc_usage("cotten_enc_create: dim > 512 unsupported");
    if (cfg->max_seq < 1 || max_batch < 1 || max_queries < 1)
      enc_usage("cotten_enc_create: max_seq, max_batch, max_queries must be >= 1");
    if (!(cfg->dropout >= 0.0 && cfg->dropout < 1.0)) enc_usage("cotten_enc_create: dropout in [0,1)");
    auto* e = new cotten_encoder();
    try {
      e->cfg = *cfg;
      e->max_batch = max_batch;
      e->max_q = max_queries;
      e->d = cfg->dim;
      e->H = cfg->heads;
      e->dh = e->d / e->H;
      e->L = cfg->layers;
      e->id_count = cfg->vocab + 2;
      e->C = e->id_count;
      const int64_t d = e->d;
      auto add = [&](int64_t r, int64_t c) {
        e->rows.push_back(r);
        e->cols.push_back(c);
        return (int)e->rows.size() - 1;
      };
      e->t_item = add(e->id_count, d);
      e->t_pos = add(cfg->max_seq, d);
      for (int64_t l = 0; l < e->L; ++l) {
        cotten_encoder::LayerIdx x{};
        x.wq = add(d, e->dh);
        for (int64_t k = 1; k < 3 * e->H; ++k) add(d, e->dh);  // rest of w_q, w_k, w_v
        x.wo = add(d, d);
        x.w1 = add(d, 4 * d);
        x.b1 = add(1, 4 * d);
        x.w2 = add(4 * d, d);
        x.b2 = add(1, d);
        x.g1 = add(1, d);
        x.be1 = add(1, d);
        x.g2 = add(1, d);
        x.be2 = add(1, d);
        e->li.push_back(x);
      }
      e->t_head_w = add(d, e->id_count);
      e->t_head_b = add(1, e->id_count);
      e->off.assign(e->rows.size() + 1, 0);
      for (size_t i = 0; i < e->rows.size(); ++i) e->off[i + 1] = e->off[i] + e->rows[i] * e->cols[i];
      e->count = e->off.back();

      ENC_BLAS(cublasCreate(&e->blas));
      ENC_BLAS(cublasSetMathMode(e->blas, CUBLAS_PEDANTIC_MATH));  // plain FP32, no TF32
      const int64_t R = max_batch * cfg->max_seq;
      const int64_t L = e->L;
      e->params = e->alloc<float>(e->count);
      e->grads = e->alloc<float>(e->count);
      e->adam1 = e->alloc<float>(e->count);
      e->adam2 = e->alloc<float>(e->count);
      e->m = e->alloc<double>(L);
      e->gm = e->alloc<double>(L);
      e->m1m = e->alloc<double>(L);
      e->m2m = e->alloc<double>(L);
      ENC_CUDA(cudaMemset(e->params, 0, e->count * sizeof(float)));
      ENC_CUDA(cudaMemset(e->grads, 0, e->count * sizeof(float)));
      ENC_CUDA(cudaMemset(e->adam1, 0, e->count * sizeof(float)));
      ENC_CUDA(cudaMemset(e->adam2, 0, e->count * sizeof(float)));
      std::vector<double> ones(L, 1.0);  // attn.m = 1.0 (encoder.cpp:45)
      ENC_CUDA(cudaMemcpy(e->m, ones.data(), L * sizeof(double), cudaMemcpyHostToDevice));
      ENC_CUDA(cudaMemset(e->gm, 0, L * sizeof(double)));
      ENC_CUDA(cudaMemset(e->m1m, 0, L * sizeof(double)));
      ENC_CUDA(cudaMemset(e->m2m, 0, L * sizeof(double)));
      e->act.resize(L);
      for (auto& a : e->act) {
        a.x = e->alloc<float>(R * d);
        a.qkv = e->alloc<float>(R * 3 * d);
        a.o3 = e->alloc<float>(R * 3 * d);
        a.S = e->alloc<float>(max_batch * e->H * e->dh * e->dh);
        a.xhat1 = e->alloc<float>(R * d);
        a.inv1 = e->alloc<float>(R);
        a.h1 = e->alloc<float>(R * d);
        a.z1 = e->alloc<float>(R * 4 * d);
        a.a1 = e->alloc<float>(R * 4 * d);
        a.xhat2 = e->alloc<float>(R * d);
        a.inv2 = e->alloc<float>(R);
      }
      e->x_final = e->alloc<float>(R * d);
      e->wcat = e->alloc<float>(L * 3 * d * d);
      e->dwcat = e->alloc<float>(L * 3 * d * d);
      if (cfg->dropout > 0.0) e->masks = e->alloc<float>((1 + 2 * L) * R * d);
      e->valid = e->alloc<uint8_t>(R);
      e->tmp_d = e->alloc<float>(R * d);
      e->tmp_d2 = e->alloc<float>(R * d);
      e->dgrad = e->alloc<float>(R * d);
      e->d4 = e->alloc<float>(R * 4 * d);
      e->do3 = e->alloc<float>(R * 3 * d);
      e->dqkv = e->alloc<float>(R * 3 * d);
      e->gathered = e->alloc<float>(max_queries * d);
      e->logits = e->alloc<float>(max_queries * e->C);
      e->dgath = e->alloc<float>(max_queries * d);
      e->loss_rows = e->alloc<double>(max_queries);
      e->k_active = e->alloc<int>(1);
      const int64_t cmax = std::max<int64_t>(4 * d, e->C);
      e->col_part = e->alloc<float>(kColSlabs * cmax);
      e->norm_part = e->alloc<double>(kNormBlocks);
      e->clip_scale = e->alloc<double>(1);
      e->asm_counts = e->alloc<int32_t>(max_batch);
      e->asm_starts = e->alloc<int32_t>(max_batch);
      *out = e;
    } catch (...) {
      delete e;
      throw;
    }
  });
}

int cotten_enc_destroy(cotten_encoder* enc) {
  return enc_guarded([&] { delete enc; });
}

int64_t cotten_enc_tensor_count(const cotten_encoder* enc) {
  return enc ? (int64_t)enc->rows.size() : -1;
}
int cotten_enc_layout(const cotten_encoder* enc, int64_t* offsets, int64_t* rows, int64_t* cols) {
  return enc_guarded([&] {
    if (!enc) enc_usage("cotten_enc_layout: null encoder");
    for (size_t i = 0; i < enc->rows.size(); ++i) {
      if (offsets) offsets[i] = enc->off[i];
      if (rows) rows[i] = enc->rows[i];
      if (cols) cols[i] = enc->cols[i];
    }
    if (offsets) offsets[enc->rows.size()] = enc->count;
  });
}
float* cotten_enc_params(cotten_encoder* enc) { return enc ? enc->params : nullptr; }
float* cotten_enc_grads(cotten_encoder* enc) { return enc ? enc->grads : nullptr; }
double* cotten_enc_m_params(cotten_encoder* enc) { return enc ? enc->m : nullptr; }
double* cotten_enc_m_grads(cotten_encoder* enc) { return enc ? enc->gm : nullptr; }
float* cotten_enc_logits(cotten_encoder* enc) { return enc ? enc->logits : nullptr; }

int cotten_enc_assemble(cotten_encoder* e, const int32_t* items, const int64_t* offsets, int64_t B,
                        int64_t n, int train, double p_mask, int bert, uint64_t seed, int32_t* ids,
                        uint8_t* valid, int32_t* query_rows, int32_t* targets, int32_t* k_total,
                        void* stream) {
  return enc_guarded([&] {
    if (!e || !items || !offsets || !ids || !valid || !query_rows || !targets || !k_total)
      enc_usage("cotten_enc_assemble: null argument");
    if (B < 1 || B > e->max_batch) enc_usage("cotten_enc_assemble: batch size outside [1, max_batch]");
    if (n < 1) enc_usage("fit_sequence: length must be >= 1");
    if (train && !(p_mask > 0.0 && p_mask < 1.0)) enc_usage("mask_sequence: p_mask must be in (0,1)");
    cudaStream_t st = (cudaStream_t)stream;
    int* status = cotten::status_word_for_current_device();
    const unsigned g = (unsigned)((B + 7) / 8);
    assemble_kernel<<<g, 256, 0, st>>>(items, offsets, B, (int)n, train, p_mask, bert, seed,
                                       e->cfg.vocab, 0, e->asm_counts, nullptr, ids, valid,
                                       query_rows, targets, e->max_q, status);
    scan_counts_kernel<<<1, 1024, 0, st>>>(e->asm_counts, B, e->asm_starts, k_total, e->max_q, status);
    assemble_kernel<<<g, 256, 0, st>>>(items, offsets, B, (int)n, train, p_mask, bert, seed,
                                       e->cfg.vocab, 1, e->asm_counts, e->asm_starts, ids, valid,
                                       query_rows, targets, e->max_q, status);
    fill_inactive_kernel<<<grid_for(e->max_q), 256, 0, st>>>(query_rows, k_total, e->max_q);
    ENC_CUDA(cudaGetLastError());
  });
}

int cotten_enc_forward(cotten_encoder* e, const int32_t* ids, int64_t B, int64_t n,
                       const int32_t* query_rows, int64_t K, int train, uint64_t dropout_seed,
                       const float* dropout_masks, float* logits, void* stream) {
  return enc_guarded([&] {
    if (!e || !ids || !query_rows) enc_usage("model_forward: null argument");
    if (B < 1 || B > e->max_batch) enc_usage("model_forward: batch size outside [1, max_batch]");
    if (n < 1 || n > e->cfg.max_seq) enc_usage("embed: sequence longer than max_seq");
    if (K < 1 || K > e->max_q) enc_usage("model_forward: query count outside [1, max_queries]");
    cudaStream_t st = (cudaStream_t)stream;
    ENC_BLAS(cublasSetStream(e->blas, st));
    int* status = cotten::status_word_for_current_device();
    const int64_t d = e->d, R = B * n, L = e->L;
    const bool drop = train && e->cfg.dropout > 0.0;
    e->B = B;
    e->n = n;
    e->K = K;
    e->qrows = query_rows;
    e->ids = ids;
    e->train = train != 0;
    const float* masks = nullptr;
    if (drop) {
      if (dropout_masks) {
        masks = dropout_masks;
      } else {
        const int64_t cnt = (1 + 2 * L) * R * d;
        dropout_mask_kernel<<<grid_for(cnt), 256, 0, st>>>(e->masks, cnt, e->cfg.dropout,
                                                           dropout_seed, 0xD0);
        masks = e->masks;
      }
    }
    e->mask_src = masks;
    auto mask_of = [&](int64_t i) -> const float* { return masks ? masks + i * R * d : nullptr; };

    // W_q / W_k / W_v of every layer side by side
    for (int64_t l = 0; l < L; ++l)
      pack_qkv_kernel<<<grid_for(3 * d * d), 256, 0, st>>>(e->P(e->li[l].wq), e->wcat + l * 3 * d * d,
                                                           (int)d, (int)e->dh, (int)(3 * e->H), 0);
    embed_kernel<<<grid_for(R * d), 256, 0, st>>>(ids, R, (int)n, (int)d, e->id_count, e->P(e->t_item),
                                                  e->P(e->t_pos), mask_of(0), e->act[0].x, e->valid,
                                                  status);
    ENC_CUDA(cudaGetLastError());
    const cotten_desc od = op_desc(e, B, n);
    const unsigned ln_grid = (unsigned)((R + 7) / 8);
    for (int64_t l = 0; l < L; ++l) {
      auto& a = e->act[l];
      const auto& ix = e->li[l];
      float* x_next = l + 1 < L ? e->act[l + 1].x : e->x_final;
      // multi_head_attention (attention.cpp:487-526)
      gemm_rm(e->blas, false, false, R, 3 * d, d, a.x, d, e->wcat + l * 3 * d * d, 3 * d, a.qkv, 3 * d);
      ENC_OP(cotten_fwd_mdev(&od, a.qkv, a.qkv + d, a.qkv + 2 * d, e->valid, e->m + l, a.o3, a.S,
                             nullptr, st));
      gemm_rm(e->blas, false, false, R, d, d, a.o3, 3 * d, e->P(ix.wo), d, e->tmp_d, d);
      // dropout + residual + LN1 (encoder.cpp:190-196)
      residual_ln_kernel<<<ln_grid, 256, 0, st>>>(e->tmp_d, (int)d, nullptr, mask_of(1 + 2 * l), a.x,
                                                   e->P(ix.g1), e->P(ix.be1), (float)e->cfg.ln_eps, R,
                                                   (int)d, a.h1, a.xhat1, a.inv1);
      // FFN (encoder.cpp:198-203)
      gemm_rm(e->blas, false, false, R, 4 * d, d, a.h1, d, e->P(ix.w1), 4 * d, a.z1, 4 * d);
      bias_gelu_kernel<<<grid_for(R * 4 * d), 256, 0, st>>>(a.z1, e->P(ix.b1), a.a1, R, (int)(4 * d));
      gemm_rm(e->blas, false, false, R, d, 4 * d, a.a1, 4 * d, e->P(ix.w2), d, e->tmp_d, d);
      // bias + dropout + residual + LN2 (encoder.cpp:204-211)
      residual_ln_kernel<<<ln_grid, 256, 0, st>>>(e->tmp_d, (int)d, e->P(ix.b2), mask_of(2 + 2 * l),
                                                   a.h1, e->P(ix.g2), e->P(ix.be2),
                                                   (float)e->cfg.ln_eps, R, (int)d, x_next, a.xhat2,
                                                   a.inv2);
      ENC_CUDA(cudaGetLastError());
    }
    // gather + prediction_scores (encoder.cpp:313-324, :259-264)
    gather_rows_kernel<<<grid_for(K * d), 256, 0, st>>>(e->x_final, query_rows, K, (int)d, e->gathered);
    float* lg = logits ? logits : e->logits;
    gemm_rm(e->blas, false, false, K, e->C, d, e->gathered, d, e->P(e->t_head_w), e->C, lg, e->C);
    head_bias_kernel<<<grid_for(K * e->C), 256, 0, st>>>(lg, e->P(e->t_head_b), query_rows, K, (int)e->C);
    count_active_kernel<<<1, 1024, 0, st>>>(query_rows, K, e->k_active);
    if (lg != e->logits)
      ENC_CUDA(cudaMemcpyAsync(e->logits, lg, K * e->C * sizeof(float), cudaMemcpyDeviceToDevice, st));
    ENC_CUDA(cudaGetLastError());
    e->have_fwd = true;
  });
}

int cotten_enc_loss(cotten_encoder* e, const int32_t* targets, double* loss, void* stream) {
  return enc_guarded([&] {
    if (!e || !targets || !loss) enc_usage("nll_loss: null argument");
    if (!e->have_fwd) enc_usage("nll_loss: no forward to take the loss of");
    cudaStream_t st = (cudaStream_t)stream;
    int* status = cotten::status_word_for_current_device();
    nll_kernel<<<(unsigned)e->K, kNllThreads, 0, st>>>(e->logits, targets, e->qrows, e->k_active,
                                                       e->cfg.vocab, e->loss_rows, status);
    loss_reduce_kernel<<<1, 256, 0, st>>>(e->loss_rows, e->K, e->k_active, loss);
    ENC_CUDA(cudaGetLastError());
  });
}

int cotten_enc_backward(cotten_encoder* e, const float* d_logits, void* stream) {
  return enc_guarded([&] {
    if (!e) enc_usage("model_backward: null encoder");
    if (!e->have_fwd) enc_usage("model_backward: cache missing");
    cudaStream_t st = (cudaStream_t)stream;
    ENC_BLAS(cublasSetStream(e->blas, st));
    const int64_t d = e->d, R = e->B * e->n, L = e->L, K = e->K, C = e->C;
    const float* dl = d_logits ? d_logits : e->logits;
    const float* masks = e->mask_src;
    auto mask_of = [&](int64_t i) -> const float* { return masks ? masks + i * R * d : nullptr; };
    // head (encoder.cpp:333-336)
    gemm_rm(e->blas, true, false, d, C, K, e->gathered, d, dl, C, e->G(e->t_head_w), C);
    colsum(e, dl, C, nullptr, 0, K, C, e->G(e->t_head_b), st);
    gemm_rm(e->blas, false, true, K, d, C, dl, C, e->P(e->t_head_w), C, e->dgath, d);
    ENC_CUDA(cudaMemsetAsync(e->dgrad, 0, R * d * sizeof(float), st));
    scatter_rows_kernel<<<grid_for(K * d), 256, 0, st>>>(e->dgath, e->qrows, K, (int)d, e->dgrad);
    const cotten_desc od = op_desc(e, e->B, e->n);
    const unsigned ln_grid = (unsigned)((R + 7) / 8);
    for (int64_t l = L - 1; l >= 0; --l) {
      auto& a = e->act[l];
      const auto& ix = e->li[l];
      // LN2 backward (encoder.cpp:223-224): ds2 -> tmp_d; dz2 = ds2 * drop2 -> tmp_d2
      ln_bwd_kernel<<<ln_grid, 256, 0, st>>>(e->dgrad, a.xhat2, a.inv2, e->P(ix.g2), R, (int)d, e->tmp_d,
                                             mask_of(2 + 2 * l), e->tmp_d2, (int)d);
      colsum(e, e->dgrad, d, a.xhat2, d, R, d, e->G(ix.g2), st);
      colsum(e, e->dgrad, d, nullptr, 0, R, d, e->G(ix.be2), st);
      // FFN branch (encoder.cpp:226-240)
      gemm_rm(e->blas, true, false, 4 * d, d, R, a.a1, 4 * d, e->tmp_d2, d, e->G(ix.w2), d);
      colsum(e, e->tmp_d2, d, nullptr, 0, R, d, e->G(ix.b2), st);
      gemm_rm(e->blas, false, true, R, 4 * d, d, e->tmp_d2, d, e->P(ix.w2), d, e->d4, 4 * d);
      gelu_bwd_kernel<<<grid_for(R * 4 * d), 256, 0, st>>>(e->d4, a.z1, R * 4 * d);
      gemm_rm(e->blas, true, false, d, 4 * d, R, a.h1, d, e->d4, 4 * d, e->G(ix.w1), 4 * d);
      colsum(e, e->d4, 4 * d, nullptr, 0, R, 4 * d, e->G(ix.b1), st);
      // dh1 = da1 W1^T + ds2 (residual): ds2 already in tmp_d, beta = 1
      gemm_rm(e->blas, false, true, R, d, 4 * d, e->d4, 4 * d, e->P(ix.w1), 4 * d, e->tmp_d, d, 1.f);
      // LN1 backward (encoder.cpp:242-243): ds1 -> dh (kept for the residual),
      // d_attn = ds1 * drop1 -> tmp_d2
      ln_bwd_kernel<<<ln_grid, 256, 0, st>>>(e->tmp_d, a.xhat1, a.inv1, e->P(ix.g1), R, (int)d, e->dgrad,
                                             mask_of(1 + 2 * l), e->tmp_d2, (int)d);
      colsum(e, e->tmp_d, d, a.xhat1, d, R, d, e->G(ix.g1), st);
      colsum(e, e->tmp_d, d, nullptr, 0, R, d, e->G(ix.be1), st);
      // multi_head_attention_backward (attention.cpp:528-565)
      gemm_rm(e->blas, true, false, d, d, R, a.o3, 3 * d, e->tmp_d2, d, e->G(ix.wo), d);
      gemm_rm(e->blas, false, true, R, d, d, e->tmp_d2, d, e->P(ix.wo), d, e->do3, 3 * d);
      ENC_OP(cotten_bwd_mdev(&od, a.qkv, a.qkv + d, a.qkv + 2 * d, e->valid, e->m + l, e->do3, a.S,
                             e->dqkv, e->dqkv + d, e->dqkv + 2 * d, nullptr, e->gm + l, st));
      float* dwc = e->dwcat + l * 3 * d * d;
      gemm_rm(e->blas, true, false, d, 3 * d, R, a.x, d, e->dqkv, 3 * d, dwc, 3 * d);
      pack_qkv_kernel<<<grid_for(3 * d * d), 256, 0, st>>>(dwc, e->G(ix.wq), (int)d, (int)e->dh,
                                                           (int)(3 * e->H), 1);
      // dx = dQKV Wcat^T + ds1 (residual, encoder.cpp:254-255): ds1 is in dh, beta = 1
      gemm_rm(e->blas, false, true, R, d, 3 * d, e->dqkv, 3 * d, e->wcat + l * 3 * d * d, 3 * d,
              e->dgrad, d, 1.f);
      ENC_CUDA(cudaGetLastError());
    }
    // embedding (encoder.cpp:363-373)
    ENC_CUDA(cudaMemsetAsync(e->G(e->t_item), 0, e->rows[e->t_item] * d * sizeof(float), st));
    ENC_CUDA(cudaMemsetAsync(e->G(e->t_pos), 0, e->rows[e->t_pos] * d * sizeof(float), st));
    embed_bwd_item_kernel<<<grid_for(R * d), 256, 0, st>>>(e->dgrad, mask_of(0), e->ids, R, (int)d,
                                                           e->id_count, e->G(e->t_item));
    embed_bwd_pos_kernel<<<grid_for(e->n * d), 256, 0, st>>>(e->dgrad, mask_of(0), e->B, (int)e->n,
                                                             (int)d, e->G(e->t_pos));
    ENC_CUDA(cudaGetLastError());
  });
}

int cotten_enc_clip_adam(cotten_encoder* e, double max_norm, double lr, double weight_decay,
                         double* norm_out, void* stream) {
  return enc_guarded([&] {
    if (!e) enc_usage("adam_step: null encoder");
    if (!(max_norm > 0.0)) enc_usage("clip_gradients: max_norm must be > 0");
    cudaStream_t st = (cudaStream_t)stream;
    sumsq_stage1<<<kNormBlocks, 256, 0, st>>>(e->grads, e->count, e->norm_part);
    clip_scale_kernel<<<1, 32, 0, st>>>(e->norm_part, kNormBlocks, e->gm, (int)e->L, max_norm,
                                         e->clip_scale, norm_out);
    e->adam_step += 1;
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;  // AdamState (training.hpp:40-46)
    const double bc1 = 1.0 - std::pow(b1, (double)e->adam_step);
    const double bc2 = 1.0 - std::pow(b2, (double)e->adam_step);
    adam_kernel<<<grid_for(e->count), 256, 0, st>>>(e->params, e->grads, e->adam1, e->adam2, e->count,
                                                    e->clip_scale, (float)lr, (float)weight_decay,
                                                    (float)b1, (float)b2, (float)eps, (float)bc1,
                                                    (float)bc2);
    adam_m_kernel<<<1, 32, 0, st>>>(e->m, e->gm, e->m1m, e->m2m, (int)e->L, e->clip_scale, lr,
                                    weight_decay, b1, b2, eps, bc1, bc2);
    ENC_CUDA(cudaGetLastError());
  });
}

}  // extern "C"
