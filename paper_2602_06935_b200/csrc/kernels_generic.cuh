// Generic-D cosine-attention kernels: any head_dim that fits shared memory,
// any seq_len, f32 / bf16 (fp32 accumulate) and f64.  One CTA per
// (sequence, head) unit; rows stream through shared memory in tiles of TR
// rows, the d x d state lives in shared memory, and each thread owns a fixed
// set of its entries (so no atomics and a fixed summation order).
//
// This path serves the reference's arbitrary-shape tests (d_h = 1..16,
// acceptance.cpp:63) and the f64 instantiation used by the C++ adapter; the
// benchmarked shapes go through kernels_d32.cuh.
#pragma once
#include "common.cuh"

namespace cotten {

constexpr int kGenThreads = 256;

template <typename A>
__host__ __device__ inline int gen_tile_rows(int64_t D) {
  return D <= 64 ? 32 : 16;
}

template <typename A>
__host__ inline size_t gen_fwd_smem(int64_t D) {
  const int TR = gen_tile_rows<A>(D);
  return sizeof(A) * (D * D + 2 * TR * D + TR);
}
// GG: the d x d gradient state G lives in a global workspace instead of
// shared memory (large head_dim in f64, where S and G do not both fit).
template <typename A>
__host__ inline size_t gen_bwd_smem(int64_t D, bool GG = false) {
  const int TR = gen_tile_rows<A>(D);
  return sizeof(A) * ((GG ? 1 : 2) * D * D + 4 * TR * D + 2 * TR + kGenThreads / 32);
}

template <typename T, typename A>
__device__ __forceinline__ void gen_load_tile(A* dst, const T* src, int64_t base, int64_t t0,
                                              int rows, const OpParams& p) {
  const int D = (int)p.D;
  for (int idx = threadIdx.x; idx < rows * D; idx += blockDim.x) {
    const int r = idx / D, j = idx - r * D;
    dst[idx] = ld_acc(src + base + (t0 + r) * p.sn + j);
  }
}

// Row norms of a tile: rinv[r] = 1/sqrt(|x_r|^2 + eps) (attention.cpp:83-87),
// or 0 for a padded row when use_mask; optionally stores sqrt(|x_r|^2+eps)
// (1.0 for padded rows, attention.cpp:336) to norm_out[t0 + r].
template <typename A>
__device__ __forceinline__ void gen_row_norms(const A* tile, A* rinv, int rows, int D,
                                              const uint8_t* vrow, int64_t t0, bool use_mask,
                                              A eps, A* norm_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int r = warp; r < rows; r += nw) {
    A ss = 0;
    for (int j = lane; j < D; j += 32) ss += tile[r * D + j] * tile[r * D + j];
    ss = warp_sum(ss);
    if (lane == 0) {
      const bool valid = !use_mask || vrow == nullptr || vrow[t0 + r] != 0;
      const A nrm = sqrt(ss + eps);
      rinv[r] = valid ? A(1) / nrm : A(0);
      if (norm_out) norm_out[t0 + r] = valid ? nrm : A(1);
    }
  }
}

template <typename T, typename A>
__device__ void gen_fill_nan(const OpParams& p, T* dst, int64_t base) {
  const int D = (int)p.D;
  for (int64_t idx = threadIdx.x; idx < p.N * D; idx += blockDim.x) {
    const int64_t r = idx / D, j = idx - r * D;
    st_from(dst + base + r * p.sn + j, (A)NAN);
  }
}

// Forward (attention.cpp:297-395).  out == nullptr: only the saved state.
template <typename T, typename A>
__global__ void __launch_bounds__(kGenThreads) cos_fwd_generic(const OpParams p) {
  const KernelStamp stamp_(p);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_cnt;
  const int D = (int)p.D;
  const int TR = gen_tile_rows<A>(D);
  A* S = reinterpret_cast<A*>(smem_raw);
  A* kt = S + D * D;
  A* vt = kt + TR * D;
  A* rinv = vt + TR * D;

  const int64_t unit = blockIdx.x;
  const int64_t b = unit / p.H, h = unit - b * p.H;
  const int64_t base = b * p.sb + h * p.sh;
  const T* Q = static_cast<const T*>(p.q);
  const T* K = static_cast<const T*>(p.k);
  const T* V = static_cast<const T*>(p.v);
  const uint8_t* vrow = p.valid ? p.valid + b * p.msb : nullptr;
  A* norms = p.saved_norms ? static_cast<A*>(p.saved_norms) + unit * 2 * p.N : nullptr;

  const int64_t true_n = block_true_count(p, b, &s_cnt);
  if (true_n == 0) {  // the reference's UsageError (attention.cpp:44)
    if (threadIdx.x == 0 && p.status) atomicOr(p.status, 1);
    if (p.out) gen_fill_nan<T, A>(p, static_cast<T*>(p.out), base);
    return;
  }
  const A scale = (A)exp(-op_m(p) * log((double)true_n));  // :303-304, in fp64
  const A eps = (A)p.eps;
  const int nthr = blockDim.x;
  for (int e = threadIdx.x; e < D * D; e += nthr) S[e] = 0;
  __syncthreads();

  // Pass 1 (:328-361): S += K~^T V over row tiles.
  for (int64_t t0 = 0; t0 < p.N; t0 += TR) {
    const int rows = (int)min64(TR, p.N - t0);
    gen_load_tile<T, A>(kt, K, base, t0, rows, p);
    gen_load_tile<T, A>(vt, V, base, t0, rows, p);
    __syncthreads();
    gen_row_norms<A>(kt, rinv, rows, D, vrow, t0, true, eps, norms ? norms + p.N : nullptr);
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * D; idx += nthr) {
      const int r = idx / D;
      const bool valid = vrow == nullptr || vrow[t0 + r] != 0;
      kt[idx] = valid ? kt[idx] * rinv[r] : A(0);  // select: padded K never read
    }
    __syncthreads();
    for (int e = threadIdx.x; e < D * D; e += nthr) {
      const int a = e / D, c = e - a * D;
      A acc = S[e];
      for (int r = 0; r < rows; ++r) acc += kt[r * D + a] * vt[r * D + c];
      S[e] = acc;
    }
    __syncthreads();
  }
  if (p.saved_S) {
    A* dstS = static_cast<A*>(p.saved_S) + unit * (int64_t)D * D;
    for (int e = threadIdx.x; e < D * D; e += nthr) dstS[e] = S[e];
  }
  if (p.out == nullptr && norms == nullptr) return;

  // Pass 2 (:363-388): O = s * Q~ S for every row, padded included.
  T* O = static_cast<T*>(p.out);
  for (int64_t t0 = 0; t0 < p.N; t0 += TR) {
    const int rows = (int)min64(TR, p.N - t0);
    gen_load_tile<T, A>(kt, Q, base, t0, rows, p);
    __syncthreads();
    gen_row_norms<A>(kt, rinv, rows, D, nullptr, t0, false, eps, norms);
    __syncthreads();
    if (O) {
      for (int idx = threadIdx.x; idx < rows * D; idx += nthr) {
        const int r = idx / D, c = idx - r * D;
        A acc = 0;
        for (int a = 0; a < D; ++a) acc += (scale * (kt[r * D + a] * rinv[r])) * S[a * D + c];
        st_from(O + base + (t0 + r) * p.sn + c, acc);
      }
    }
    __syncthreads();
  }
}

// Backward (attention.cpp:397-441) given the saved S.
template <typename T, typename A, bool GG>
__global__ void __launch_bounds__(kGenThreads) cos_bwd_generic(const OpParams p) {
  const KernelStamp stamp_(p);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_cnt;
  const int D = (int)p.D;
  const int TR = gen_tile_rows<A>(D);
  A* S = reinterpret_cast<A*>(smem_raw);
  A* G = GG ? static_cast<A*>(p.workspace) + (int64_t)blockIdx.x * D * D : S + D * D;
  A* t1 = (GG ? S : G) + D * D;  // Q~ / K~ tile
  A* t2 = t1 + TR * D;  // dO / V tile
  A* t3 = t2 + TR * D;  // dQ~ / dK~ tile
  A* t4 = t3 + TR * D;  // dV tile
  A* rinv = t4 + TR * D;
  A* proj = rinv + TR;
  A* red = proj + TR;

  const int64_t unit = blockIdx.x;
  const int64_t b = unit / p.H, h = unit - b * p.H;
  const int64_t base = b * p.sb + h * p.sh;
  const T* Q = static_cast<const T*>(p.q);
  const T* K = static_cast<const T*>(p.k);
  const T* V = static_cast<const T*>(p.v);
  const T* dO = static_cast<const T*>(p.dout);
  T* dQ = static_cast<T*>(p.dq);
  T* dK = static_cast<T*>(p.dk);
  T* dV = static_cast<T*>(p.dv);
  const uint8_t* vrow = p.valid ? p.valid + b * p.msb : nullptr;
  const int nthr = blockDim.x;

  const int64_t true_n = block_true_count(p, b, &s_cnt);
  if (true_n == 0) {
    if (threadIdx.x == 0 && p.status) atomicOr(p.status, 1);
    gen_fill_nan<T, A>(p, dQ, base);
    gen_fill_nan<T, A>(p, dK, base);
    gen_fill_nan<T, A>(p, dV, base);
    if (threadIdx.x == 0 && p.dm_unit) p.dm_unit[unit] = NAN;
    return;
  }
  const double log_n = log((double)true_n);  // :402-403
  const A scale = (A)exp(-op_m(p) * log_n);
  const A eps = (A)p.eps;

  const A* srcS = static_cast<const A*>(p.saved_S) + unit * (int64_t)D * D;
  for (int e = threadIdx.x; e < D * D; e += nthr) {
    S[e] = srcS[e];
    G[e] = 0;
  }
  __syncthreads();

  // Phase A: G = Q~^T dO (:405) and dQ (:410-411, :421-428), all rows.
  for (int64_t t0 = 0; t0 < p.N; t0 += TR) {
    const int rows = (int)min64(TR, p.N - t0);
    gen_load_tile<T, A>(t1, Q, base, t0, rows, p);
    gen_load_tile<T, A>(t2, dO, base, t0, rows, p);
    __syncthreads();
    gen_row_norms<A>(t1, rinv, rows, D, nullptr, t0, false, eps, nullptr);
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * D; idx += nthr) t1[idx] *= rinv[idx / D];
    __syncthreads();
    for (int e = threadIdx.x; e < D * D; e += nthr) {
      const int a = e / D, c = e - a * D;
      A acc = G[e];
      for (int r = 0; r < rows; ++r) acc += t1[r * D + a] * t2[r * D + c];
      G[e] = acc;
    }
    for (int idx = threadIdx.x; idx < rows * D; idx += nthr) {
      const int r = idx / D, a = idx - r * D;
      A acc = 0;
      for (int c = 0; c < D; ++c) acc += t2[r * D + c] * S[a * D + c];
      t3[idx] = scale * acc;
    }
    __syncthreads();
    {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int r = warp; r < rows; r += nthr >> 5) {
        A pr = 0;
        for (int j = lane; j < D; j += 32) pr += t3[r * D + j] * t1[r * D + j];
        pr = warp_sum(pr);
        if (lane == 0) proj[r] = pr;
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * D; idx += nthr) {
      const int r = idx / D, j = idx - r * D;
      st_from(dQ + base + (t0 + r) * p.sn + j, (t3[idx] - proj[r] * t1[idx]) * rinv[r]);
    }
    __syncthreads();
  }

  // dm = -ln(n) * s * <G, S> (:408), fixed-order block reduction; dA = s*G.
  {
    A part = 0;
    for (int e = threadIdx.x; e < D * D; e += nthr) part += G[e] * S[e];
    part = warp_sum(part);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      A dot = 0;
      for (int w = 0; w < (nthr >> 5); ++w) dot += red[w];
      if (p.dm_unit) p.dm_unit[unit] = -log_n * (double)scale * (double)dot;
    }
    for (int e = threadIdx.x; e < D * D; e += nthr) G[e] *= scale;  // dA (:412-413)
    __syncthreads();
  }

  // Phase B: dK~ = V dA^T (:415), dV = K~ dA (:416), masked rows exactly 0.
  for (int64_t t0 = 0; t0 < p.N; t0 += TR) {
    const int rows = (int)min64(TR, p.N - t0);
    gen_load_tile<T, A>(t1, K, base, t0, rows, p);
    gen_load_tile<T, A>(t2, V, base, t0, rows, p);
    __syncthreads();
    gen_row_norms<A>(t1, rinv, rows, D, vrow, t0, true, eps, nullptr);
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * D; idx += nthr) {
      const int r = idx / D;
      const bool valid = vrow == nullptr || vrow[t0 + r] != 0;
      t1[idx] = valid ? t1[idx] * rinv[r] : A(0);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * D; idx += nthr) {
      const int r = idx / D, a = idx - r * D;
      A acc_k = 0, acc_v = 0;
      for (int c = 0; c < D; ++c) {
        acc_k += t2[r * D + c] * G[a * D + c];  // dK~[r][a] = sum_c V[r][c] dA[a][c]
        acc_v += t1[r * D + c] * G[c * D + a];  // dV[r][a]  = sum_c K~[r][c] dA[c][a]
      }
      t3[idx] = acc_k;
      t4[idx] = acc_v;
    }
    __syncthreads();
    {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int r = warp; r < rows; r += nthr >> 5) {
        A pr = 0;
        for (int j = lane; j < D; j += 32) pr += t3[r * D + j] * t1[r * D + j];
        pr = warp_sum(pr);
        if (lane == 0) proj[r] = pr;
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * D; idx += nthr) {
      const int r = idx / D, j = idx - r * D;
      const bool valid = vrow == nullptr || vrow[t0 + r] != 0;
      const int64_t o = base + (t0 + r) * p.sn + j;
      st_from(dK + o, valid ? (t3[idx] - proj[r] * t1[idx]) * rinv[r] : A(0));  // :430-437
      st_from(dV + o, valid ? t4[idx] : A(0));                                   // :439
    }
    __syncthreads();
  }
}

// Deterministic fixed-order sum of the per-unit dm values (the reference sums
// over heads, attention.cpp:555, then sequences, encoder.cpp:375).
__global__ void __launch_bounds__(256) dm_reduce_kernel(const double* dm_unit, int64_t units,
                                                        double* dm_total) {
  __shared__ double red[8];
  double part = 0.0;
  const int64_t per = (units + blockDim.x - 1) / blockDim.x;
  const int64_t lo = threadIdx.x * per, hi = min64(units, lo + per);
  for (int64_t u = lo; u < hi; ++u) part += dm_unit[u];  // contiguous chunks, in order
  part = warp_sum(part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *dm_total = t;
  }
}

}  // namespace cotten
