// Register-tiled FP32-pipe kernels for head_dim 64 and 128, f32 or bf16 in
// HBM, fp32 arithmetic: the d_h = 64 / 128 rows of BASELINE config #5 (the
// long-sequence sweep).  One CTA of 256 threads per (sequence, head) unit;
// many units per SM (48-160 KB of shared memory per CTA).
//
//   forward   pass 1: S = K~^T V            (attention.cpp:328-361)
//             pass 2: O = s Q~ S             (:363-388)
//   backward  phase A: G = Q~^T dO, dQ~ = s dO S^T, dQ Jacobian   (:405, :410-411, :421-428)
//             dm = -ln(n) s <G, S>, dA = s G                     (:408, :412-413)
//             phase B: dK~ = V dA^T, dV = K~ dA, dK Jacobian, masks (:415-416, :430-439)
//
// Rows stream through shared memory in tiles of TR rows (64 for d_h = 64,
// 32 for 128), double-buffered: tile i+1 is fetched into registers with
// 16-byte (f32) / 8-byte (bf16) coalesced loads while tile i is computed;
// the row norm is a shuffle reduction over the 16 / 32 threads that load
// the row, and normalisation / masking happen on the way into shared memory.
//   * reductions (S, G): thread (ab, cb) owns a (d/16) x (d/16) block of the
//     d x d state in registers; per row it reads d/16 + d/16 floats (two or
//     four 16-byte shared loads, broadcast / contiguous) for (d/16)^2 FMAs,
//     issued as FFMA2 (two fp32 FMAs per lane per instruction: a 3-register
//     FFMA issues every other cycle per SMSP, so only FFMA2 reaches the pipe's
//     rate).
//     The register block is added into a shared-memory running sum every 512
//     rows (the same accuracy bound as the tensor-core path's flush).
//   * row outputs (O, dQ~, dK~, dV): thread (rb, cb) owns rows rb + 16 k and
//     columns 4 cb + 64 g (+0..3) of the tile: 16 outputs, each 4-step of the
//     contraction is RR + 4 (RC / 4) 16-byte shared loads for 16 x 4 FMAs.
//   * the per-row dot of the Jacobians is a shuffle over the 16 threads that
//     own the row.
// The d_h = 32 shapes run on the tensor cores (kernels_tc.cuh); at d_h >= 64
// the FP32 pipe caps these kernels below the HBM roof (flop/B = d_h / 4 in
// fp32), which is what the bench reports them against.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels_generic.cuh"

namespace cotten {
namespace rt {

#ifndef COTTEN_RT128_THREADS
#define COTTEN_RT128_THREADS 256
#endif

template <int D>
struct Cfg {
  // threads per CTA: d_h 128 runs one CTA per SM (its state alone is 64-128 KB,
  // ncu: 12.5 % warps active, short-scoreboard stalls first); 512 threads
  // (COTTEN_RT128_THREADS=512: CB 32, RC 4) measured no faster — the
  // shared-memory port (L1/TEX 69-79 %) bounds it, not latency
  // (profiles/r02aa_rt512) — so 256 stays
  static constexpr int NT = D >= 128 ? COTTEN_RT128_THREADS : 256;
  // thread tid = (row index) * CB + cb: cb picks the 4-column groups
  // cb + CB g of a row (state and outputs alike)
  static constexpr int CB = (D >= 128 && NT == 512) ? 32 : (D / 4 < 16 ? D / 4 : 16);  // 8 / 16 / 32
  static constexpr int RB = NT / CB;             // distinct row indices (32 / 16 / 16)
  static constexpr int RC = D / CB;              // columns per thread (4 / 4 / 4)
  static constexpr int RA = D * D / (NT * RC);   // state rows per thread (1 / 4 / 8)
  static constexpr int RR = (D >= 128 && NT == 512) ? 2 : 16 / RC;  // output rows per thread (4 / 4 / 2)
  static constexpr int TR = RB * RR;             // tile rows (128 / 64 / 32)
  static constexpr int F4 = D / 4;               // 4-element groups per row
  static constexpr int LD = TR * F4 / NT;        // 4-element loads per thread per tile
  static constexpr int kFlushTiles = 512 / TR;  // running-sum flush period (512 rows)
  // tile row stride: +16 B so rows rb and rb + 1 (read together by a warp in
  // the row outputs) fall in different banks
  static constexpr int LDT = D + 4;
  // two tile buffers (double-buffered: tile i+1's loads are in flight while
  // tile i is computed) of two tensors each, the state(s), 1/norm per buffer
  static constexpr size_t fwd_smem = sizeof(float) * (4 * TR * LDT + D * D + 2 * TR);
  static constexpr size_t bwd_smem =
      sizeof(float) * (4 * TR * LDT + 2 * D * D + 2 * TR) + (NT / 32) * sizeof(double);
};

__device__ __forceinline__ float4 ld4(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float4 ld4(const __nv_bfloat16* p) {
  const uint2 u = __ldcs(reinterpret_cast<const uint2*>(p));
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(a, b, c, d));
}
__device__ __forceinline__ void st4(__nv_bfloat16* p, float a, float b, float c, float d) {
  const __nv_bfloat162 x = __floats2bfloat162_rn(a, b), y = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<const uint32_t*>(&x);
  u.y = *reinterpret_cast<const uint32_t*>(&y);
  __stcs(reinterpret_cast<uint2*>(p), u);
}

enum TileMode { kRaw, kQuery, kKey };

// Rows [t0, t0 + TR) of X into registers (rows >= N are zeros); thread
// tid holds 4-element groups f = tid + 256 k (row f / F4, group f % F4).
template <typename T, int D>
__device__ __forceinline__ void fetch_tile(float4 (&reg)[Cfg<D>::LD], const T* X, int64_t base,
                                           int64_t sn, int64_t N, int64_t t0) {
  using C = Cfg<D>;
#pragma unroll
  for (int k = 0; k < C::LD; ++k) {
    const int f = threadIdx.x + C::NT * k;
    const int64_t row = t0 + f / C::F4;
    reg[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < N) reg[k] = ld4(X + base + row * sn + 4 * (f % C::F4));
  }
}
// The fetched rows into sm[TR][D].  kQuery: every row < N scaled by
// 1/sqrt(|x|^2 + eps) (:366-377); kKey: valid rows scaled, padded rows exact
// zeros by select (:334-342).  rinv[r] = the factor; norm_out (optional):
// sqrt(|x|^2 + eps), 1.0 for padded keys (:336, :343).
template <int D>
__device__ __forceinline__ void put_tile(float* sm, float* rinv, const float4 (&reg)[Cfg<D>::LD],
                                         int64_t N, int64_t t0, TileMode mode, const uint8_t* vrow,
                                         float eps, float* norm_out) {
  using C = Cfg<D>;
#pragma unroll
  for (int k = 0; k < C::LD; ++k) {
    const int f = threadIdx.x + C::NT * k;
    const int r = f / C::F4, c4 = f % C::F4;
    const int64_t row = t0 + r;
    float4 v = reg[k];
    if (mode != kRaw) {
      float ss = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
#pragma unroll
      for (int o = C::F4 / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const float nrm = sqrtf(ss + eps);
      const float inv = 1.0f / nrm;
      const bool keep = row < N && (mode == kQuery || vrow == nullptr || vrow[row] != 0);
      const float m = keep ? inv : 0.f;
      v = keep ? make_float4(v.x * m, v.y * m, v.z * m, v.w * m) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (c4 == 0) {
        rinv[r] = inv;
        if (norm_out && row < N) norm_out[row] = keep ? nrm : 1.0f;
      }
    }
    *reinterpret_cast<float4*>(sm + r * C::LDT + 4 * c4) = v;
  }
}

// acc[i][j] += x[r][a_i] y[r][c_j] over the tile's rows (a_i = 64(i/4) + 4ab + i%4).
template <int D>
__device__ __forceinline__ void reduce_tile(float (&acc)[Cfg<D>::RA][Cfg<D>::RC], const float* x,
                                            const float* y, int rows, int ab, int cb) {
  using C = Cfg<D>;
#pragma unroll 2
  for (int r = 0; r < rows; ++r) {
    float xa[C::RA], yc[C::RC];
    if constexpr (C::RA == 1) {
      xa[0] = x[r * C::LDT + ab];
    } else {
#pragma unroll
      for (int g = 0; g < C::RA / 4; ++g) {
        const float4 u = *reinterpret_cast<const float4*>(x + r * C::LDT + 64 * g + 4 * ab);
        xa[4 * g] = u.x; xa[4 * g + 1] = u.y; xa[4 * g + 2] = u.z; xa[4 * g + 3] = u.w;
      }
    }
#pragma unroll
    for (int g = 0; g < C::RC / 4; ++g) {
      const float4 u = *reinterpret_cast<const float4*>(y + r * C::LDT + 4 * (cb + C::CB * g));
      yc[4 * g] = u.x; yc[4 * g + 1] = u.y; yc[4 * g + 2] = u.z; yc[4 * g + 3] = u.w;
    }
#pragma unroll
    for (int i = 0; i < C::RA; ++i)
#pragma unroll
      for (int j = 0; j < C::RC; j += 2) {  // FFMA2: the FP32 pipe's full rate
        const float2 r2 = __ffma2_rn(make_float2(xa[i], xa[i]), make_float2(yc[j], yc[j + 1]),
                                     make_float2(acc[i][j], acc[i][j + 1]));
        acc[i][j] = r2.x;
        acc[i][j + 1] = r2.y;
      }
  }
}

// run[a_i][c_j] += acc[i][j]; acc = 0 (each thread its own entries).
template <int D>
__device__ __forceinline__ void flush_state(float (&acc)[Cfg<D>::RA][Cfg<D>::RC], float* run, int ab,
                                            int cb) {
  using C = Cfg<D>;
#pragma unroll
  for (int i = 0; i < C::RA; ++i) {
    const int a = C::RA == 1 ? ab : 64 * (i / 4) + 4 * ab + (i % 4);
#pragma unroll
    for (int g = 0; g < C::RC / 4; ++g) {
      float4* q = reinterpret_cast<float4*>(run + a * D + 4 * (cb + C::CB * g));
      float4 v = *q;
      v.x += acc[i][4 * g]; v.y += acc[i][4 * g + 1]; v.z += acc[i][4 * g + 2]; v.w += acc[i][4 * g + 3];
      *q = v;
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][4 * g + e] = 0.f;
    }
  }
}

// out[k][j] = sum_x X[rb + 16k][x] M[x][c_j]  (c_j = 64(j/4) + 4cb + j%4)
template <int D>
__device__ __forceinline__ void rowout_tile(float (&out)[Cfg<D>::RR][Cfg<D>::RC], const float* X,
                                            const float* M, int rb, int cb) {
  using C = Cfg<D>;
#pragma unroll
  for (int k = 0; k < C::RR; ++k)
#pragma unroll
    for (int j = 0; j < C::RC; ++j) out[k][j] = 0.f;
#pragma unroll 2
  for (int x = 0; x < D; x += 4) {
    float4 xr[C::RR];
#pragma unroll
    for (int k = 0; k < C::RR; ++k) xr[k] = *reinterpret_cast<const float4*>(X + (rb + C::RB * k) * C::LDT + x);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float m[C::RC];
#pragma unroll
      for (int g = 0; g < C::RC / 4; ++g) {
        const float4 u = *reinterpret_cast<const float4*>(M + (x + e) * D + 4 * (cb + C::CB * g));
        m[4 * g] = u.x; m[4 * g + 1] = u.y; m[4 * g + 2] = u.z; m[4 * g + 3] = u.w;
      }
#pragma unroll
      for (int k = 0; k < C::RR; ++k) {
        const float xv = e == 0 ? xr[k].x : e == 1 ? xr[k].y : e == 2 ? xr[k].z : xr[k].w;
#pragma unroll
        for (int j = 0; j < C::RC; j += 2) {
          const float2 r2 = __ffma2_rn(make_float2(xv, xv), make_float2(m[j], m[j + 1]),
                                       make_float2(out[k][j], out[k][j + 1]));
          out[k][j] = r2.x;
          out[k][j + 1] = r2.y;
        }
      }
    }
  }
}

// Row dot sum_j out[k][j] * X[rb + 16k][c_j] over the 16 threads owning the row.
template <int D>
__device__ __forceinline__ float row_dot(const float (&o)[Cfg<D>::RC], const float* xrow, int cb) {
  using C = Cfg<D>;
  float d = 0.f;
#pragma unroll
  for (int g = 0; g < C::RC / 4; ++g) {
    const float4 u = *reinterpret_cast<const float4*>(xrow + 4 * (cb + C::CB * g));
    d = fmaf(o[4 * g], u.x, d);
    d = fmaf(o[4 * g + 1], u.y, d);
    d = fmaf(o[4 * g + 2], u.z, d);
    d = fmaf(o[4 * g + 3], u.w, d);
  }
#pragma unroll
  for (int s = C::CB / 2; s > 0; s >>= 1) d += __shfl_xor_sync(0xffffffffu, d, s);
  return d;
}

template <typename T, int D>
__device__ __forceinline__ void store_row(T* dst, const float (&o)[Cfg<D>::RC], int cb) {
  using C = Cfg<D>;
#pragma unroll
  for (int g = 0; g < C::RC / 4; ++g)
    st4(dst + 4 * (cb + C::CB * g), o[4 * g], o[4 * g + 1], o[4 * g + 2], o[4 * g + 3]);
}

template <typename T, int D>
__global__ void __launch_bounds__(Cfg<D>::NT) cos_fwd_rt(const OpParams p) {
  const KernelStamp stamp_(p);
  using C = Cfg<D>;
  extern __shared__ __align__(16) float sm[];
  constexpr int TD = C::TR * C::LDT;
  float* tiles = sm;              // [buffer][tensor][TR][D]
  float* Ssm = tiles + 4 * TD;    // running S, then the B operand of O = Q~ S
  float* rinv_all = Ssm + D * D;  // [buffer][TR]
  __shared__ int s_cnt;
  const int64_t unit = blockIdx.x, N = p.N;
  const int64_t b = unit / p.H, h = unit - b * p.H;
  const int64_t base = b * p.sb + h * p.sh;
  const uint8_t* vrow = p.valid ? p.valid + b * p.msb : nullptr;
  float* norms = p.saved_norms ? static_cast<float*>(p.saved_norms) + unit * 2 * N : nullptr;
  const int64_t true_n = block_true_count(p, b, &s_cnt);
  if (true_n == 0) {  // the reference's UsageError (attention.cpp:44)
    if (threadIdx.x == 0 && p.status) atomicOr(p.status, 1);
    if (p.out) gen_fill_nan<T, float>(p, static_cast<T*>(p.out), base);
    return;
  }
  const float scale = (float)exp(-op_m(p) * log((double)true_n));  // :303-304, in fp64
  const float eps = (float)p.eps;
  const int tid = threadIdx.x, ab = tid / C::CB, cb = tid % C::CB;
  for (int e = tid; e < D * D; e += C::NT) Ssm[e] = 0.f;

  float acc[C::RA][C::RC];
#pragma unroll
  for (int i = 0; i < C::RA; ++i)
#pragma unroll
    for (int j = 0; j < C::RC; ++j) acc[i][j] = 0.f;
  const T* K = static_cast<const T*>(p.k);
  const T* V = static_cast<const T*>(p.v);
  const T* Q = static_cast<const T*>(p.q);
  float4 ra[C::LD], rb4[C::LD];
  fetch_tile<T, D>(ra, K, base, p.sn, N, 0);
  fetch_tile<T, D>(rb4, V, base, p.sn, N, 0);
  int nt = 0;
  for (int64_t t0 = 0; t0 < N; t0 += C::TR, ++nt) {
    float* X0 = tiles + (nt & 1) * 2 * TD;
    float* X1 = X0 + TD;
    float* rinv = rinv_all + (nt & 1) * C::TR;
    put_tile<D>(X0, rinv, ra, N, t0, kKey, vrow, eps, norms ? norms + N : nullptr);
    put_tile<D>(X1, rinv, rb4, N, t0, kRaw, vrow, eps, nullptr);
    __syncthreads();  // also: every thread is done with the tile this buffer held two steps ago
    if (t0 + C::TR < N) {
      fetch_tile<T, D>(ra, K, base, p.sn, N, t0 + C::TR);
      fetch_tile<T, D>(rb4, V, base, p.sn, N, t0 + C::TR);
    }
    reduce_tile<D>(acc, X0, X1, (int)min64(C::TR, N - t0), ab, cb);
    if ((nt + 1) % C::kFlushTiles == 0 || t0 + C::TR >= N) flush_state<D>(acc, Ssm, ab, cb);
  }
  __syncthreads();
  if (p.saved_S) {
    float* dst = static_cast<float*>(p.saved_S) + unit * (int64_t)D * D;
    for (int e = tid; e < D * D / 4; e += C::NT)
      reinterpret_cast<float4*>(dst)[e] = reinterpret_cast<const float4*>(Ssm)[e];
  }
  if (p.out == nullptr && norms == nullptr) return;

  T* O = static_cast<T*>(p.out);
  const int rb = tid / C::CB;
  fetch_tile<T, D>(ra, Q, base, p.sn, N, 0);
  nt = 0;
  for (int64_t t0 = 0; t0 < N; t0 += C::TR, ++nt) {
    float* X0 = tiles + (nt & 1) * 2 * TD;
    float* rinv = rinv_all + (nt & 1) * C::TR;
    put_tile<D>(X0, rinv, ra, N, t0, kQuery, nullptr, eps, norms);
    __syncthreads();
    if (t0 + C::TR < N) fetch_tile<T, D>(ra, Q, base, p.sn, N, t0 + C::TR);
    if (O) {
      float o[C::RR][C::RC];
      rowout_tile<D>(o, X0, Ssm, rb, cb);
#pragma unroll
      for (int k = 0; k < C::RR; ++k) {
        const int64_t row = t0 + rb + C::RB * k;
#pragma unroll
        for (int j = 0; j < C::RC; ++j) o[k][j] *= scale;
        if (row < N) store_row<T, D>(O + base + row * p.sn, o[k], cb);
      }
    }
  }
}

template <typename T, int D>
__global__ void __launch_bounds__(Cfg<D>::NT) cos_bwd_rt(const OpParams p) {
  const KernelStamp stamp_(p);
  using C = Cfg<D>;
  extern __shared__ __align__(16) float sm[];
  constexpr int TD = C::TR * C::LDT;
  float* tiles = sm;                // [buffer][Q~ or K~ | dO or V][TR][D]
  float* Bt = tiles + 4 * TD;       // S^T (phase A), then dA^T (phase B)
  float* Bn = Bt + D * D;           // G running sum, then dA
  float* rinv_all = Bn + D * D;     // [buffer][TR]
  double* red = reinterpret_cast<double*>(rinv_all + 2 * C::TR);
  __shared__ int s_cnt;
  const int64_t unit = blockIdx.x, N = p.N;
  const int64_t b = unit / p.H, h = unit - b * p.H;
  const int64_t base = b * p.sb + h * p.sh;
  const uint8_t* vrow = p.valid ? p.valid + b * p.msb : nullptr;
  T* dQ = static_cast<T*>(p.dq);
  T* dK = static_cast<T*>(p.dk);
  T* dV = static_cast<T*>(p.dv);
  const int64_t true_n = block_true_count(p, b, &s_cnt);
  if (true_n == 0) {
    if (threadIdx.x == 0 && p.status) atomicOr(p.status, 1);
    gen_fill_nan<T, float>(p, dQ, base);
    gen_fill_nan<T, float>(p, dK, base);
    gen_fill_nan<T, float>(p, dV, base);
    if (threadIdx.x == 0 && p.dm_unit) p.dm_unit[unit] = NAN;
    return;
  }
  const double log_n = log((double)true_n);  // :402-403
  const float scale = (float)exp(-op_m(p) * log_n);
  const float eps = (float)p.eps;
  const int tid = threadIdx.x, ab = tid / C::CB, cb = tid % C::CB, rb = ab;

  // S^T into Bt (Bt[c][a] = S[a][c], conflict-free smem writes), G = 0
  const float* gS = static_cast<const float*>(p.saved_S) + unit * (int64_t)D * D;
  for (int e = tid; e < D * D; e += C::NT) {
    const int c = e / D, a = e - c * D;
    Bt[e] = __ldg(gS + a * D + c);
    Bn[e] = 0.f;
  }

  float acc[C::RA][C::RC];
#pragma unroll
  for (int i = 0; i < C::RA; ++i)
#pragma unroll
    for (int j = 0; j < C::RC; ++j) acc[i][j] = 0.f;
  const T* Q = static_cast<const T*>(p.q);
  const T* dO = static_cast<const T*>(p.dout);
  const T* K = static_cast<const T*>(p.k);
  const T* V = static_cast<const T*>(p.v);
  float4 ra[C::LD], rb4[C::LD];
  fetch_tile<T, D>(ra, Q, base, p.sn, N, 0);
  fetch_tile<T, D>(rb4, dO, base, p.sn, N, 0);
  int nt = 0;
  // Phase A: G = Q~^T dO over all rows; dQ (all rows)
  for (int64_t t0 = 0; t0 < N; t0 += C::TR, ++nt) {
    float* X0 = tiles + (nt & 1) * 2 * TD;
    float* X1 = X0 + TD;
    float* rinv = rinv_all + (nt & 1) * C::TR;
    put_tile<D>(X0, rinv, ra, N, t0, kQuery, nullptr, eps, nullptr);
    put_tile<D>(X1, rinv, rb4, N, t0, kRaw, nullptr, eps, nullptr);
    __syncthreads();
    if (t0 + C::TR < N) {
      fetch_tile<T, D>(ra, Q, base, p.sn, N, t0 + C::TR);
      fetch_tile<T, D>(rb4, dO, base, p.sn, N, t0 + C::TR);
    }
    reduce_tile<D>(acc, X0, X1, (int)min64(C::TR, N - t0), ab, cb);
    if ((nt + 1) % C::kFlushTiles == 0 || t0 + C::TR >= N) flush_state<D>(acc, Bn, ab, cb);
    float o[C::RR][C::RC];
    rowout_tile<D>(o, X1, Bt, rb, cb);  // dO S^T
#pragma unroll
    for (int k = 0; k < C::RR; ++k) {
      const int r = rb + C::RB * k;
#pragma unroll
      for (int j = 0; j < C::RC; ++j) o[k][j] *= scale;
      const float d = row_dot<D>(o[k], X0 + r * C::LDT, cb);
      const float iv = rinv[r];
#pragma unroll
      for (int g = 0; g < C::RC / 4; ++g) {
        const float4 q = *reinterpret_cast<const float4*>(X0 + r * C::LDT + 4 * (cb + C::CB * g));
        o[k][4 * g] = (o[k][4 * g] - d * q.x) * iv;
        o[k][4 * g + 1] = (o[k][4 * g + 1] - d * q.y) * iv;
        o[k][4 * g + 2] = (o[k][4 * g + 2] - d * q.z) * iv;
        o[k][4 * g + 3] = (o[k][4 * g + 3] - d * q.w) * iv;
      }
      if (t0 + r < N) store_row<T, D>(dQ + base + (t0 + r) * p.sn, o[k], cb);
    }
  }
  fetch_tile<T, D>(ra, K, base, p.sn, N, 0);  // phase B's first tile, in flight during dm / dA
  fetch_tile<T, D>(rb4, V, base, p.sn, N, 0);
  __syncthreads();

  // dm = -ln(n) s <G, S> (:408): fixed-order (thread, warp tree, warps in order)
  {
    double part = 0.0;
    for (int e = tid; e < D * D; e += C::NT) {
      const int a = e / D, c = e - a * D;
      part += (double)(Bn[e] * Bt[c * D + a]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((tid & 31) == 0) red[tid >> 5] = part;
    __syncthreads();
    if (tid == 0 && p.dm_unit) {
      double dot = 0.0;
      for (int w = 0; w < C::NT / 32; ++w) dot += red[w];
      p.dm_unit[unit] = -log_n * (double)scale * dot;
    }
  }
  // dA = s G (:412-413): dA^T into Bt (B of dK~ = V dA^T), dA in place in Bn (B of dV = K~ dA)
  for (int e = tid; e < D * D; e += C::NT) {
    const int c = e / D, a = e - c * D;
    Bt[e] = scale * Bn[a * D + c];
  }
  __syncthreads();
  for (int e = tid; e < D * D; e += C::NT) Bn[e] *= scale;

  // Phase B: dK (valid rows), dV (valid rows); padded rows exact zeros (:430-439)
  nt = 0;
  for (int64_t t0 = 0; t0 < N; t0 += C::TR, ++nt) {
    float* X0 = tiles + (nt & 1) * 2 * TD;
    float* X1 = X0 + TD;
    float* rinv = rinv_all + (nt & 1) * C::TR;
    put_tile<D>(X0, rinv, ra, N, t0, kKey, vrow, eps, nullptr);
    put_tile<D>(X1, rinv, rb4, N, t0, kRaw, vrow, eps, nullptr);
    __syncthreads();
    if (t0 + C::TR < N) {
      fetch_tile<T, D>(ra, K, base, p.sn, N, t0 + C::TR);
      fetch_tile<T, D>(rb4, V, base, p.sn, N, t0 + C::TR);
    }
    {
      float o[C::RR][C::RC];
      rowout_tile<D>(o, X1, Bt, rb, cb);  // dK~ = V dA^T
#pragma unroll
      for (int k = 0; k < C::RR; ++k) {
        const int r = rb + C::RB * k;
        const int64_t row = t0 + r;
        const bool f = row < N && (vrow == nullptr || vrow[row] != 0);
        const float d = row_dot<D>(o[k], X0 + r * C::LDT, cb);
        const float iv = rinv[r];
#pragma unroll
        for (int g = 0; g < C::RC / 4; ++g) {
          const float4 q = *reinterpret_cast<const float4*>(X0 + r * C::LDT + 4 * (cb + C::CB * g));
          o[k][4 * g] = f ? (o[k][4 * g] - d * q.x) * iv : 0.f;
          o[k][4 * g + 1] = f ? (o[k][4 * g + 1] - d * q.y) * iv : 0.f;
          o[k][4 * g + 2] = f ? (o[k][4 * g + 2] - d * q.z) * iv : 0.f;
          o[k][4 * g + 3] = f ? (o[k][4 * g + 3] - d * q.w) * iv : 0.f;
        }
        if (row < N) store_row<T, D>(dK + base + row * p.sn, o[k], cb);
      }
    }
    {
      float o[C::RR][C::RC];
      rowout_tile<D>(o, X0, Bn, rb, cb);  // dV = K~ dA
#pragma unroll
      for (int k = 0; k < C::RR; ++k) {
        const int64_t row = t0 + rb + C::RB * k;
        const bool f = row < N && (vrow == nullptr || vrow[row] != 0);
#pragma unroll
        for (int j = 0; j < C::RC; ++j) o[k][j] = f ? o[k][j] : 0.f;
        if (row < N) store_row<T, D>(dV + base + row * p.sn, o[k], cb);
      }
    }
  }
}

}  // namespace rt

// d_h 64 / 128, f32 or bf16, 16-byte (f32) / 8-byte (bf16) aligned rows.
template <typename T>
inline bool rt_supported(const OpParams& p, bool bwd) {
  if (sizeof(T) == 8) return false;
  // d_h 64 / 128 (f32, bf16); d_h 32 only for bf16 (f32 d_h = 32 runs on the tensor cores)
  if (p.D != 64 && p.D != 128 && !(p.D == 32 && sizeof(T) == 2)) return false;
  if (p.N < 1 || p.N > (int64_t)1 << 30) return false;
  const uintptr_t align = sizeof(T) == 4 ? 16 : 8;
  if (p.sn % 4 || p.sh % 4 || p.sb % 4) return false;
  const void* ptrs[] = {p.q, p.k, p.v, bwd ? p.dout : nullptr, bwd ? nullptr : p.out,
                        bwd ? p.dq : nullptr, bwd ? p.dk : nullptr, bwd ? p.dv : nullptr};
  for (const void* q : ptrs)
    if (q && reinterpret_cast<uintptr_t>(q) % align) return false;
  if (p.saved_S && reinterpret_cast<uintptr_t>(p.saved_S) % 16) return false;
  if (bwd && p.saved_S == nullptr) return false;
  return true;
}

template <typename T>
inline void launch_rt_fwd(const OpParams& p, cudaStream_t st) {
  auto go = [&](auto kern, size_t smem, int nt) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<(unsigned)(p.B * p.H), nt, smem, st>>>(p);
  };
  if (p.D == 32) go(rt::cos_fwd_rt<T, 32>, rt::Cfg<32>::fwd_smem, rt::Cfg<32>::NT);
  else if (p.D == 64) go(rt::cos_fwd_rt<T, 64>, rt::Cfg<64>::fwd_smem, rt::Cfg<64>::NT);
  else go(rt::cos_fwd_rt<T, 128>, rt::Cfg<128>::fwd_smem, rt::Cfg<128>::NT);
}
template <typename T>
inline void launch_rt_bwd(const OpParams& p, cudaStream_t st) {
  auto go = [&](auto kern, size_t smem, int nt) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<(unsigned)(p.B * p.H), nt, smem, st>>>(p);
  };
  if (p.D == 32) go(rt::cos_bwd_rt<T, 32>, rt::Cfg<32>::bwd_smem, rt::Cfg<32>::NT);
  else if (p.D == 64) go(rt::cos_bwd_rt<T, 64>, rt::Cfg<64>::bwd_smem, rt::Cfg<64>::NT);
  else go(rt::cos_bwd_rt<T, 128>, rt::Cfg<128>::bwd_smem, rt::Cfg<128>::NT);
}

}  // namespace cotten
