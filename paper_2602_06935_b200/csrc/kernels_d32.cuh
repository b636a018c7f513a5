// Fast fp32 cosine-attention kernels for head_dim 32 (the ML-1M / ML-20M /
// Beauty shapes: model d = 64, 2 heads) and seq_len <= 256.
//
// One CTA per (sequence, head) unit, NW = ceil(N/32) warps.  At entry one
// thread issues TMA tensor loads (cp.async.bulk.tensor, 128-byte swizzle) of
// the unit's whole N x 32 tiles into shared memory: the forward waits for K,V
// while Q is still in flight; the backward waits for Q,dO while K,V land.
// Nothing but the outputs (and the d x d state S, 4 KB) goes back to HBM: no
// Q~, K~ or N x N buffer ever exists.
//
// Warp w owns rows [32w, 32w+32).  Per row block it
//   * normalises its rows in place (8 lanes per row, shuffle-reduced norms),
//   * accumulates a 32x32 row-reduction  R += x_i^T y_i   (S = K~^T V,
//     G = Q~^T dO): lane (ag, bg) holds R[8ag..8ag+8][4bg..4bg+4] as 16
//     float2 accumulators updated with FFMA2 (packed fp32 FMA, one scalar
//     operand broadcast) — 16 FFMA2 per row for 3 LDS.128,
//   * or emits a row-output  o_i = x_i M  (O = Q S, dQ~ = dO S^T,
//     dV = K~ dA, dK~ = V dA^T): lane (rg, cg) holds rows rg+8j (j<4) x
//     columns {4cg..4cg+3, 16+4cg..16+4cg+3}, again 16 FFMA2 per contraction
//     step for 3 LDS.128; the 128-byte swizzle makes the 8 row groups hit
//     8 distinct bank groups.
// Per-warp partial reductions are summed through shared memory in a fixed
// order (deterministic).  Mask semantics follow attention.cpp exactly:
// padded K rows are selected to zero (never read), dK/dV rows of padded
// positions are written as exact zeros, Q/dQ cover every row.
#pragma once
#include <cuda.h>

#include <initializer_list>
#include <type_traits>

#include "common.cuh"

namespace cotten {
namespace d32 {

constexpr int kD = 32;
constexpr uint32_t kRowBytes = 128;
constexpr int kMaxN = 256;

__host__ __device__ constexpr uint32_t tile_bytes(int N) {
  return ((uint32_t)N * kRowBytes + 1023u) & ~1023u;  // 1024-aligned for the 128B swizzle
}

// ---- PTX wrappers ---------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Byte offset of 16-byte chunk c of row r in a 128B-swizzled tile (TMA
// CU_TENSOR_MAP_SWIZZLE_128B: chunk index XOR (row mod 8)).
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)r * kRowBytes + ((uint32_t)(c ^ (r & 7)) << 4);
}
__device__ __forceinline__ float4 lds4(const uint8_t* t, int r, int c) {
  return *reinterpret_cast<const float4*>(t + swz(r, c));
}
__device__ __forceinline__ void sts4(uint8_t* t, int r, int c, float4 v) {
  *reinterpret_cast<float4*>(t + swz(r, c)) = v;
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float s, float2 c) {
  return __ffma2_rn(a, make_float2(s, s), c);
}

// ---- building blocks (all warp-level) --------------------------------------

// Normalise rows [r0, r0+32) ∩ [0, N) of a swizzled tile in place:
// x <- valid ? x / sqrt(|x|^2 + eps) : 0   (attention.cpp:83-87, :334-342, :366-372)
// inv[r] <- valid ? 1/sqrt(|x|^2+eps) : 0; norm_out[r] <- valid ? sqrt(..) : 1 (:336,:343,:374)
__device__ __forceinline__ void normalize_rows(uint8_t* t, int r0, int N, const uint8_t* vflag,
                                               float eps, float* inv, float* norm_out, int lane) {
  const int sub = lane >> 3, c = lane & 7;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const int r = r0 + 4 * g + sub;
    const int rl = r < N ? r : N - 1;
    float4 x = lds4(t, rl, c);
    float ss = x.x * x.x;
    ss = fmaf(x.y, x.y, ss);
    ss = fmaf(x.z, x.z, ss);
    ss = fmaf(x.w, x.w, ss);
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    ss += __shfl_xor_sync(0xffffffffu, ss, 4);
    if (r < N) {
      const bool valid = vflag == nullptr || vflag[r] != 0;
      const float nrm = sqrtf(ss + eps);
      const float iv = 1.0f / nrm;
      x = valid ? make_float4(x.x * iv, x.y * iv, x.z * iv, x.w * iv)
                : make_float4(0.f, 0.f, 0.f, 0.f);
      sts4(t, r, c, x);
      if (c == 0) {
        if (inv) inv[r] = valid ? iv : 0.f;
        if (norm_out) norm_out[r] = valid ? nrm : 1.0f;
      }
    }
  }
}

// acc[y][xp] += x[8ag+2xp .. +1] * y[4bg+y] over rows [r0, min(r0+32, N)).
__device__ __forceinline__ void row_reduce(const uint8_t* X, const uint8_t* Y, int r0, int N,
                                           float2 (&acc)[4][4], int lane) {
  const int ag = lane >> 3, bg = lane & 7;
  const int r1 = min(r0 + 32, N);
#pragma unroll 2
  for (int r = r0; r < r1; ++r) {
    const float4 x0 = lds4(X, r, 2 * ag), x1 = lds4(X, r, 2 * ag + 1);
    const float4 y = lds4(Y, r, bg);
    const float2 xp[4] = {f2(x0.x, x0.y), f2(x0.z, x0.w), f2(x1.x, x1.y), f2(x1.z, x1.w)};
    const float ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int yy = 0; yy < 4; ++yy)
#pragma unroll
      for (int p = 0; p < 4; ++p) acc[yy][p] = fma2(xp[p], ys[yy], acc[yy][p]);
  }
}

// Store a warp's 32x32 partial (row-reduction layout) to part[a*32 + b].
__device__ __forceinline__ void store_partial(float* part, const float2 (&acc)[4][4], int lane) {
  const int ag = lane >> 3, bg = lane & 7;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int a = 8 * ag + 2 * p;
    *reinterpret_cast<float4*>(part + a * 32 + 4 * bg) =
        make_float4(acc[0][p].x, acc[1][p].x, acc[2][p].x, acc[3][p].x);
    *reinterpret_cast<float4*>(part + (a + 1) * 32 + 4 * bg) =
        make_float4(acc[0][p].y, acc[1][p].y, acc[2][p].y, acc[3][p].y);
  }
}

// o[j][0..3] (row r0+rg+8j, columns chunk cg then chunk cg+4) = x_row . M
// with M a plain row-major 32x32 matrix in shared memory.
__device__ __forceinline__ void row_output(const uint8_t* X, const float* M, int r0, int N,
                                           float2 (&o)[4][4], int lane) {
  const int rg = lane >> 2, cg = lane & 3;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int p = 0; p < 4; ++p) o[j][p] = f2(0.f, 0.f);
  int rows[4];
  bool ok[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = r0 + rg + 8 * j;
    ok[j] = r < N;
    rows[j] = ok[j] ? r : N - 1;
  }
#pragma unroll 2
  for (int c = 0; c < 8; ++c) {
    float4 xv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      xv[j] = lds4(X, rows[j], c);
      if (!ok[j]) xv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int aa = 0; aa < 4; ++aa) {
      const float* mrow = M + (4 * c + aa) * 32;
      const float4 m0 = *reinterpret_cast<const float4*>(mrow + 4 * cg);
      const float4 m1 = *reinterpret_cast<const float4*>(mrow + 16 + 4 * cg);
      const float2 mp[4] = {f2(m0.x, m0.y), f2(m0.z, m0.w), f2(m1.x, m1.y), f2(m1.z, m1.w)};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float xs = aa == 0 ? xv[j].x : aa == 1 ? xv[j].y : aa == 2 ? xv[j].z : xv[j].w;
#pragma unroll
        for (int p = 0; p < 4; ++p) o[j][p] = fma2(mp[p], xs, o[j][p]);
      }
    }
  }
}

// The 8 values of row r that lane (rg, cg) owns in a row-output: chunk cg, chunk cg+4.
__device__ __forceinline__ void own_cols(const uint8_t* X, int r, int cg, float (&v)[8]) {
  const float4 a = lds4(X, r, cg), b = lds4(X, r, cg + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void unpack(const float2 (&o)[4], float (&v)[8]) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    v[2 * p] = o[p].x;
    v[2 * p + 1] = o[p].y;
  }
}
__device__ __forceinline__ void store_row(float* dst, int cg, const float (&v)[8]) {
  *reinterpret_cast<float4*>(dst + 4 * cg) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(dst + 16 + 4 * cg) = make_float4(v[4], v[5], v[6], v[7]);
}
// Sum over the 4 lanes (cg = 0..3) sharing a row.
__device__ __forceinline__ float row_sum4(float x) {
  x += __shfl_xor_sync(0xffffffffu, x, 1);
  x += __shfl_xor_sync(0xffffffffu, x, 2);
  return x;
}

// ---- shared-memory plan (host and device agree) ---------------------------

struct FwdPlan {
  uint32_t tb, off_k, off_v, off_q, off_s, off_part, off_flag, off_bar, bytes;
  __host__ __device__ FwdPlan(int N, int NW) {
    tb = tile_bytes(N);
    off_k = 0;
    off_v = tb;
    off_q = 2 * tb;
    off_s = 3 * tb;                                            // S, 32x32 floats
    const uint32_t part = (uint32_t)NW * 4096u;                // per-warp partials
    off_part = part <= 2 * tb ? 0 : off_s + 4096;              // overlay K,V when they fit
    off_flag = (part <= 2 * tb ? off_s + 4096 : off_part + part);
    off_bar = (off_flag + kMaxN + 15) & ~15u;
    bytes = off_bar + 16;
  }
};

struct BwdPlan {
  uint32_t tb, off_q, off_do, off_k, off_v, off_st, off_inv, off_flag, off_bar, bytes;
  uint32_t off_part, off_da, off_dat, extra;
  __host__ __device__ BwdPlan(int N, int NW) {
    tb = tile_bytes(N);
    off_q = 0;
    off_do = tb;
    off_k = 2 * tb;
    off_v = 3 * tb;
    off_st = 4 * tb;                     // S^T, 32x32
    off_inv = off_st + 4096;             // 1/n_q then 1/n_k, N floats each
    off_flag = off_inv + 2 * kMaxN * 4;  // valid flags
    const uint32_t part = (uint32_t)NW * 4096u;
    // partials, then dA and dA^T, overlay the dead Q~/dO tiles when they fit
    const bool fits = part <= 2 * tb && 8192u <= 2 * tb;
    extra = fits ? 0 : (part > 8192u ? part : 8192u);
    off_part = fits ? 0 : (off_flag + kMaxN + 1023) & ~1023u;
    off_da = off_part;
    off_dat = off_part + 4096;
    off_bar = ((fits ? off_flag + kMaxN : off_part + extra) + 15) & ~15u;
    off_red = off_bar + 16;  // per-warp dm partials (doubles)
    bytes = off_red + 8 * 8;
  }
  uint32_t off_red;
};

// Count valid rows of the unit's sequence, stash per-row flags (attention.cpp:26-33).
__device__ __forceinline__ int load_flags(const OpParams& p, int64_t b, int N, uint8_t* flag) {
  const uint8_t* vrow = p.valid ? p.valid + b * p.msb : nullptr;
  int cnt = 0;
  for (int base = 0; base < N; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int f = 0;
    if (i < N) {
      f = vrow == nullptr || vrow[i] != 0;
      flag[i] = (uint8_t)f;
    }
    cnt += __syncthreads_count(f);
  }
  return cnt;
}

// ---- forward ---------------------------------------------------------------

template <int NW>
__global__ void __launch_bounds__(NW * 32) cos_fwd_d32_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const OpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = (int)p.N;
  const FwdPlan plan(N, NW);
  uint8_t* Kt = smem + plan.off_k;
  uint8_t* Vt = smem + plan.off_v;
  uint8_t* Qt = smem + plan.off_q;
  float* Ss = reinterpret_cast<float*>(smem + plan.off_s);
  float* part = reinterpret_cast<float*>(smem + plan.off_part);
  uint8_t* flag = smem + plan.off_flag;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + plan.off_bar);

  const int unit = blockIdx.x;
  const int b = unit / (int)p.H, h = unit - b * (int)p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bytes = (uint32_t)N * kRowBytes;

  if (threadIdx.x == 0) {
    prefetch_map(&tk);
    prefetch_map(&tv);
    prefetch_map(&tq);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
    mbar_expect_tx(&bar[0], 2 * bytes);
    tma_load_4d(Kt, &tk, 0, 0, h, b, &bar[0]);
    tma_load_4d(Vt, &tv, 0, 0, h, b, &bar[0]);
    mbar_expect_tx(&bar[1], bytes);
    tma_load_4d(Qt, &tq, 0, 0, h, b, &bar[1]);
  }
  const int true_n = load_flags(p, b, N, flag);  // contains __syncthreads (barrier init visible)
  const int64_t base = (int64_t)b * p.sb + (int64_t)h * p.sh;
  float* O = static_cast<float*>(p.out);
  float* norms = p.saved_norms ? static_cast<float*>(p.saved_norms) + (int64_t)unit * 2 * N
                               : nullptr;
  if (true_n == 0) {  // UsageError in the reference (attention.cpp:44)
    mbar_wait(&bar[0], 0);
    mbar_wait(&bar[1], 0);
    if (threadIdx.x == 0 && p.status) atomicOr(p.status, 1);
    if (O)
      for (int i = threadIdx.x; i < N * kD; i += blockDim.x)
        O[base + (int64_t)(i / kD) * p.sn + (i % kD)] = __int_as_float(0x7fc00000);
    return;
  }
  const float scale = (float)exp(-p.m * log((double)true_n));  // :303-304, fp64
  const float eps = (float)p.eps;
  const int r0 = warp * 32;

  // Pass 1 (:328-361): S = K~^T V.
  mbar_wait(&bar[0], 0);
  float2 acc[4][4];
#pragma unroll
  for (int y = 0; y < 4; ++y)
#pragma unroll
    for (int x = 0; x < 4; ++x) acc[y][x] = f2(0.f, 0.f);
  if (r0 < N) {
    normalize_rows(Kt, r0, N, flag, eps, nullptr, norms ? norms + N : nullptr, lane);
    __syncwarp();
    row_reduce(Kt, Vt, r0, N, acc, lane);
  }
  __syncthreads();  // all warps done reading K~, V before partials overlay them
  store_partial(part + warp * 1024, acc, lane);
  __syncthreads();
  float* gS = p.saved_S ? static_cast<float*>(p.saved_S) + (int64_t)unit * 1024 : nullptr;
  for (int e4 = threadIdx.x; e4 < 256; e4 += NW * 32) {
    float4 s = reinterpret_cast<const float4*>(part)[e4];
#pragma unroll
    for (int w = 1; w < NW; ++w) {  // fixed order: deterministic
      const float4 t = reinterpret_cast<const float4*>(part + w * 1024)[e4];
      s.x += t.x;
      s.y += t.y;
      s.z += t.z;
      s.w += t.w;
    }
    reinterpret_cast<float4*>(Ss)[e4] = s;
    if (gS) reinterpret_cast<float4*>(gS)[e4] = s;
  }
  __syncthreads();
  if (O == nullptr && norms == nullptr) return;

  // Pass 2 (:363-388): O = s * Q~ S for every row (padded rows included).
  mbar_wait(&bar[1], 0);
  if (r0 < N) {
    float2 o[4][4];
    row_output(Qt, Ss, r0, N, o, lane);
    const int rg = lane >> 2, cg = lane & 3;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + rg + 8 * j;
      const int rl = r < N ? r : N - 1;
      float qv[8];
      own_cols(Qt, rl, cg, qv);
      float ss = 0.f;
#pragma unroll
      for (int x = 0; x < 8; ++x) ss = fmaf(qv[x], qv[x], ss);
      ss = row_sum4(ss);
      const float nrm = sqrtf(ss + eps);
      const float w = scale * (1.0f / nrm);
      if (r < N) {
        float v[8];
        unpack(o[j], v);
#pragma unroll
        for (int x = 0; x < 8; ++x) v[x] *= w;
        if (O) store_row(O + base + (int64_t)r * p.sn, cg, v);
        if (norms && cg == 0) norms[r] = nrm;
      }
    }
  }
}

// ---- backward ----------------------------------------------------------------

template <int NW>
__global__ void __launch_bounds__(NW * 32) cos_bwd_d32_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
    const OpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = (int)p.N;
  const BwdPlan plan(N, NW);
  uint8_t* Qt = smem + plan.off_q;
  uint8_t* Gt = smem + plan.off_do;  // dO
  uint8_t* Kt = smem + plan.off_k;
  uint8_t* Vt = smem + plan.off_v;
  float* St = reinterpret_cast<float*>(smem + plan.off_st);
  float* inv_q = reinterpret_cast<float*>(smem + plan.off_inv);
  float* inv_k = inv_q + kMaxN;
  uint8_t* flag = smem + plan.off_flag;
  float* part = reinterpret_cast<float*>(smem + plan.off_part);
  float* dA = reinterpret_cast<float*>(smem + plan.off_da);
  float* dAt = reinterpret_cast<float*>(smem + plan.off_dat);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + plan.off_bar);
  double* red = reinterpret_cast<double*>(smem + plan.off_red);

  const int unit = blockIdx.x;
  const int b = unit / (int)p.H, h = unit - b * (int)p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bytes = (uint32_t)N * kRowBytes;

  if (threadIdx.x == 0) {
    prefetch_map(&tq);
    prefetch_map(&tdo);
    prefetch_map(&tk);
    prefetch_map(&tv);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
    mbar_expect_tx(&bar[0], 2 * bytes);
    tma_load_4d(Qt, &tq, 0, 0, h, b, &bar[0]);
    tma_load_4d(Gt, &tdo, 0, 0, h, b, &bar[0]);
    mbar_expect_tx(&bar[1], 2 * bytes);
    tma_load_4d(Kt, &tk, 0, 0, h, b, &bar[1]);
    tma_load_4d(Vt, &tv, 0, 0, h, b, &bar[1]);
  }
  // S^T from the saved state (St[c][a] = S[a][c]).
  const float* gS = static_cast<const float*>(p.saved_S) + (int64_t)unit * 1024;
  for (int e4 = threadIdx.x; e4 < 256; e4 += NW * 32) {
    const float4 s = reinterpret_cast<const float4*>(gS)[e4];
    const int a = e4 >> 3, c = (e4 & 7) * 4;
    St[(c + 0) * 32 + a] = s.x;
    St[(c + 1) * 32 + a] = s.y;
    St[(c + 2) * 32 + a] = s.z;
    St[(c + 3) * 32 + a] = s.w;
  }
  const int true_n = load_flags(p, b, N, flag);
  const int64_t base = (int64_t)b * p.sb + (int64_t)h * p.sh;
  float* dQ = static_cast<float*>(p.dq);
  float* dK = static_cast<float*>(p.dk);
  float* dV = static_cast<float*>(p.dv);
  if (true_n == 0) {
    mbar_wait(&bar[0], 0);
    mbar_wait(&bar[1], 0);
    if (threadIdx.x == 0) {
      if (p.status) atomicOr(p.status, 1);
      if (p.dm_unit) p.dm_unit[unit] = __longlong_as_double(0x7ff8000000000000ll);
    }
    const float qnan = __int_as_float(0x7fc00000);
    for (int i = threadIdx.x; i < N * kD; i += blockDim.x) {
      const int64_t o = base + (int64_t)(i / kD) * p.sn + (i % kD);
      dQ[o] = qnan;
      dK[o] = qnan;
      dV[o] = qnan;
    }
    return;
  }
  const double log_n = log((double)true_n);  // :402-403
  const float scale = (float)exp(-p.m * log_n);
  const float eps = (float)p.eps;
  const int r0 = warp * 32;
  const int rg = lane >> 2, cg = lane & 3;

  // Phase A: dQ (:410-411, :421-428) and G = Q~^T dO (:405), every row.
  mbar_wait(&bar[0], 0);
  float2 acc[4][4];
#pragma unroll
  for (int y = 0; y < 4; ++y)
#pragma unroll
    for (int x = 0; x < 4; ++x) acc[y][x] = f2(0.f, 0.f);
  if (r0 < N) {
    normalize_rows(Qt, r0, N, nullptr, eps, inv_q, nullptr, lane);
    __syncwarp();
    {
      float2 o[4][4];
      row_output(Gt, St, r0, N, o, lane);  // g = dO S^T (unscaled)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + rg + 8 * j;
        const int rl = r < N ? r : N - 1;
        float g[8], qh[8];
        unpack(o[j], g);
        own_cols(Qt, rl, cg, qh);
        float pr = 0.f;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          g[x] *= scale;
          pr = fmaf(g[x], qh[x], pr);
        }
        pr = row_sum4(pr);
        if (r < N) {
          const float iv = inv_q[r];
#pragma unroll
          for (int x = 0; x < 8; ++x) g[x] = (g[x] - pr * qh[x]) * iv;
          store_row(dQ + base + (int64_t)r * p.sn, cg, g);
        }
      }
    }
    row_reduce(Qt, Gt, r0, N, acc, lane);
  }
  __syncthreads();  // Q~ and dO are dead: partials overlay them
  store_partial(part + warp * 1024, acc, lane);
  __syncthreads();
  constexpr int PER = (256 + NW * 32 - 1) / (NW * 32);
  float4 gsum[PER];
  double dot = 0.0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e4 = threadIdx.x + k * NW * 32;
    if (e4 < 256) {
      float4 s = reinterpret_cast<const float4*>(part)[e4];
#pragma unroll
      for (int w = 1; w < NW; ++w) {
        const float4 t = reinterpret_cast<const float4*>(part + w * 1024)[e4];
        s.x += t.x;
        s.y += t.y;
        s.z += t.z;
        s.w += t.w;
      }
      gsum[k] = s;
      const int a = e4 >> 3, c = (e4 & 7) * 4;  // <G, S> (:408)
      float d = s.x * St[(c + 0) * 32 + a];
      d = fmaf(s.y, St[(c + 1) * 32 + a], d);
      d = fmaf(s.z, St[(c + 2) * 32 + a], d);
      d = fmaf(s.w, St[(c + 3) * 32 + a], d);
      dot += (double)d;
    }
  }
  __syncthreads();  // partial reads done before dA overwrites them
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e4 = threadIdx.x + k * NW * 32;
    if (e4 < 256) {
      const int a = e4 >> 3, c = (e4 & 7) * 4;
      const float4 s = make_float4(gsum[k].x * scale, gsum[k].y * scale, gsum[k].z * scale,
                                   gsum[k].w * scale);  // dA = s G (:412-413)
      reinterpret_cast<float4*>(dA)[e4] = s;
      dAt[(c + 0) * 32 + a] = s.x;
      dAt[(c + 1) * 32 + a] = s.y;
      dAt[(c + 2) * 32 + a] = s.z;
      dAt[(c + 3) * 32 + a] = s.w;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if (lane == 0) red[warp] = dot;
  __syncthreads();
  if (threadIdx.x == 0 && p.dm_unit) {
    double t = 0.0;
    for (int w = 0; w < NW; ++w) t += red[w];
    p.dm_unit[unit] = -log_n * (double)scale * t;  // :408
  }

  // Phase B: dV = K~ dA (:416), dK~ = V dA^T (:415) -> dK (:430-437); padded rows 0 (:439).
  mbar_wait(&bar[1], 0);
  if (r0 < N) {
    const bool any_valid = __any_sync(0xffffffffu, r0 + lane < N && flag[r0 + lane] != 0);
    if (!any_valid) {  // whole block padded: exact zeros, nothing to compute
      const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + rg + 8 * j;
        if (r < N) {
          store_row(dK + base + (int64_t)r * p.sn, cg, z);
          store_row(dV + base + (int64_t)r * p.sn, cg, z);
        }
      }
    } else {
      normalize_rows(Kt, r0, N, flag, eps, inv_k, nullptr, lane);
      __syncwarp();
      float2 o[4][4];
      row_output(Kt, dA, r0, N, o, lane);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + rg + 8 * j;
        if (r < N) {
          float v[8];
          unpack(o[j], v);
          if (!flag[r])
#pragma unroll
            for (int x = 0; x < 8; ++x) v[x] = 0.f;
          store_row(dV + base + (int64_t)r * p.sn, cg, v);
        }
      }
      row_output(Vt, dAt, r0, N, o, lane);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + rg + 8 * j;
        const int rl = r < N ? r : N - 1;
        float g[8], kh[8];
        unpack(o[j], g);
        own_cols(Kt, rl, cg, kh);
        float pr = 0.f;
#pragma unroll
        for (int x = 0; x < 8; ++x) pr = fmaf(g[x], kh[x], pr);
        pr = row_sum4(pr);
        if (r < N) {
          const bool valid = flag[r] != 0;
          const float iv = inv_k[r];
#pragma unroll
          for (int x = 0; x < 8; ++x) g[x] = valid ? (g[x] - pr * kh[x]) * iv : 0.f;
          store_row(dK + base + (int64_t)r * p.sn, cg, g);
        }
      }
    }
  }
}

}  // namespace d32

// ---- host side ------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// 4-D map over (D, N, H, B) with a (32, N, 1, 1) box and 128-byte swizzle.
inline bool make_unit_map(CUtensorMap* map, const void* base, const OpParams& p) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)p.D, (cuuint64_t)p.N, (cuuint64_t)p.H, (cuuint64_t)p.B};
  cuuint64_t strides[3] = {(cuuint64_t)p.sn * 4, (cuuint64_t)p.sh * 4, (cuuint64_t)p.sb * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)p.N, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline bool d32_layout_ok(const OpParams& p, std::initializer_list<const void*> ptrs) {
  if (p.D != 32 || p.N < 1 || p.N > d32::kMaxN) return false;
  if ((p.sn * 4) % 16 || (p.sh * 4) % 16 || (p.sb * 4) % 16) return false;
  if (p.B > (1ll << 31) || p.H > (1ll << 31) || p.B * p.H > (1ll << 31) - 1) return false;
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<uintptr_t>(q) & 15)) return false;
  return encode_fn() != nullptr;
}

template <typename T>
inline bool fast_fwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, float>::value) {
    return false;
  } else {
    return d32_layout_ok(p, {p.q, p.k, p.v, p.out});
  }
}
template <typename T>
inline bool fast_bwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, float>::value) {
    return false;
  } else {
    return p.saved_S != nullptr && d32_layout_ok(p, {p.q, p.k, p.v, p.dout, p.dq, p.dk, p.dv});
  }
}

template <int NW>
inline cudaError_t launch_fwd_nw(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                                 const OpParams& p, cudaStream_t st) {
  const d32::FwdPlan plan((int)p.N, NW);
  auto kern = d32::cos_fwd_d32_kernel<NW>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.bytes);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)(p.B * p.H), NW * 32, plan.bytes, st>>>(q, k, v, p);
  return cudaGetLastError();
}
template <int NW>
inline cudaError_t launch_bwd_nw(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                                 const CUtensorMap& g, const OpParams& p, cudaStream_t st) {
  const d32::BwdPlan plan((int)p.N, NW);
  auto kern = d32::cos_bwd_d32_kernel<NW>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.bytes);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)(p.B * p.H), NW * 32, plan.bytes, st>>>(q, k, v, g, p);
  return cudaGetLastError();
}

// Returns the number of kernel launches (1), or throws via the caller's check
// of cudaGetLastError.
template <typename T>
inline int launch_fast_fwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv;
  if (!make_unit_map(&mq, p.q, p) || !make_unit_map(&mk, p.k, p) || !make_unit_map(&mv, p.v, p))
    return -1;
  const int nw = (int)((p.N + 31) / 32);
  cudaError_t e;
  switch (nw) {
    case 1: e = launch_fwd_nw<1>(mq, mk, mv, p, st); break;
    case 2: e = launch_fwd_nw<2>(mq, mk, mv, p, st); break;
    case 3: e = launch_fwd_nw<3>(mq, mk, mv, p, st); break;
    case 4: e = launch_fwd_nw<4>(mq, mk, mv, p, st); break;
    case 5: e = launch_fwd_nw<5>(mq, mk, mv, p, st); break;
    case 6: e = launch_fwd_nw<6>(mq, mk, mv, p, st); break;
    case 7: e = launch_fwd_nw<7>(mq, mk, mv, p, st); break;
    default: e = launch_fwd_nw<8>(mq, mk, mv, p, st); break;
  }
  return e == cudaSuccess ? 1 : -1;
}
template <typename T>
inline int launch_fast_bwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mg;
  if (!make_unit_map(&mq, p.q, p) || !make_unit_map(&mk, p.k, p) ||
      !make_unit_map(&mv, p.v, p) || !make_unit_map(&mg, p.dout, p))
    return -1;
  const int nw = (int)((p.N + 31) / 32);
  cudaError_t e;
  switch (nw) {
    case 1: e = launch_bwd_nw<1>(mq, mk, mv, mg, p, st); break;
    case 2: e = launch_bwd_nw<2>(mq, mk, mv, mg, p, st); break;
    case 3: e = launch_bwd_nw<3>(mq, mk, mv, mg, p, st); break;
    case 4: e = launch_bwd_nw<4>(mq, mk, mv, mg, p, st); break;
    case 5: e = launch_bwd_nw<5>(mq, mk, mv, mg, p, st); break;
    case 6: e = launch_bwd_nw<6>(mq, mk, mv, mg, p, st); break;
    case 7: e = launch_bwd_nw<7>(mq, mk, mv, mg, p, st); break;
    default: e = launch_bwd_nw<8>(mq, mk, mv, mg, p, st); break;
  }
  return e == cudaSuccess ? 1 : -1;
}

}  // namespace cotten
