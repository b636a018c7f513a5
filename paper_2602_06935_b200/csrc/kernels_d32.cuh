// Fast fp32 cosine-attention kernels for head_dim 32 — the ML-1M / ML-20M /
// Beauty shapes (model d = 64 over 2 heads) — and seq_len <= 1024.
//
// Design: warp per unit.  Every warp of a persistent CTA owns whole
// (sequence, head) units (unit = warp_id + k * total_warps) and streams their
// 32-row tiles (cp.async.bulk.tensor, 128-byte swizzle, 4 KB per tensor per
// chunk; rows past N are zero-filled by the TMA bounds check) through its own
// NSTG-deep ring of shared-memory stages, each guarded by one mbarrier.  Lane
// 0 re-arms a stage the moment the warp has consumed it, so NSTG-1 chunks are
// always in flight.  No CTA barrier, no cross-warp reduction: the 32x32 state
// (S in the forward, G in the backward) accumulates in the warp's registers in
// row order, so results are deterministic and warps never wait on each other.
//
// Per 32-row chunk the warp
//   * normalises rows in place (8 lanes per row, shuffle-reduced norms),
//   * accumulates a row-reduction  R += x_i^T y_i   (S = K~^T V, G = Q~^T dO):
//     lane (ag, bg) holds R[8ag..8ag+8][4bg..4bg+4] as 16 float2 registers
//     updated with FFMA2 (packed fp32 FMA, scalar operand broadcast):
//     16 FFMA2 per row for 3 LDS.128,
//   * or a row-output  o_i = x_i M  (O = Q S, dQ~ = dO S^T, dV = K~ dA,
//     dK~ = V dA^T): lane (rg, cg) holds rows rg+8j (j<4) x columns
//     {4cg..4cg+3, 16+4cg..16+4cg+3}, 16 FFMA2 per contraction step for
//     3 LDS.128; the 128-byte swizzle puts the 8 row groups on 8 bank groups.
// Nothing but the outputs and the 4 KB state S per unit reaches HBM: no Q~,
// K~ or N x N buffer exists.  Mask semantics follow attention.cpp exactly:
// padded K rows are selected to zero (never read), dK / dV rows of padded
// positions are exact zeros, Q and dQ cover every row, and s = exp(-m ln n)
// comes from fp64 (a host table for n <= 256, fp64 in-kernel above).
#pragma once
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <initializer_list>
#include <type_traits>

#include "common.cuh"

namespace cotten {
namespace d32 {

constexpr int kD = 32;
constexpr uint32_t kRowBytes = 128;
constexpr uint32_t kTile = 32 * kRowBytes;  // one 32-row chunk of one tensor
constexpr int kMaxN = 1024;                 // flag words / prefetch registers
constexpr int kTabN = 256;                  // host-computed scale table range

// s[n] = exp(-m ln n) (attention.cpp:303-304, :402-403) and
// coef[n] = -ln(n) * s[n] (:408), in fp64 on the host; entry 0 is NaN (the
// reference's UsageError for a sequence without real rows).
struct ScaleTable {
  float s[kTabN + 1];
  double coef[kTabN + 1];
};

__device__ __forceinline__ float scale_of(const ScaleTable& t, int n, double m) {
  return n <= kTabN ? t.s[n] : (float)exp(-m * log((double)n));
}
__device__ __forceinline__ double coef_of(const ScaleTable& t, int n, double m) {
  return n <= kTabN ? t.coef[n] : -log((double)n) * (double)(float)exp(-m * log((double)n));
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
}
// Order this thread's (and, after __syncwarp, the warp's) generic-proxy reads
// of a stage before the async-proxy TMA write that refills it.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps until the phase
// completes instead of spinning on issue slots its neighbours need.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000)
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

__device__ __forceinline__ float4 ld4(const uint8_t* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ void st4(uint8_t* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float s, float2 c) {
  return __ffma2_rn(a, make_float2(s, s), c);
}
__device__ __forceinline__ float sel4(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// ---- chunk-level building blocks (one warp, one 128B-swizzled 32-row tile) --

// In place: x <- valid ? x / sqrt(|x|^2 + eps) : 0 for rows [0, rows) of the
// tile (attention.cpp:83-87, :334-342, :366-372); valid = bit r of vword.
// inv[r] <- valid ? 1/sqrt(..) : 0, norm_out[r] <- valid ? sqrt(..) : 1 (:336).
__device__ __forceinline__ void normalize_tile(uint8_t* X, int rows, uint32_t vword, float eps,
                                               float* inv, float* norm_out, int lane) {
  const int sub = lane >> 3, c = lane & 7;
  uint8_t* be = X + sub * kRowBytes + ((c ^ sub) << 4);        // rows with (r & 7) == sub
  uint8_t* bo = X + sub * kRowBytes + ((c ^ (sub + 4)) << 4);  // rows with (r & 7) == sub + 4
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    if (4 * g >= rows) break;  // warp-uniform
    const int r = 4 * g + sub;
    uint8_t* a = (g & 1 ? bo : be) + 512 * g;
    float4 x = ld4(a);
    float ss = x.x * x.x;
    ss = fmaf(x.y, x.y, ss);
    ss = fmaf(x.z, x.z, ss);
    ss = fmaf(x.w, x.w, ss);
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    ss += __shfl_xor_sync(0xffffffffu, ss, 4);
    if (r < rows) {
      const bool valid = (vword >> r) & 1u;
      const float nrm = sqrtf(ss + eps);
      const float iv = 1.0f / nrm;
      x = valid ? make_float4(x.x * iv, x.y * iv, x.z * iv, x.w * iv)
                : make_float4(0.f, 0.f, 0.f, 0.f);
      st4(a, x);
      if (c == 0) {
        if (inv != nullptr) inv[r] = valid ? iv : 0.f;
        if (norm_out != nullptr) norm_out[r] = valid ? nrm : 1.0f;
      }
    }
  }
}

// acc[y][p] += x[8ag+2p .. +1] * y[4bg+y] over rows [0, round8(rows)) of the
// tiles; rows >= N were zero-filled by the TMA and padded K rows zeroed.
__device__ __forceinline__ void row_reduce_tile(const uint8_t* X, const uint8_t* Y, int rows,
                                                float2 (&acc)[4][4], int lane) {
  const int ag = lane >> 3, bg = lane & 7;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (8 * t >= rows) break;  // warp-uniform
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int r = 8 * t + s;
      const float4 x0 = ld4(X + r * kRowBytes + (((2 * ag) ^ s) << 4));
      const float4 x1 = ld4(X + r * kRowBytes + (((2 * ag + 1) ^ s) << 4));
      const float4 y = ld4(Y + r * kRowBytes + ((bg ^ s) << 4));
      const float2 xp[4] = {f2(x0.x, x0.y), f2(x0.z, x0.w), f2(x1.x, x1.y), f2(x1.z, x1.w)};
#pragma unroll
      for (int yy = 0; yy < 4; ++yy)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[yy][p] = fma2(xp[p], sel4(y, yy), acc[yy][p]);
    }
  }
}

// Row-reduction registers -> row-major 32x32 matrix (optionally scaled).
__device__ __forceinline__ void store_rowmajor(float* M, const float2 (&acc)[4][4], float sc,
                                               int lane) {
  const int ag = lane >> 3, bg = lane & 7;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int a = 8 * ag + 2 * p;
    *reinterpret_cast<float4*>(M + a * 32 + 4 * bg) = make_float4(
        acc[0][p].x * sc, acc[1][p].x * sc, acc[2][p].x * sc, acc[3][p].x * sc);
    *reinterpret_cast<float4*>(M + (a + 1) * 32 + 4 * bg) = make_float4(
        acc[0][p].y * sc, acc[1][p].y * sc, acc[2][p].y * sc, acc[3][p].y * sc);
  }
}
// ... and its transpose (M^T[b][a] = R[a][b]): row b = 4bg+y, columns 8ag..8ag+7.
__device__ __forceinline__ void store_transposed(float* Mt, const float2 (&acc)[4][4], float sc,
                                                 int lane) {
  const int ag = lane >> 3, bg = lane & 7;
#pragma unroll
  for (int y = 0; y < 4; ++y) {
    float* row = Mt + (4 * bg + y) * 32 + 8 * ag;
    *reinterpret_cast<float4*>(row) = make_float4(acc[y][0].x * sc, acc[y][0].y * sc,
                                                  acc[y][1].x * sc, acc[y][1].y * sc);
    *reinterpret_cast<float4*>(row + 4) = make_float4(acc[y][2].x * sc, acc[y][2].y * sc,
                                                      acc[y][3].x * sc, acc[y][3].y * sc);
  }
}

// o[j][.] (tile row rg+8j; columns chunk cg then chunk cg+4) = x_row . M, M a
// plain row-major 32x32 fp32 matrix in shared memory (broadcast reads).
__device__ __forceinline__ void row_output_tile(const uint8_t* X, const float* M,
                                                float2 (&o)[4][4], int lane) {
  const int rg = lane >> 2, cg = lane & 3;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int p = 0; p < 4; ++p) o[j][p] = f2(0.f, 0.f);
  const uint8_t* xb = X + rg * kRowBytes;
  const float* mb = M + 4 * cg;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint8_t* xc = xb + ((c ^ rg) << 4);  // (r & 7) == rg for the four rows
    float4 xv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) xv[j] = ld4(xc + 1024 * j);
#pragma unroll
    for (int aa = 0; aa < 4; ++aa) {
      const float* mrow = mb + (4 * c + aa) * 32;
      const float4 m0 = *reinterpret_cast<const float4*>(mrow);
      const float4 m1 = *reinterpret_cast<const float4*>(mrow + 16);
      const float2 mp[4] = {f2(m0.x, m0.y), f2(m0.z, m0.w), f2(m1.x, m1.y), f2(m1.z, m1.w)};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int p = 0; p < 4; ++p) o[j][p] = fma2(mp[p], sel4(xv[j], aa), o[j][p]);
    }
  }
}

// The 8 values of tile row rg+8j that lane (rg, cg) owns in a row-output.
__device__ __forceinline__ void own_cols(const uint8_t* X, int j, int lane, float (&v)[8]) {
  const int rg = lane >> 2, cg = lane & 3;
  const uint8_t* xb = X + (rg + 8 * j) * kRowBytes;
  const float4 a = ld4(xb + ((cg ^ rg) << 4)), b = ld4(xb + (((cg + 4) ^ rg) << 4));
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
__device__ __forceinline__ float row_sum4(float x) {  // over the 4 lanes sharing a row
  x += __shfl_xor_sync(0xffffffffu, x, 1);
  x += __shfl_xor_sync(0xffffffffu, x, 2);
  return x;
}

// ---- per-warp shared-memory plan ------------------------------------------

template <bool BWD, int NSTG>
struct WarpPlan {
  static constexpr uint32_t kStage = 2 * kTile;  // two tensors per chunk
  static constexpr uint32_t off_mat = NSTG * kStage;
  static constexpr uint32_t off_mat2 = off_mat + 4096;  // bwd: dA (mat 1 holds S^T, then dA^T)
  static constexpr uint32_t off_inv = off_mat + (BWD ? 8192 : 4096);
  static constexpr uint32_t off_flag = off_inv + (BWD ? 128 : 0);
  static constexpr uint32_t off_bar = off_flag + 4 * (kMaxN / 32);
  static constexpr uint32_t bytes = (off_bar + 8 * NSTG + 1023) / 1024 * 1024;
};

// The valid-flag bytes of unit u's sequence for rows lane + 32k (k < nc),
// packed four per register: fetched one unit ahead.
__device__ __forceinline__ void fetch_flags(const OpParams& p, int u, int units, int nc, int lane,
                                            uint32_t (&fr)[kMaxN / 128]) {
#pragma unroll
  for (int i = 0; i < kMaxN / 128; ++i) fr[i] = 0;
  if (u >= units) return;
  if (p.valid == nullptr) {
#pragma unroll
    for (int i = 0; i < kMaxN / 128; ++i) fr[i] = 0x01010101u;
    return;
  }
  const uint8_t* row = p.valid + (int64_t)(u / (int)p.H) * p.msb;
  const int N = (int)p.N;
#pragma unroll
  for (int k = 0; k < kMaxN / 32; ++k) {
    if (k >= nc) break;
    const int r = lane + 32 * k;
    const uint32_t f = r < N ? (uint32_t)(__ldg(row + r) != 0) : 0u;
    fr[k >> 2] |= f << (8 * (k & 3));
  }
}
// Flag words (bit l of word k = row 32k+l valid) into shared memory; true_n.
__device__ __forceinline__ int publish_flags(const uint32_t (&fr)[kMaxN / 128], int nc,
                                             uint32_t* flagw, int lane) {
  int n = 0;
#pragma unroll
  for (int k = 0; k < kMaxN / 32; ++k) {
    if (k >= nc) break;
    const uint32_t w = __ballot_sync(0xffffffffu, (fr[k >> 2] >> (8 * (k & 3))) & 1u);
    if (lane == 0) flagw[k] = w;
    n += __popc(w);
  }
  __syncwarp();
  return n;
}

// ---- forward ---------------------------------------------------------------

template <int NSTG>
__global__ void __launch_bounds__(256) cos_fwd_d32_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const OpParams p,
    const __grid_constant__ ScaleTable tab) {
  using PL = WarpPlan<false, NSTG>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  uint8_t* ws = smem + warp * PL::bytes;
  float* Sm = reinterpret_cast<float*>(ws + PL::off_mat);
  uint32_t* flagw = reinterpret_cast<uint32_t*>(ws + PL::off_flag);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ws + PL::off_bar);

  const int N = (int)p.N, H = (int)p.H;
  const int units = (int)(p.B * p.H);
  const int nc = (N + 31) / 32;
  const int gw = blockIdx.x * wpc + warp, tw = gridDim.x * wpc;
  float* O = static_cast<float*>(p.out);
  float* norms_all = static_cast<float*>(p.saved_norms);
  float* gS_all = static_cast<float*>(p.saved_S);
  const bool want_q = O != nullptr || norms_all != nullptr;
  const int J = want_q ? 2 * nc : nc;  // jobs (chunk loads) per unit
  const int my_units = gw < units ? (units - 1 - gw) / tw + 1 : 0;
  const long total = (long)my_units * J;
  if (my_units == 0) return;

  if (lane == 0) {
    for (int s = 0; s < NSTG; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
    prefetch_map(&tk);
    prefetch_map(&tv);
    if (want_q) prefetch_map(&tq);
  }
  __syncwarp();
  // Lane 0: load job j (chunk t of this warp's k-th unit) into stage j % NSTG.
  auto issue = [&](long j) {
    if (j >= total) return;
    const int k = (int)(j / J), t = (int)(j - (long)k * J);
    const int u = gw + k * tw;
    const int b = u / H, h = u - b * H;
    const int s = (int)(j % NSTG);
    uint8_t* st = ws + s * PL::kStage;
    if (t < nc) {
      mbar_expect_tx(&bar[s], 2 * kTile);
      tma_load_4d(st, &tk, 0, 32 * t, h, b, &bar[s]);
      tma_load_4d(st + kTile, &tv, 0, 32 * t, h, b, &bar[s]);
    } else {
      mbar_expect_tx(&bar[s], kTile);
      tma_load_4d(st, &tq, 0, 32 * (t - nc), h, b, &bar[s]);
    }
  };
  if (lane == 0)
    for (int j = 0; j < NSTG; ++j) issue(j);

  const float eps = (float)p.eps;
  const int rg = lane >> 2, cg = lane & 3;
  uint32_t fnext[kMaxN / 128];
  fetch_flags(p, gw, units, nc, lane, fnext);
  long j = 0;
  for (int k = 0; k < my_units; ++k) {
    const int u = gw + k * tw;
    const int b = u / H, h = u - b * H;
    uint32_t fcur[kMaxN / 128];
#pragma unroll
    for (int i = 0; i < kMaxN / 128; ++i) fcur[i] = fnext[i];
    fetch_flags(p, u + tw, units, nc, lane, fnext);  // next unit, hidden behind this one
    const int true_n = publish_flags(fcur, nc, flagw, lane);
    if (true_n == 0 && lane == 0 && p.status) atomicOr(p.status, 1);  // :44 (NaN outputs)
    const int64_t base = (int64_t)b * p.sb + (int64_t)h * p.sh;
    float* norms = norms_all ? norms_all + (int64_t)u * 2 * N : nullptr;

    // Pass 1 (:328-361): S = K~^T V, streamed over 32-row chunks.
    float2 acc[4][4];
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int x = 0; x < 4; ++x) acc[y][x] = f2(0.f, 0.f);
    for (int c = 0; c < nc; ++c, ++j) {
      const int s = (int)(j % NSTG);
      mbar_wait(&bar[s], (uint32_t)((j / NSTG) & 1));
      uint8_t* Kt = ws + s * PL::kStage;
      const int rows = min(32, N - 32 * c);
      normalize_tile(Kt, rows, flagw[c], eps, nullptr, norms ? norms + N + 32 * c : nullptr,
                     lane);
      __syncwarp();
      row_reduce_tile(Kt, Kt + kTile, rows, acc, lane);
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        issue(j + NSTG);
      }
    }
    store_rowmajor(Sm, acc, 1.0f, lane);
    __syncwarp();
    if (gS_all) {  // saved state for the backward
      float4* dst = reinterpret_cast<float4*>(gS_all + (int64_t)u * 1024);
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[lane + 32 * i] = reinterpret_cast<const float4*>(Sm)[lane + 32 * i];
    }
    if (!want_q) continue;

    // Pass 2 (:363-388): O = s * Q~ S for every row (padded rows included).
    const float scale = true_n > 0 ? scale_of(tab, true_n, p.m) : __int_as_float(0x7fc00000);
    for (int c = 0; c < nc; ++c, ++j) {
      const int s = (int)(j % NSTG);
      mbar_wait(&bar[s], (uint32_t)((j / NSTG) & 1));
      const uint8_t* Qt = ws + s * PL::kStage;
      float2 o[4][4];
      row_output_tile(Qt, Sm, o, lane);
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int r = 32 * c + rg + 8 * jj;
        float qv[8];
        own_cols(Qt, jj, lane, qv);
        float ss = 0.f;
#pragma unroll
        for (int x = 0; x < 8; ++x) ss = fmaf(qv[x], qv[x], ss);
        ss = row_sum4(ss);
        const float nrm = sqrtf(ss + eps);
        const float w = scale * (1.0f / nrm);
        if (r < N) {
          float v[8];
          unpack(o[jj], v);
#pragma unroll
          for (int x = 0; x < 8; ++x) v[x] *= w;
          if (O) store_row(O + base + (int64_t)r * p.sn, cg, v);
          if (norms && cg == 0) norms[r] = nrm;
        }
      }
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        issue(j + NSTG);
      }
    }
  }
}

// ---- backward ----------------------------------------------------------------

template <int NSTG>
__global__ void __launch_bounds__(256) cos_bwd_d32_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
    const OpParams p, const __grid_constant__ ScaleTable tab) {
  using PL = WarpPlan<true, NSTG>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  uint8_t* ws = smem + warp * PL::bytes;
  float* St = reinterpret_cast<float*>(ws + PL::off_mat);  // S^T, later dA^T
  float* dAt = St;
  float* dA = reinterpret_cast<float*>(ws + PL::off_mat2);
  float* inv = reinterpret_cast<float*>(ws + PL::off_inv);
  uint32_t* flagw = reinterpret_cast<uint32_t*>(ws + PL::off_flag);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ws + PL::off_bar);

  const int N = (int)p.N, H = (int)p.H;
  const int units = (int)(p.B * p.H);
  const int nc = (N + 31) / 32;
  const int gw = blockIdx.x * wpc + warp, tw = gridDim.x * wpc;
  const int J = 2 * nc;
  const int my_units = gw < units ? (units - 1 - gw) / tw + 1 : 0;
  const long total = (long)my_units * J;
  if (my_units == 0) return;

  if (lane == 0) {
    for (int s = 0; s < NSTG; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
    prefetch_map(&tq);
    prefetch_map(&tdo);
    prefetch_map(&tk);
    prefetch_map(&tv);
  }
  __syncwarp();
  auto issue = [&](long j) {  // lane 0: phase A chunks (Q, dO), then phase B (K, V)
    if (j >= total) return;
    const int k = (int)(j / J), t = (int)(j - (long)k * J);
    const int u = gw + k * tw;
    const int b = u / H, h = u - b * H;
    const int s = (int)(j % NSTG);
    uint8_t* st = ws + s * PL::kStage;
    const bool a = t < nc;
    const int row = 32 * (a ? t : t - nc);
    mbar_expect_tx(&bar[s], 2 * kTile);
    tma_load_4d(st, a ? &tq : &tk, 0, row, h, b, &bar[s]);
    tma_load_4d(st + kTile, a ? &tdo : &tv, 0, row, h, b, &bar[s]);
  };
  if (lane == 0)
    for (int j = 0; j < NSTG; ++j) issue(j);

  const float eps = (float)p.eps;
  const int rg = lane >> 2, cg = lane & 3;
  const int ag = lane >> 3, bg = lane & 7;
  float* dQ = static_cast<float*>(p.dq);
  float* dK = static_cast<float*>(p.dk);
  float* dV = static_cast<float*>(p.dv);
  const float* gS_all = static_cast<const float*>(p.saved_S);
  uint32_t fnext[kMaxN / 128];
  fetch_flags(p, gw, units, nc, lane, fnext);
  float4 snext[8];  // row `lane` of the next unit's saved S
  {
    const float4* src = reinterpret_cast<const float4*>(gS_all + (int64_t)gw * 1024 + lane * 32);
#pragma unroll
    for (int i = 0; i < 8; ++i) snext[i] = __ldg(src + i);
  }
  long j = 0;
  for (int k = 0; k < my_units; ++k) {
    const int u = gw + k * tw;
    const int b = u / H, h = u - b * H;
    // S^T[c][a] = S[a][c]: lane a writes column a (conflict-free).
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      St[(4 * i + 0) * 32 + lane] = snext[i].x;
      St[(4 * i + 1) * 32 + lane] = snext[i].y;
      St[(4 * i + 2) * 32 + lane] = snext[i].z;
      St[(4 * i + 3) * 32 + lane] = snext[i].w;
    }
    uint32_t fcur[kMaxN / 128];
#pragma unroll
    for (int i = 0; i < kMaxN / 128; ++i) fcur[i] = fnext[i];
    if (u + tw < units) {  // next unit's flags and S, hidden behind this unit
      fetch_flags(p, u + tw, units, nc, lane, fnext);
      const float4* src =
          reinterpret_cast<const float4*>(gS_all + (int64_t)(u + tw) * 1024 + lane * 32);
#pragma unroll
      for (int i = 0; i < 8; ++i) snext[i] = __ldg(src + i);
    }
    const int true_n = publish_flags(fcur, nc, flagw, lane);  // includes __syncwarp
    if (true_n == 0 && lane == 0) {
      if (p.status) atomicOr(p.status, 1);
    }
    const float scale = true_n > 0 ? scale_of(tab, true_n, p.m) : __int_as_float(0x7fc00000);
    const int64_t base = (int64_t)b * p.sb + (int64_t)h * p.sh;

    // Phase A: dQ (:410-411, :421-428) and G = Q~^T dO (:405), every row.
    float2 acc[4][4];
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int x = 0; x < 4; ++x) acc[y][x] = f2(0.f, 0.f);
    for (int c = 0; c < nc; ++c, ++j) {
      const int s = (int)(j % NSTG);
      mbar_wait(&bar[s], (uint32_t)((j / NSTG) & 1));
      uint8_t* Qt = ws + s * PL::kStage;
      const uint8_t* Gt = Qt + kTile;  // dO
      const int rows = min(32, N - 32 * c);
      normalize_tile(Qt, rows, 0xffffffffu, eps, inv, nullptr, lane);
      __syncwarp();
      float2 o[4][4];
      row_output_tile(Gt, St, o, lane);  // dO S^T (unscaled)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int rl = rg + 8 * jj;
        const int r = 32 * c + rl;
        float g[8], qh[8];
        unpack(o[jj], g);
        own_cols(Qt, jj, lane, qh);
        float pr = 0.f;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          g[x] *= scale;
          pr = fmaf(g[x], qh[x], pr);
        }
        pr = row_sum4(pr);
        if (r < N) {
          const float iv = inv[rl];
#pragma unroll
          for (int x = 0; x < 8; ++x) g[x] = (g[x] - pr * qh[x]) * iv;
          store_row(dQ + base + (int64_t)r * p.sn, cg, g);
        }
      }
      row_reduce_tile(Qt, Gt, rows, acc, lane);
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        issue(j + NSTG);
      }
    }
    // dm = -ln(n) s <G, S> (:408): lane's block of G against S[a][b] = S^T[b][a].
    {
      float d = 0.f;
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const float* row = St + (4 * bg + y) * 32 + 8 * ag;
        const float4 s0 = *reinterpret_cast<const float4*>(row);
        const float4 s1 = *reinterpret_cast<const float4*>(row + 4);
        d = fmaf(acc[y][0].x, s0.x, d);
        d = fmaf(acc[y][0].y, s0.y, d);
        d = fmaf(acc[y][1].x, s0.z, d);
        d = fmaf(acc[y][1].y, s0.w, d);
        d = fmaf(acc[y][2].x, s1.x, d);
        d = fmaf(acc[y][2].y, s1.y, d);
        d = fmaf(acc[y][3].x, s1.z, d);
        d = fmaf(acc[y][3].y, s1.w, d);
      }
      double dot = (double)d;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (lane == 0 && p.dm_unit)
        p.dm_unit[u] = true_n > 0 ? coef_of(tab, true_n, p.m) * dot
                                  : __longlong_as_double(0x7ff8000000000000ll);
    }
    __syncwarp();  // S^T reads done: dA^T may overwrite it
    store_rowmajor(dA, acc, scale, lane);    // dA = s G (:412-413)
    store_transposed(dAt, acc, scale, lane);
    __syncwarp();

    // Phase B: dV = K~ dA (:416), dK~ = V dA^T (:415) -> dK (:430-437); padded rows 0 (:439).
    for (int c = 0; c < nc; ++c, ++j) {
      const int s = (int)(j % NSTG);
      mbar_wait(&bar[s], (uint32_t)((j / NSTG) & 1));
      uint8_t* Kt = ws + s * PL::kStage;
      const uint8_t* Vt = Kt + kTile;
      const int rows = min(32, N - 32 * c);
      const uint32_t vw = flagw[c];
      float* krow = dK + base + (int64_t)(32 * c + rg) * p.sn;
      float* vrow = dV + base + (int64_t)(32 * c + rg) * p.sn;
      if (vw == 0u) {  // whole chunk padded: exact zeros, nothing to compute
        const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          if (rg + 8 * jj < rows) {
            store_row(krow + (int64_t)8 * jj * p.sn, cg, z);
            store_row(vrow + (int64_t)8 * jj * p.sn, cg, z);
          }
      } else {
        normalize_tile(Kt, rows, vw, eps, inv, nullptr, lane);
        __syncwarp();
        float2 o[4][4];
        row_output_tile(Kt, dA, o, lane);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int rl = rg + 8 * jj;
          if (rl < rows) {
            float v[8];
            unpack(o[jj], v);
            if (!((vw >> rl) & 1u))
#pragma unroll
              for (int x = 0; x < 8; ++x) v[x] = 0.f;
            store_row(vrow + (int64_t)8 * jj * p.sn, cg, v);
          }
        }
        row_output_tile(Vt, dAt, o, lane);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int rl = rg + 8 * jj;
          float g[8], kh[8];
          unpack(o[jj], g);
          own_cols(Kt, jj, lane, kh);
          float pr = 0.f;
#pragma unroll
          for (int x = 0; x < 8; ++x) pr = fmaf(g[x], kh[x], pr);
          pr = row_sum4(pr);
          if (rl < rows) {
            const bool valid = (vw >> rl) & 1u;
            const float iv = inv[rl];
#pragma unroll
            for (int x = 0; x < 8; ++x) g[x] = valid ? (g[x] - pr * kh[x]) * iv : 0.f;
            store_row(krow + (int64_t)8 * jj * p.sn, cg, g);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        issue(j + NSTG);
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

// 4-D map over (D, N, H, B), (32, 32, 1, 1) box, 128-byte swizzle; rows past
// N fall outside the map and are zero-filled.
inline bool make_unit_map(CUtensorMap* map, const void* base, const OpParams& p) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)p.D, (cuuint64_t)p.N, (cuuint64_t)p.H, (cuuint64_t)p.B};
  cuuint64_t strides[3] = {(cuuint64_t)p.sn * 4, (cuuint64_t)p.sh * 4, (cuuint64_t)p.sb * 4};
  cuuint32_t box[4] = {32, 32, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline bool d32_layout_ok(const OpParams& p, std::initializer_list<const void*> ptrs) {
  if (p.D != 32 || p.N < 1 || p.N > d32::kMaxN) return false;
  if ((p.sn * 4) % 16 || (p.sh * 4) % 16 || (p.sb * 4) % 16) return false;
  if (p.B * p.H > (1ll << 31) - 1) return false;
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<uintptr_t>(q) & 15)) return false;
  return encode_fn() != nullptr;
}

template <typename T>
inline bool fast_fwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, float>::value) {
    return false;
  } else {
    return d32_layout_ok(p, {p.q, p.k, p.v, p.out, p.saved_S});
  }
}
template <typename T>
inline bool fast_bwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, float>::value) {
    return false;
  } else {
    return p.saved_S != nullptr &&
           d32_layout_ok(p, {p.q, p.k, p.v, p.dout, p.dq, p.dk, p.dv, p.saved_S});
  }
}

inline d32::ScaleTable scale_table(double m, int N) {
  d32::ScaleTable t{};
  t.s[0] = std::nanf("");
  t.coef[0] = std::nan("");
  for (int n = 1; n <= std::min(N, d32::kTabN); ++n) {
    const double ln = std::log(static_cast<double>(n));
    const double s = std::exp(-m * ln);  // attention.cpp:304 / :403, in fp64
    t.s[n] = static_cast<float>(s);
    t.coef[n] = -ln * static_cast<double>(t.s[n]);
  }
  return t;
}

inline int sm_count() {
  static int n = [] {
    int dev = 0, c = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    return c;
  }();
  return n;
}

// Persistent launch: one CTA per SM with as many unit-warps as fit in shared
// memory (<= 8), but never more warps than units.
template <typename Kern, typename... Args>
inline cudaError_t launch_warps(Kern kern, uint32_t per_warp, int units, cudaStream_t st,
                                Args... args) {
  const int wpc = std::max(1, std::min<int>(8, (int)((227u * 1024u) / per_warp)));
  const int total = std::min(units, wpc * sm_count());
  const int grid = (total + wpc - 1) / wpc;
  const uint32_t smem = per_warp * (uint32_t)wpc;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, wpc * 32, smem, st>>>(args...);
  return cudaGetLastError();
}

constexpr int kFwdStages = 3;
constexpr int kBwdStages = 3;

template <typename T>
inline int launch_fast_fwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv;
  if (!make_unit_map(&mq, p.q, p) || !make_unit_map(&mk, p.k, p) || !make_unit_map(&mv, p.v, p))
    return -1;
  const d32::ScaleTable tab = scale_table(p.m, (int)p.N);
  const cudaError_t e = launch_warps(d32::cos_fwd_d32_kernel<kFwdStages>,
                                     d32::WarpPlan<false, kFwdStages>::bytes, (int)(p.B * p.H), st,
                                     mq, mk, mv, p, tab);
  return e == cudaSuccess ? 1 : -1;
}
template <typename T>
inline int launch_fast_bwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mg;
  if (!make_unit_map(&mq, p.q, p) || !make_unit_map(&mk, p.k, p) ||
      !make_unit_map(&mv, p.v, p) || !make_unit_map(&mg, p.dout, p))
    return -1;
  const d32::ScaleTable tab = scale_table(p.m, (int)p.N);
  const cudaError_t e = launch_warps(d32::cos_bwd_d32_kernel<kBwdStages>,
                                     d32::WarpPlan<true, kBwdStages>::bytes, (int)(p.B * p.H), st,
                                     mq, mk, mv, mg, p, tab);
  return e == cudaSuccess ? 1 : -1;
}

}  // namespace cotten
