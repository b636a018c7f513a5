// Fast fp32 cosine-attention kernels for head_dim 32 (the ML-1M / ML-20M /
// Beauty shapes: model d = 64 over 2 heads) and seq_len <= 256.
//
// Persistent, warp-specialised CTAs (a few per SM, sized from the shared-
// memory budget).  One producer warp streams each unit's N x 32 tiles
// (cp.async.bulk.tensor, 128-byte swizzle) into a ring of NS shared-memory
// slots guarded by full/empty mbarriers, in the order the consumers need
// them — forward: K, V, Q; backward: Q, dO, K, V — so the next unit's tiles
// land while the current one is computed.  NW = ceil(N/32) consumer warps;
// warp w owns rows [32w, 32w+32) of every tile.  Per row block it
//   * normalises its rows in place (8 lanes per row, shuffle-reduced norms),
//   * accumulates a 32x32 row-reduction  R += x_i^T y_i   (S = K~^T V,
//     G = Q~^T dO): lane (ag, bg) holds R[8ag..8ag+8][4bg..4bg+4] as 16
//     float2 accumulators updated with FFMA2 (packed fp32 FMA with one
//     scalar operand broadcast) — 16 FFMA2 per row for 3 LDS.128,
//   * or emits a row-output  o_i = x_i M  (O = Q S, dQ~ = dO S^T,
//     dV = K~ dA, dK~ = V dA^T): lane (rg, cg) holds rows rg+8j (j<4) x
//     columns {4cg..4cg+3, 16+4cg..16+4cg+3}, again 16 FFMA2 per contraction
//     step for 3 LDS.128; the 128-byte swizzle puts the 8 row groups on 8
//     distinct bank groups.
// All swizzled addresses are per-lane base registers plus immediates.  Per-
// warp partial reductions are summed through shared memory in a fixed order
// (deterministic), overlaying the tiles they were computed from.  Nothing
// but the outputs and the 4 KB state S reaches HBM: no Q~, K~ or N x N.
// Mask semantics follow attention.cpp exactly: padded K rows are selected to
// zero (never read), dK / dV rows of padded positions are exact zeros, Q and
// dQ cover every row, s = exp(-m ln true_n) is computed in fp64 on the host.
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
constexpr int kMaxN = 256;

// Per-call constants the host computes in fp64 exactly as attention.cpp:
// s[n] = exp(-m ln n) (:303-304, :402-403), coef[n] = -ln(n) * s[n] (:408).
struct ScaleTable {
  float s[kMaxN + 1];
  double coef[kMaxN + 1];
};

// A slot holds round8(N) rows (rows [N, round8(N)) are kept zero so row
// reductions run whole 8-row groups), rounded up to the 1 KB alignment of the
// 128B swizzle.  Row-outputs of a last 32-row block may read up to 31 rows
// past it (into the next slot or the matrices after the ring); those rows
// only feed outputs that are never stored.
__host__ __device__ constexpr uint32_t tile_bytes(int N) {
  // >= 4 KB: a slot must also hold one warp's 32x32 partial sums
  return (((uint32_t)(N + 7) / 8u * 8u * kRowBytes) + 1023u) / 1024u * 1024u < 4096u
             ? 4096u
             : (((uint32_t)(N + 7) / 8u * 8u * kRowBytes) + 1023u) / 1024u * 1024u;
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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps until the phase
// completes instead of spinning on issue slots the co-resident CTA needs.
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
// Named barrier 1 over the consumer warps only (the producer never joins).
template <int NW>
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
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

// ---- building blocks (warp-level; X, Y are 128B-swizzled tiles) ------------

// In place: x <- valid ? x / sqrt(|x|^2 + eps) : 0 for rows [r0, r0+32) ∩ [0, N)
// (attention.cpp:83-87, :334-342, :366-372); inv[r] <- 1/sqrt(..) (0 if padded).
__device__ __forceinline__ void normalize_rows(uint8_t* X, int r0, int N, const uint8_t* flag,
                                               float eps, float* inv, float* norm_out,
                                               int lane) {
  const int sub = lane >> 3, c = lane & 7;
  uint8_t* be = X + (r0 + sub) * kRowBytes + ((c ^ sub) << 4);        // rows with (r&7) = sub
  uint8_t* bo = X + (r0 + sub) * kRowBytes + ((c ^ (sub + 4)) << 4);  // rows with (r&7) = sub+4
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const int r = r0 + 4 * g + sub;
    if (r0 + 4 * g >= N) break;  // warp-uniform
    uint8_t* a = (g & 1 ? bo : be) + 512 * g;
    float4 x = ld4(a);
    float ss = x.x * x.x;
    ss = fmaf(x.y, x.y, ss);
    ss = fmaf(x.z, x.z, ss);
    ss = fmaf(x.w, x.w, ss);
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    ss += __shfl_xor_sync(0xffffffffu, ss, 4);
    if (r < N) {
      const bool valid = flag == nullptr || flag[r] != 0;
      // MUFU.RSQ (<= 2 ulp): the IEEE sqrt + divide sequences cost ~25
      // instructions per row group and 10 KB of code, for no visible accuracy
      const float iv = rsqrtf(ss + eps);
      const float nrm = (ss + eps) * iv;
      x = valid ? make_float4(x.x * iv, x.y * iv, x.z * iv, x.w * iv)
                : make_float4(0.f, 0.f, 0.f, 0.f);
      st4(a, x);
      if (c == 0) {
        if (inv != nullptr) inv[r] = valid ? iv : 0.f;
        if (norm_out != nullptr) norm_out[r] = valid ? nrm : 1.0f;  // :336, :343
      }
    }
  }
}

// acc[y][p] += x[8ag+2p .. +1] * y[4bg+y] for rows [r0, min(r0+32, round8(N))).
// Rows in [N, round32(N)) of every slot are zero (see zero_tails).
__device__ __forceinline__ void row_reduce(const uint8_t* X, const uint8_t* Y, int r0, int N,
                                           float2 (&acc)[4][4], int lane) {
  const int ag = lane >> 3, bg = lane & 7;
  const uint8_t* xb = X + r0 * kRowBytes;
  const uint8_t* yb = Y + r0 * kRowBytes;
#pragma unroll 1
  for (int t = 0; t < 4; ++t) {
    if (r0 + 8 * t >= N) break;  // warp-uniform
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int rr = 8 * t + s;
      const float4 x0 = ld4(xb + rr * kRowBytes + (((2 * ag) ^ s) << 4));
      const float4 x1 = ld4(xb + rr * kRowBytes + (((2 * ag + 1) ^ s) << 4));
      const float4 y = ld4(yb + rr * kRowBytes + ((bg ^ s) << 4));
      const float2 xp[4] = {f2(x0.x, x0.y), f2(x0.z, x0.w), f2(x1.x, x1.y), f2(x1.z, x1.w)};
#pragma unroll
      for (int yy = 0; yy < 4; ++yy)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[yy][p] = fma2(xp[p], sel4(y, yy), acc[yy][p]);
    }
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

// o[j][.] (row r0+rg+8j, columns chunk cg then chunk cg+4) = x_row . M with M
// a plain row-major 32x32 fp32 matrix in shared memory.  Rows >= N produce
// values that are never stored.
__device__ __forceinline__ void row_output(const uint8_t* X, const float* M, int r0,
                                           float2 (&o)[4][4], int lane) {
  const int rg = lane >> 2, cg = lane & 3;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int p = 0; p < 4; ++p) o[j][p] = f2(0.f, 0.f);
  const uint8_t* xb = X + (r0 + rg) * kRowBytes;
  const float* mb = M + 4 * cg;
  // Not unrolled over c: the fully unrolled form (650 SASS instructions per
  // call site, ~100 KB for the backward) thrashed the instruction cache.
#pragma unroll 1
  for (int c = 0; c < 8; ++c) {
    const uint8_t* xc = xb + ((c ^ rg) << 4);  // (r & 7) == rg for all four rows
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

// The 8 values of row r0+rg+8j that lane (rg, cg) owns in a row-output.
__device__ __forceinline__ void own_cols(const uint8_t* X, int r0, int j, int lane,
                                         float (&v)[8]) {
  const int rg = lane >> 2, cg = lane & 3;
  const uint8_t* xb = X + (r0 + rg + 8 * j) * kRowBytes;
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
__device__ __forceinline__ float row_sum4(float x) {  // over the 4 lanes of a row
  x += __shfl_xor_sync(0xffffffffu, x, 1);
  x += __shfl_xor_sync(0xffffffffu, x, 2);
  return x;
}

// Sum the NW per-warp partials (spread over two tiles: warps < half in A,
// the rest in B) into dst[e] in a fixed order; returns the per-thread
// float4s in out4 (PER of them).
template <int NW, int PER>
__device__ __forceinline__ void reduce_partials(const float* A, const float* B, int tid,
                                                float4 (&out4)[PER]) {
  constexpr int HALF = (NW + 1) / 2;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e4 = tid + k * NW * 32;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e4 < 256) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const float* src = (w < HALF ? A + w * 1024 : B + (w - HALF) * 1024);
        const float4 t = reinterpret_cast<const float4*>(src)[e4];
        s.x += t.x;
        s.y += t.y;
        s.z += t.z;
        s.w += t.w;
      }
    }
    out4[k] = s;
  }
}
template <int NW>
__device__ __forceinline__ float* partial_slot(uint8_t* A, uint8_t* B, int warp) {
  constexpr int HALF = (NW + 1) / 2;
  return reinterpret_cast<float*>(warp < HALF ? A + warp * 4096 : B + (warp - HALF) * 4096);
}

// ---- ring + shared-memory plan --------------------------------------------

struct Plan {
  uint32_t tb;       // bytes per slot
  int ns;            // slots
  uint32_t off_ring, off_mat, off_inv, off_flag, off_misc, off_bar, bytes;
  // mats: forward S (4 KB); backward S^T, dA, dA^T (12 KB)
  __host__ __device__ Plan(int N, int NS, bool bwd) {
    tb = tile_bytes(N);
    ns = NS;
    off_ring = 0;
    off_mat = off_ring + (uint32_t)NS * tb;
    off_inv = off_mat + (bwd ? 2 * 4096 : 4096);  // bwd: [S^T | dA^T] overlay, then dA
    off_flag = off_inv + (bwd ? 2 * kMaxN * 4 : 0);
    off_misc = off_flag + kMaxN;  // per-warp counts (8 ints), then dm partials (8 doubles)
    off_bar = off_misc + 32 + 8 * 8;
    bytes = off_bar + 2 * 8 * (uint32_t)NS;  // full[NS], empty[NS]
  }
};

struct RingPos {
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next(int ns) {
    if (++slot == ns) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

// Zero rows [N, round8(N)) of every slot once, so row-reductions may run
// whole 8-row groups and row-outputs never read uninitialised memory.
__host__ __device__ constexpr uint32_t tail_end(int N) { return (uint32_t)(N + 7) / 8u * 8u * kRowBytes; }

__device__ __forceinline__ void zero_tails(uint8_t* ring, const Plan& pl, int N, int tid,
                                           int nthreads) {
  const uint32_t lo = (uint32_t)N * kRowBytes;
  const uint32_t per = (tail_end(N) - lo) / 16;
  for (uint32_t i = tid; i < per * (uint32_t)pl.ns; i += nthreads) {
    const uint32_t s = i / per, k = i - s * per;
    st4(ring + s * pl.tb + lo + 16 * k, make_float4(0.f, 0.f, 0.f, 0.f));
  }
}

// Consumer-side, one unit ahead: the valid flag of row tid of unit u's
// sequence (registers; consumed by publish_flags at the next unit).
__device__ __forceinline__ int fetch_flag(const OpParams& p, int u, int units, int tid) {
  if (u >= units || tid >= (int)p.N) return 0;
  if (p.valid == nullptr) return 1;
  const int64_t b = u / (int)p.H;
  return __ldg(p.valid + b * p.msb + tid) != 0;
}
// Saved S of unit u (backward), one unit ahead: element pairs (a, c4..c4+3).
template <int PERS, int NW>
__device__ __forceinline__ void fetch_S(const OpParams& p, int u, int units, int tid,
                                        float4 (&sr)[PERS]) {
  if (u >= units) return;
  const float* gS = static_cast<const float*>(p.saved_S) + (int64_t)u * 1024;
#pragma unroll
  for (int k = 0; k < PERS; ++k) {
    const int i = tid + k * NW * 32;
    if (i < 256) sr[k] = __ldg(reinterpret_cast<const float4*>(gS + (i & 31) * 32 + (i >> 5) * 4));
  }
}
// Valid flags into flag[] and true_n (attention.cpp:26-33); one consumer sync.
template <int NW>
__device__ __forceinline__ int publish_flags(int f, int N, uint8_t* flag, int* cnt, int tid) {
  if (tid < N) flag[tid] = (uint8_t)f;  // NW*32 >= N
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if ((tid & 31) == 0) cnt[tid >> 5] = __popc(m);
  consumer_sync<NW>();
  int n = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) n += cnt[w];
  return n;
}

// ---- forward ---------------------------------------------------------------

template <int NW, int NS>
__global__ void __launch_bounds__((NW + 1) * 32) cos_fwd_d32_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const OpParams p,
    const __grid_constant__ ScaleTable tab) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const KernelStamp stamp_(p);
  const int N = (int)p.N, H = (int)p.H;
  const int units = (int)(p.B * p.H);
  const Plan pl(N, NS, false);
  uint8_t* ring = smem + pl.off_ring;
  float* Ss = reinterpret_cast<float*>(smem + pl.off_mat);
  uint8_t* flag = smem + pl.off_flag;
  int* cnt = reinterpret_cast<int*>(smem + pl.off_misc);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + pl.off_bar);
  uint64_t* empty = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bytes = (uint32_t)N * kRowBytes;
  float* O = static_cast<float*>(p.out);
  float* norms_all = static_cast<float*>(p.saved_norms);
  const bool want_q = O != nullptr || norms_all != nullptr;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  zero_tails(ring, pl, N, threadIdx.x, blockDim.x);
  __syncthreads();

  if (warp == NW) {  // ===== producer =====
    if (lane == 0) {
      prefetch_map(&tk);
      prefetch_map(&tv);
      prefetch_map(&tq);
      RingPos pos;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        for (int t = 0; t < (want_q ? 3 : 2); ++t) {
          mbar_wait(&empty[pos.slot], pos.phase ^ 1u);
          mbar_expect_tx(&full[pos.slot], bytes);
          tma_load_4d(ring + pos.slot * pl.tb, t == 0 ? &tk : t == 1 ? &tv : &tq, 0, 0, h, b,
                      &full[pos.slot]);
          pos.next(NS);
        }
      }
    }
    return;
  }

  // ===== consumers =====
  const int tid = threadIdx.x;
  const float eps = (float)p.eps;
  const int r0 = warp * 32;
  const int rg = lane >> 2, cg = lane & 3;
  float* gS_all = static_cast<float*>(p.saved_S);
  RingPos pos;
  int fnext = fetch_flag(p, blockIdx.x, units, tid);
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int b = u / H, h = u - b * H;
    const int fcur = fnext;
    fnext = fetch_flag(p, u + gridDim.x, units, tid);  // hidden behind this unit
    const int sk = pos.slot;
    const uint32_t phk = pos.phase;
    pos.next(NS);
    const int sv = pos.slot;
    const uint32_t phv = pos.phase;
    pos.next(NS);
    int sq = -1;
    uint32_t phq = 0;
    if (want_q) {
      sq = pos.slot;
      phq = pos.phase;
      pos.next(NS);
    }
    uint8_t* Kt = ring + sk * pl.tb;
    uint8_t* Vt = ring + sv * pl.tb;
    const int true_n = publish_flags<NW>(fcur, N, flag, cnt, tid);
    const int64_t base = (int64_t)b * p.sb + (int64_t)h * p.sh;
    float* norms = norms_all ? norms_all + (int64_t)u * 2 * N : nullptr;
    if (true_n == 0) {  // UsageError in the reference (attention.cpp:44): NaN outputs
      if (tid == 0 && p.status) atomicOr(p.status, 1);
      if (O)
        for (int i = tid; i < N * kD; i += NW * 32)
          O[base + (int64_t)(i / kD) * p.sn + (i % kD)] = __int_as_float(0x7fc00000);
      mbar_wait(&full[sk], phk);
      mbar_wait(&full[sv], phv);
      if (sq >= 0) mbar_wait(&full[sq], phq);
      consumer_sync<NW>();
      if (tid == 0) {
        mbar_arrive(&empty[sk]);
        mbar_arrive(&empty[sv]);
        if (sq >= 0) mbar_arrive(&empty[sq]);
      }
      continue;
    }

    // Pass 1 (:328-361): S = K~^T V.
    float2 acc[4][4];
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int x = 0; x < 4; ++x) acc[y][x] = f2(0.f, 0.f);
    mbar_wait(&full[sk], phk);
    mbar_wait(&full[sv], phv);
    normalize_rows(Kt, r0, N, flag, eps, nullptr, norms ? norms + N : nullptr, lane);
    __syncwarp();
    row_reduce(Kt, Vt, r0, N, acc, lane);
    consumer_sync<NW>();  // every warp done with K~, V: partials overlay them
    store_partial(partial_slot<NW>(Kt, Vt, warp), acc, lane);
    consumer_sync<NW>();
    {
      constexpr int PER = (256 + NW * 32 - 1) / (NW * 32);
      float4 s4[PER];
      reduce_partials<NW, PER>(reinterpret_cast<float*>(Kt), reinterpret_cast<float*>(Vt), tid,
                               s4);
      float* gS = gS_all ? gS_all + (int64_t)u * 1024 : nullptr;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e4 = tid + k * NW * 32;
        if (e4 < 256) {
          reinterpret_cast<float4*>(Ss)[e4] = s4[k];
          if (gS) reinterpret_cast<float4*>(gS)[e4] = s4[k];
        }
      }
    }
    if (N * kRowBytes < (uint32_t)((NW + 1) / 2) * 4096u) {  // partials spilled into tails
      consumer_sync<NW>();
      for (int i = tid; i < (int)((tail_end(N) - N * kRowBytes) / 16); i += NW * 32) {
        st4(Kt + N * kRowBytes + 16 * i, make_float4(0.f, 0.f, 0.f, 0.f));
        st4(Vt + N * kRowBytes + 16 * i, make_float4(0.f, 0.f, 0.f, 0.f));
      }
    }
    consumer_sync<NW>();  // S complete; K, V slots free
    if (tid == 0) {
      mbar_arrive(&empty[sk]);
      mbar_arrive(&empty[sv]);
    }
    if (!want_q) continue;

    // Pass 2 (:363-388): O = s * Q~ S for every row (padded rows included).
    uint8_t* Qt = ring + sq * pl.tb;
    const float scale = p.m_dev ? (float)exp(-*p.m_dev * log((double)true_n)) : tab.s[true_n];
    mbar_wait(&full[sq], phq);
    float2 o[4][4];
    row_output(Qt, Ss, r0, o, lane);
    float* orow = O ? O + base + (int64_t)(r0 + rg) * p.sn : nullptr;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + rg + 8 * j;
      float qv[8];
      own_cols(Qt, r0, j, lane, qv);
      float ss = 0.f;
#pragma unroll
      for (int x = 0; x < 8; ++x) ss = fmaf(qv[x], qv[x], ss);
      ss = row_sum4(ss);
      const float iv = rsqrtf(ss + eps);
      const float nrm = (ss + eps) * iv;
      const float w = scale * iv;
      if (r < N) {
        float v[8];
        unpack(o[j], v);
#pragma unroll
        for (int x = 0; x < 8; ++x) v[x] *= w;
        if (orow) store_row(orow + (int64_t)8 * j * p.sn, cg, v);
        if (norms && cg == 0) norms[r] = nrm;
      }
    }
    consumer_sync<NW>();  // Q slot, S and flags free for the next unit
    if (tid == 0) mbar_arrive(&empty[sq]);
  }
}

// ---- backward ----------------------------------------------------------------

template <int NW, int NS>
__global__ void __launch_bounds__((NW + 1) * 32) cos_bwd_d32_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
    const OpParams p, const __grid_constant__ ScaleTable tab) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const KernelStamp stamp_(p);
  const int N = (int)p.N, H = (int)p.H;
  const int units = (int)(p.B * p.H);
  const Plan pl(N, NS, true);
  uint8_t* ring = smem + pl.off_ring;
  float* St = reinterpret_cast<float*>(smem + pl.off_mat);
  float* dA = St + 1024;
  float* dAt = St;  // S^T is dead once <G,S> is taken; dA^T reuses it
  float* inv_q = reinterpret_cast<float*>(smem + pl.off_inv);
  float* inv_k = inv_q + kMaxN;
  uint8_t* flag = smem + pl.off_flag;
  int* cnt = reinterpret_cast<int*>(smem + pl.off_misc);
  double* red = reinterpret_cast<double*>(smem + pl.off_misc + 32);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + pl.off_bar);
  uint64_t* empty = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bytes = (uint32_t)N * kRowBytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  zero_tails(ring, pl, N, threadIdx.x, blockDim.x);
  __syncthreads();

  if (warp == NW) {  // ===== producer: Q, dO, K, V per unit =====
    if (lane == 0) {
      prefetch_map(&tq);
      prefetch_map(&tdo);
      prefetch_map(&tk);
      prefetch_map(&tv);
      RingPos pos;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        for (int t = 0; t < 4; ++t) {
          mbar_wait(&empty[pos.slot], pos.phase ^ 1u);
          mbar_expect_tx(&full[pos.slot], bytes);
          const CUtensorMap* m = t == 0 ? &tq : t == 1 ? &tdo : t == 2 ? &tk : &tv;
          tma_load_4d(ring + pos.slot * pl.tb, m, 0, 0, h, b, &full[pos.slot]);
          pos.next(NS);
        }
      }
    }
    return;
  }

  // ===== consumers =====
  const int tid = threadIdx.x;
  const float eps = (float)p.eps;
  const int r0 = warp * 32;
  const int rg = lane >> 2, cg = lane & 3;
  float* dQ = static_cast<float*>(p.dq);
  float* dK = static_cast<float*>(p.dk);
  float* dV = static_cast<float*>(p.dv);
  RingPos pos;
  constexpr int PERS = (256 + NW * 32 - 1) / (NW * 32);
  float4 snext[PERS];
  fetch_S<PERS, NW>(p, blockIdx.x, units, tid, snext);
  int fnext = fetch_flag(p, blockIdx.x, units, tid);
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int b = u / H, h = u - b * H;
    // S^T from the prefetched saved state: St[c][a] = S[a][c] (a = lane: conflict-free)
#pragma unroll
    for (int k = 0; k < PERS; ++k) {
      const int i = tid + k * NW * 32;
      if (i < 256) {
        const int a = i & 31, c4 = (i >> 5) * 4;
        St[(c4 + 0) * 32 + a] = snext[k].x;
        St[(c4 + 1) * 32 + a] = snext[k].y;
        St[(c4 + 2) * 32 + a] = snext[k].z;
        St[(c4 + 3) * 32 + a] = snext[k].w;
      }
    }
    const int fcur = fnext;
    fetch_S<PERS, NW>(p, u + gridDim.x, units, tid, snext);  // next unit, hidden behind this one
    fnext = fetch_flag(p, u + gridDim.x, units, tid);
    int sl[4];
    uint32_t ph[4];
    for (int t = 0; t < 4; ++t) {
      sl[t] = pos.slot;
      ph[t] = pos.phase;
      pos.next(NS);
    }
    uint8_t* Qt = ring + sl[0] * pl.tb;
    uint8_t* Gt = ring + sl[1] * pl.tb;  // dO
    uint8_t* Kt = ring + sl[2] * pl.tb;
    uint8_t* Vt = ring + sl[3] * pl.tb;
    const int true_n = publish_flags<NW>(fcur, N, flag, cnt, tid);  // includes a consumer sync
    const int64_t base = (int64_t)b * p.sb + (int64_t)h * p.sh;
    if (true_n == 0) {
      if (tid == 0) {
        if (p.status) atomicOr(p.status, 1);
        if (p.dm_unit) p.dm_unit[u] = __longlong_as_double(0x7ff8000000000000ll);
      }
      const float qnan = __int_as_float(0x7fc00000);
      for (int i = tid; i < N * kD; i += NW * 32) {
        const int64_t o = base + (int64_t)(i / kD) * p.sn + (i % kD);
        dQ[o] = qnan;
        dK[o] = qnan;
        dV[o] = qnan;
      }
      for (int t = 0; t < 4; ++t) mbar_wait(&full[sl[t]], ph[t]);
      consumer_sync<NW>();
      if (tid == 0)
        for (int t = 0; t < 4; ++t) mbar_arrive(&empty[sl[t]]);
      continue;
    }
    const float scale = p.m_dev ? (float)exp(-*p.m_dev * log((double)true_n)) : tab.s[true_n];

    // Phase A: dQ (:410-411, :421-428) then G = Q~^T dO (:405), every row.
    mbar_wait(&full[sl[0]], ph[0]);
    mbar_wait(&full[sl[1]], ph[1]);
    normalize_rows(Qt, r0, N, nullptr, eps, inv_q, nullptr, lane);
    __syncwarp();
    {
      float2 o[4][4];
      row_output(Gt, St, r0, o, lane);  // dO S^T (unscaled)
      float* drow = dQ + base + (int64_t)(r0 + rg) * p.sn;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + rg + 8 * j;
        float g[8], qh[8];
        unpack(o[j], g);
        own_cols(Qt, r0, j, lane, qh);
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
          store_row(drow + (int64_t)8 * j * p.sn, cg, g);
        }
      }
    }
    float2 acc[4][4];
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int x = 0; x < 4; ++x) acc[y][x] = f2(0.f, 0.f);
    row_reduce(Qt, Gt, r0, N, acc, lane);
    consumer_sync<NW>();  // Q~, dO dead: partials overlay them
    store_partial(partial_slot<NW>(Qt, Gt, warp), acc, lane);
    consumer_sync<NW>();
    {
      constexpr int PER = (256 + NW * 32 - 1) / (NW * 32);
      float4 g4[PER];
      reduce_partials<NW, PER>(reinterpret_cast<float*>(Qt), reinterpret_cast<float*>(Gt), tid,
                               g4);
      double dot = 0.0;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e4 = tid + k * NW * 32;
        if (e4 < 256) {
          const int a = e4 >> 3, c = (e4 & 7) * 4;  // <G, S> (:408)
          float d = g4[k].x * St[(c + 0) * 32 + a];
          d = fmaf(g4[k].y, St[(c + 1) * 32 + a], d);
          d = fmaf(g4[k].z, St[(c + 2) * 32 + a], d);
          d = fmaf(g4[k].w, St[(c + 3) * 32 + a], d);
          dot += (double)d;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      consumer_sync<NW>();  // partials and S^T read: both regions may now be overwritten
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e4 = tid + k * NW * 32;
        if (e4 < 256) {
          const int a = e4 >> 3, c = (e4 & 7) * 4;
          const float4 s = make_float4(g4[k].x * scale, g4[k].y * scale, g4[k].z * scale,
                                       g4[k].w * scale);  // dA = s G (:412-413)
          reinterpret_cast<float4*>(dA)[e4] = s;
          dAt[(c + 0) * 32 + a] = s.x;
          dAt[(c + 1) * 32 + a] = s.y;
          dAt[(c + 2) * 32 + a] = s.z;
          dAt[(c + 3) * 32 + a] = s.w;
        }
      }
      if (N * kRowBytes < (uint32_t)((NW + 1) / 2) * 4096u)  // partials spilled into tails
        for (int i = tid; i < (int)((tail_end(N) - N * kRowBytes) / 16); i += NW * 32) {
          st4(Qt + N * kRowBytes + 16 * i, make_float4(0.f, 0.f, 0.f, 0.f));
          st4(Gt + N * kRowBytes + 16 * i, make_float4(0.f, 0.f, 0.f, 0.f));
        }
      consumer_sync<NW>();  // dA complete; Q, dO slots free
      if (lane == 0) red[warp] = dot;
      if (tid == 0) {
        mbar_arrive(&empty[sl[0]]);
        mbar_arrive(&empty[sl[1]]);
      }
    }

    // Phase B: dV = K~ dA (:416), dK~ = V dA^T (:415) -> dK (:430-437), padded rows 0 (:439).
    mbar_wait(&full[sl[2]], ph[2]);
    mbar_wait(&full[sl[3]], ph[3]);
    {
      const bool any_valid = __any_sync(0xffffffffu, r0 + lane < N && flag[r0 + lane] != 0);
      float* krow = dK + base + (int64_t)(r0 + rg) * p.sn;
      float* vrow = dV + base + (int64_t)(r0 + rg) * p.sn;
      if (!any_valid) {  // whole block padded: exact zeros, nothing to compute
        const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (r0 + rg + 8 * j < N) {
            store_row(krow + (int64_t)8 * j * p.sn, cg, z);
            store_row(vrow + (int64_t)8 * j * p.sn, cg, z);
          }
      } else {
        normalize_rows(Kt, r0, N, flag, eps, inv_k, nullptr, lane);
        __syncwarp();
        float2 o[4][4];
        row_output(Kt, dA, r0, o, lane);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = r0 + rg + 8 * j;
          if (r < N) {
            float v[8];
            unpack(o[j], v);
            if (!flag[r])
#pragma unroll
              for (int x = 0; x < 8; ++x) v[x] = 0.f;
            store_row(vrow + (int64_t)8 * j * p.sn, cg, v);
          }
        }
        row_output(Vt, dAt, r0, o, lane);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = r0 + rg + 8 * j;
          float g[8], kh[8];
          unpack(o[j], g);
          own_cols(Kt, r0, j, lane, kh);
          float pr = 0.f;
#pragma unroll
          for (int x = 0; x < 8; ++x) pr = fmaf(g[x], kh[x], pr);
          pr = row_sum4(pr);
          if (r < N) {
            const bool valid = flag[r] != 0;
            const float iv = inv_k[r];
#pragma unroll
            for (int x = 0; x < 8; ++x) g[x] = valid ? (g[x] - pr * kh[x]) * iv : 0.f;
            store_row(krow + (int64_t)8 * j * p.sn, cg, g);
          }
        }
      }
    }
    consumer_sync<NW>();  // K, V, dA, St, flags, red free for the next unit
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t += red[w];
      if (p.dm_unit) p.dm_unit[u] = (p.m_dev ? -log((double)true_n) * (double)(float)exp(-*p.m_dev * log((double)true_n)) : tab.coef[true_n]) * t;  // -ln(n) s <G,S> (:408)
      mbar_arrive(&empty[sl[2]]);
      mbar_arrive(&empty[sl[3]]);
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

inline d32::ScaleTable scale_table(double m, int N) {
  d32::ScaleTable t{};
  for (int n = 1; n <= N; ++n) {
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

// Launch a persistent ring kernel: NS = ring slots.  Grid = resident CTAs.
template <typename Kern, typename... Args>
inline cudaError_t launch_persistent(Kern kern, int threads, uint32_t smem, int units,
                                     cudaStream_t st, Args... args) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int grid = std::min(units, per_sm * sm_count());
  kern<<<grid, threads, smem, st>>>(args...);
  return cudaGetLastError();
}

// Ring depth: as many tile slots as fit in `budget` bytes, at least `min_ns`.
inline int pick_slots(int N, bool bwd, uint32_t budget, int min_ns, int max_ns) {
  int ns = max_ns;
  while (ns > min_ns && d32::Plan(N, ns, bwd).bytes > budget) --ns;
  return ns;
}

template <int NW, int NS>
inline cudaError_t fwd_nw_ns(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                             const OpParams& p, const d32::ScaleTable& tab, cudaStream_t st) {
  const d32::Plan pl((int)p.N, NS, false);
  return launch_persistent(d32::cos_fwd_d32_kernel<NW, NS>, (NW + 1) * 32, pl.bytes,
                           (int)(p.B * p.H), st, q, k, v, p, tab);
}
template <int NW, int NS>
inline cudaError_t bwd_nw_ns(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                             const CUtensorMap& g, const OpParams& p, const d32::ScaleTable& tab,
                             cudaStream_t st) {
  const d32::Plan pl((int)p.N, NS, true);
  return launch_persistent(d32::cos_bwd_d32_kernel<NW, NS>, (NW + 1) * 32, pl.bytes,
                           (int)(p.B * p.H), st, q, k, v, g, p, tab);
}

// Slot counts per kernel are chosen so that two CTAs fit per SM for the long
// tiles (N > 128: fwd 4 slots, bwd 8 slots with one CTA) and several for short.
template <int NW>
inline cudaError_t fwd_nw(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                          const OpParams& p, const d32::ScaleTable& tab, cudaStream_t st) {
  const int N = (int)p.N;
  const int ns = pick_slots(N, false, 113 * 1024, 3, 6);
  switch (ns) {
    case 3: return fwd_nw_ns<NW, 3>(q, k, v, p, tab, st);
    case 4: return fwd_nw_ns<NW, 4>(q, k, v, p, tab, st);
    case 5: return fwd_nw_ns<NW, 5>(q, k, v, p, tab, st);
    default: return fwd_nw_ns<NW, 6>(q, k, v, p, tab, st);
  }
}
template <int NW>
inline cudaError_t bwd_nw(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                          const CUtensorMap& g, const OpParams& p, const d32::ScaleTable& tab,
                          cudaStream_t st) {
  const int N = (int)p.N;
  // two (or more) CTAs per SM when a whole unit's 4 tiles fit in half the SM,
  // else one CTA with up to 8 slots
  const uint32_t budget = d32::Plan(N, 4, true).bytes <= 113 * 1024 ? 113 * 1024 : 227 * 1024;
  const int ns = pick_slots(N, true, budget, 4, 8);
  switch (ns) {
    case 4: return bwd_nw_ns<NW, 4>(q, k, v, g, p, tab, st);
    case 5: return bwd_nw_ns<NW, 5>(q, k, v, g, p, tab, st);
    case 6: return bwd_nw_ns<NW, 6>(q, k, v, g, p, tab, st);
    case 7: return bwd_nw_ns<NW, 7>(q, k, v, g, p, tab, st);
    default: return bwd_nw_ns<NW, 8>(q, k, v, g, p, tab, st);
  }
}

// Returns the number of kernel launches (1), or -1 if a tensor map could not
// be encoded (the caller reports cudaGetLastError() first).
template <typename T>
inline int launch_fast_fwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv;
  if (!make_unit_map(&mq, p.q, p) || !make_unit_map(&mk, p.k, p) || !make_unit_map(&mv, p.v, p))
    return -1;
  const d32::ScaleTable tab = scale_table(p.m, (int)p.N);
  cudaError_t e;
  switch ((int)((p.N + 31) / 32)) {
    case 1: e = fwd_nw<1>(mq, mk, mv, p, tab, st); break;
    case 2: e = fwd_nw<2>(mq, mk, mv, p, tab, st); break;
    case 3: e = fwd_nw<3>(mq, mk, mv, p, tab, st); break;
    case 4: e = fwd_nw<4>(mq, mk, mv, p, tab, st); break;
    case 5: e = fwd_nw<5>(mq, mk, mv, p, tab, st); break;
    case 6: e = fwd_nw<6>(mq, mk, mv, p, tab, st); break;
    case 7: e = fwd_nw<7>(mq, mk, mv, p, tab, st); break;
    default: e = fwd_nw<8>(mq, mk, mv, p, tab, st); break;
  }
  return e == cudaSuccess ? 1 : -1;
}
template <typename T>
inline int launch_fast_bwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mg;
  if (!make_unit_map(&mq, p.q, p) || !make_unit_map(&mk, p.k, p) ||
      !make_unit_map(&mv, p.v, p) || !make_unit_map(&mg, p.dout, p))
    return -1;
  const d32::ScaleTable tab = scale_table(p.m, (int)p.N);
  cudaError_t e;
  switch ((int)((p.N + 31) / 32)) {
    case 1: e = bwd_nw<1>(mq, mk, mv, mg, p, tab, st); break;
    case 2: e = bwd_nw<2>(mq, mk, mv, mg, p, tab, st); break;
    case 3: e = bwd_nw<3>(mq, mk, mv, mg, p, tab, st); break;
    case 4: e = bwd_nw<4>(mq, mk, mv, mg, p, tab, st); break;
    case 5: e = bwd_nw<5>(mq, mk, mv, mg, p, tab, st); break;
    case 6: e = bwd_nw<6>(mq, mk, mv, mg, p, tab, st); break;
    case 7: e = bwd_nw<7>(mq, mk, mv, mg, p, tab, st); break;
    default: e = bwd_nw<8>(mq, mk, mv, mg, p, tab, st); break;
  }
  return e == cudaSuccess ? 1 : -1;
}

}  // namespace cotten
