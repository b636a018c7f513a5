// Tensor-core (tcgen05 / TMEM) cosine-attention kernels for head_dim 32, fp32,
// any seq_len up to 16384 — the B200 hot path for the ML-1M / ML-20M / Beauty
// shapes and the d_h = 32 long-sequence sweep.
//
// Every unit (sequence b, head h) is streamed as 128-row chunks (one TMA box
// of 128 rows x 128 B, 128-byte swizzle, rows past N zero-filled by TMA):
//   forward   pass 1 over (K, V) chunks: S = K~^T V   (reduction over rows)
//             pass 2 over  Q     chunks: O = s Q~ S   (row output)
//   backward  pass 1 over (Q, dO) chunks: G = Q~^T dO, dQ~ = s dO S^T
//             pass 2 over (K, V)  chunks: dV = K~ dA,  dK~ = V dA^T   (dA = s G)
// (attention.cpp:297-395 and :397-441).  All six contractions run on the
// tensor cores as 3xTF32: every operand x is split by the worker threads
// into hi = x rounded to tf32 (low 13 mantissa bits clear) and lo = x - hi
// (exact in fp32), and the MMAs accumulate hi*hi + hi*lo + lo*hi
// (+ lo*lo for the reductions, which is free there) in fp32 TMEM — within
// ~1e-6 of fp32, well inside the 1e-5 bar, where plain TF32 is at ~4e-4.
//
//   * reductions (S, G): tcgen05.mma M=64, N=64, K=8 rows per instruction,
//     A and B both MN-major straight from the TMA tiles: A's two 32-wide
//     M atoms are [x_hi | x_lo] and B's two N atoms are [y_hi | y_lo], so one
//     instruction accumulates all four hi/lo products of 8 rows into TMEM;
//   * row outputs (O, dQ~, dV, dK~): M=128 rows, N=32, K=32 (4 k-steps x 3
//     products), A = the chunk (K-major SW128), B = the 32x32 state operand
//     (S, S^T, dA or dA^T, split hi/lo) written by the workers.
//
// Warp roles (384 threads, one CTA per SM, persistent over units; ring of 3
// slots, slot = item % 3, each = one TMA stage + one lo buffer + one TMEM
// buffer; an "item" is one 128-row chunk of one pass of one unit):
//   warps 0-3  splitter group: thread t owns row t of the chunk (= TMEM lane t):
//              row norms, masking, hi/lo split (lo into the slot's lo buffer,
//              hi in place or into TMEM as the MMA's A operand), the per-row
//              1/norm parked in TMEM for the epiloguer.
//   warps 4-7  epiloguer group: TMEM -> registers -> scale / Jacobian / mask
//              -> staged in the slot's lo buffer for the store warp; once per
//              unit the S / G epilogue (saved S, dm in a fixed order, the
//              state operands S / dA hi/lo in shared memory).
//   warp 8     TMA producer: raw chunks into the ring.
//   warp 9     MMA issuer (converged warp, one elect.sync lane) + TMEM allocator.
//   warp 10    mask warp: up to two units ahead, valid bytes -> bitmask,
//              true_n, s = exp(-m ln n), coef = -ln(n) s in fp64
//              (attention.cpp:303-304, :402-408).
//   warp 11    store warp: TMA-stores each chunk's staged outputs and frees the
//              slot's lo buffer once the store has read it.
// Nothing but the outputs, S (4 KB per unit) and dm reach HBM.
#pragma once
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kernels_d32.cuh"

namespace cotten {
namespace tc {

using d32::mbar_arrive;
using d32::mbar_expect_tx;
using d32::mbar_init;
using d32::mbar_wait;
using d32::smem_u32;
using d32::tma_load_4d;

constexpr int kRows = 128;                 // rows per chunk
constexpr uint32_t kTile = 16384;          // 128 rows x 128 B
constexpr uint32_t kStage = 2 * kTile;     // two tensors per chunk
constexpr int kRing = 3;                   // TMA stages = lo buffers = TMEM buffers
constexpr int kMaxN = 16384;               // flag bitmask capacity
// The S / G reduction accumulator is flushed into an fp32 running sum every
// kFlush chunks (512 rows), so no TMEM accumulation chain exceeds 64 MMA steps
// whatever N is (accuracy of long sequences; a no-op for N <= 512).
constexpr int kFlush = 4;
constexpr int kGroups = 2;                 // worker groups (alternate chunks)
constexpr int kWorkerWarps = 4 * kGroups;
constexpr int kWarpProducer = kWorkerWarps;
constexpr int kWarpMma = kWorkerWarps + 1;
constexpr int kWarpMask = kWorkerWarps + 2;
constexpr int kWarpStore = kWorkerWarps + 3;
// 12 warps: registers are allocated as if for 12 warps anyway (168 per thread).
constexpr int kThreads = (kWorkerWarps + 4) * 32;

// Shared-memory plan (bytes; every operand region 1024-aligned for SW128).
constexpr uint32_t kOffRaw = 0;
constexpr uint32_t kOffLo = kOffRaw + kRing * kStage;      // kRing lo buffers
constexpr uint32_t kOffOps = kOffLo + kRing * kStage;      // 6 x 4 KB state operands
constexpr uint32_t kOffFlags = kOffOps + 6 * 4096;         // 2 x 2 KB bitmasks
constexpr uint32_t kOffMisc = kOffFlags + 2 * (kMaxN / 8);  // 2 x 16 B unit constants, tmem base
constexpr uint32_t kOffBar = kOffMisc + 128;  // misc: UnitConst[2], tmem base, dm partials[4]
constexpr uint32_t kSmemBytes = kOffBar + 32 * 8;
// state operands (32 rows x 128 B each, hi/lo pairs): 0/1 = S rows (bwd: K-major
// B of dQ~ = dO S^T; fwd: 32-byte granules, MN-major B of O = Q~ S), 2/3 = dA
// rows (K-major B of dK~ = V dA^T), 4/5 = dA rows in 32-byte granules (MN-major
// B of dV = K~ dA)
constexpr uint32_t kOpBytes = 4096;

// TMEM: 512 columns.  Backward: [0, 64) G; buffer b at kBwdBuf0 + 128 b:
// pass 1 [+0, +32) dQ~, [+32, +96) dO hi/lo A operand, [+96, +128) q~;
// pass 2 [+0, +32) dV, [+32, +64) dK~, [+64, +128) K~ hi/lo A operand
// (V, the A operand of dK~ = V dA^T, stays in shared memory); the row's
// 1/norm at column kBwdInv + b (all three splitter -> epiloguer hand-offs).
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kBwdBuf0 = 64;
constexpr uint32_t kBwdBufCols = 128;
constexpr uint32_t kBwdInv = kBwdBuf0 + kRing * kBwdBufCols;
// Forward: [0, 64) S; buffer b at kFwdBuf0 + 96 b: [+0, +32) O,
// [+32, +96) Q~ hi/lo A operand.
constexpr uint32_t kFwdBuf0 = 64;
constexpr uint32_t kFwdBufCols = 96;

// Ring position of item `it` (slot, phase parity); a division by a constant.
__device__ __forceinline__ int slot3(int it) { return it % kRing; }
__device__ __forceinline__ uint32_t par3(int it) { return (uint32_t)(it / kRing) & 1u; }

struct UnitConst {  // per flag slot, written by the mask warp
  int tn;
  float s;
  double coef;
};

// ---- tcgen05 / TMA-store PTX ------------------------------------------------

// One lane of a converged warp (the MMA issuer runs the whole warp through
// its loop so that descriptors stay in uniform registers and no per-MMA
// uniformity loop is generated around a diverged single-lane issue).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .pred P1;\nelect.sync _|P1, 0xffffffff;\nselp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ uint32_t idesc_tf32(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// Shared-memory matrix descriptor (sm_100 version bits).  layout 2 =
// SWIZZLE_128B (16-byte granules, K-major operands); layout 1 =
// SWIZZLE_128B_BASE32B (32-byte granules) — the only MN-major layout tf32
// accepts (measured: scripts/dev/mma_probe3.cu).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                          uint32_t layout = 2) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&r)[32]) {
  uint32_t* u = reinterpret_cast<uint32_t*>(r);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
        "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
        "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
        "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(taddr));
}
// A operand rows into TMEM: lane = this thread's row, 32 consecutive columns.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&r)[32]) {
  const uint32_t* u = reinterpret_cast<const uint32_t*>(r);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]),
      "r"(u[8]), "r"(u[9]), "r"(u[10]), "r"(u[11]), "r"(u[12]), "r"(u[13]), "r"(u[14]),
      "r"(u[15]), "r"(u[16]), "r"(u[17]), "r"(u[18]), "r"(u[19]), "r"(u[20]), "r"(u[21]),
      "r"(u[22]), "r"(u[23]), "r"(u[24]), "r"(u[25]), "r"(u[26]), "r"(u[27]), "r"(u[28]),
      "r"(u[29]), "r"(u[30]), "r"(u[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// D (TMEM) += A (TMEM, K-major: lane = row, column = k) * B (smem descriptor).
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b,
                                            uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0,
                                             int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// L2 prefetch of one TMA box (no shared memory, no barrier): deepens the load
// pipeline beyond the 3-slot ring, whose slots stay busy from the load to the
// store of their chunk.
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2,
                                                int c3) {
  asm volatile(
      "cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// L2 prefetch of a contiguous global range (bytes: a multiple of 16).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(src)),
               "r"(bytes)
               : "memory");
}
// A/B switches of the start-up and ring-release schedule (profiles/)
#ifndef COTTEN_ISSUED_GATE
#define COTTEN_ISSUED_GATE 0  // measured: ML-20M bwd 0.757 -> 0.735 with it (profiles/r02s_start)
#endif
#ifndef COTTEN_WARM_L2
#define COTTEN_WARM_L2 1
#endif
#ifndef COTTEN_EARLY_RAW_RELEASE
#define COTTEN_EARLY_RAW_RELEASE 1
#endif
// Per-line L2 prefetch of a global range (any alignment).
__device__ __forceinline__ void prefetch_l2_lines(const void* src, int64_t bytes) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(127);
  const uintptr_t a1 = reinterpret_cast<uintptr_t>(src) + bytes;
  for (uintptr_t a = a0; a < a1; a += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}
// The chunk item `it` of this CTA's persistent schedule (units blockIdx.x +
// j gridDim.x, each P passes x C chunks): false past the last unit.
struct ItemPos {
  int b, h, ps, c;
};
__device__ __forceinline__ bool item_pos(int it, int P, int C, int units, int H, ItemPos& o) {
  const int per = P * C;
  const int j = it / per, rem = it - j * per;
  const int u = blockIdx.x + j * gridDim.x;
  if (u >= units) return false;
  o.b = u / H;
  o.h = u - o.b * H;
  o.ps = rem / C;
  o.c = rem - o.ps * C;
  return true;
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// End of a store warp: every store was already followed by bulk_wait_read0
// (its shared-memory source is read); the full wait for the global writes is
// kept (COTTEN_TAIL_FULL_WAIT=0 — exiting without it, as CUTLASS's TMA
// epilogues do — measured neutral at ML-1M / ML-20M, profiles/r02r_tail).
#ifndef COTTEN_TAIL_FULL_WAIT
#define COTTEN_TAIL_FULL_WAIT 1
#endif
__device__ __forceinline__ void store_tail() {
  if (COTTEN_TAIL_FULL_WAIT) bulk_wait0();
}

// ---- row access in a 128B-swizzled 128-row tile -----------------------------

__device__ __forceinline__ uint32_t chunk_off(int row, int j) {
  return (uint32_t)row * 128u + ((uint32_t)(j ^ (row & 7)) << 4);
}
__device__ __forceinline__ void load_row(const uint8_t* tile, int row, float (&x)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 v = *reinterpret_cast<const float4*>(tile + chunk_off(row, j));
    x[4 * j] = v.x;
    x[4 * j + 1] = v.y;
    x[4 * j + 2] = v.z;
    x[4 * j + 3] = v.w;
  }
}
__device__ __forceinline__ void store_row(uint8_t* tile, int row, const float (&x)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<float4*>(tile + chunk_off(row, j)) =
        make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
}
// Same for the 32-byte-granule swizzle (TMA SWIZZLE_128B_ATOM_32B): 32-byte
// granule g of row r sits at granule g ^ (r & 3).
__device__ __forceinline__ uint32_t chunk_off32(int row, int j) {
  return (uint32_t)row * 128u + ((uint32_t)((j >> 1) ^ (row & 3)) << 5) + ((uint32_t)(j & 1) << 4);
}
// Rows r, r+1, .. of a warp hit only 4 distinct 16-byte bank groups if every
// lane walks its granules in the same order; lanes with bit 2 of the row set
// take the two halves of each 32-byte granule in swapped order, so each
// LDS/STS.128 of the warp spans all 8 bank groups (4 wavefronts, the minimum).
__device__ __forceinline__ void load_row32(const uint8_t* tile, int row, float (&x)[32]) {
  const uint32_t sw = (uint32_t)((row >> 2) & 1) << 4;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint8_t* g = tile + (uint32_t)row * 128u + ((uint32_t)(q ^ (row & 3)) << 5);
    const float4 a = *reinterpret_cast<const float4*>(g + sw);
    const float4 b = *reinterpret_cast<const float4*>(g + (sw ^ 16u));
    const bool s = sw != 0;
    x[8 * q + 0] = s ? b.x : a.x;
    x[8 * q + 1] = s ? b.y : a.y;
    x[8 * q + 2] = s ? b.z : a.z;
    x[8 * q + 3] = s ? b.w : a.w;
    x[8 * q + 4] = s ? a.x : b.x;
    x[8 * q + 5] = s ? a.y : b.y;
    x[8 * q + 6] = s ? a.z : b.z;
    x[8 * q + 7] = s ? a.w : b.w;
  }
}
__device__ __forceinline__ void store_row32(uint8_t* tile, int row, const float (&x)[32]) {
  const uint32_t sw = (uint32_t)((row >> 2) & 1) << 4;
  const bool s = sw != 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint8_t* g = tile + (uint32_t)row * 128u + ((uint32_t)(q ^ (row & 3)) << 5);
    const float4 lo4 = make_float4(x[8 * q], x[8 * q + 1], x[8 * q + 2], x[8 * q + 3]);
    const float4 hi4 = make_float4(x[8 * q + 4], x[8 * q + 5], x[8 * q + 6], x[8 * q + 7]);
    *reinterpret_cast<float4*>(g + sw) = s ? hi4 : lo4;
    *reinterpret_cast<float4*>(g + (sw ^ 16u)) = s ? lo4 : hi4;
  }
}
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
#ifndef COTTEN_TC_ROUND_LO
#define COTTEN_TC_ROUND_LO 0
#endif
__device__ __forceinline__ float tf32_lo(float x, float hi) {
#if COTTEN_TC_ROUND_LO
  return tf32_hi(x - hi);
#else
  return x - hi;
#endif
}
// hi in place of the TMA tile, lo into the lo buffer.
__device__ __forceinline__ void store_split(uint8_t* hi_tile, uint8_t* lo_tile, int row,
                                            const float (&x)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      h[e] = tf32_hi(x[4 * j + e]);
      l[e] = tf32_lo(x[4 * j + e], h[e]);
    }
    *reinterpret_cast<float4*>(hi_tile + chunk_off(row, j)) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(lo_tile + chunk_off(row, j)) = make_float4(l[0], l[1], l[2], l[3]);
  }
}
__device__ __forceinline__ void store_split32(uint8_t* hi_tile, uint8_t* lo_tile, int row,
                                              const float (&x)[32]) {
  float h[32], l[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    h[k] = tf32_hi(x[k]);
    l[k] = tf32_lo(x[k], h[k]);
  }
  store_row32(hi_tile, row, h);
  store_row32(lo_tile, row, l);
}
// ---- packed fp32x2 row arithmetic (FFMA2 / FMUL2: half the FP instructions) ----
__device__ __forceinline__ float2 f2p(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float sumsq(const float (&x)[32]) {
  float2 a0 = f2p(0.f, 0.f), a1 = f2p(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    a0 = __ffma2_rn(f2p(x[k], x[k + 1]), f2p(x[k], x[k + 1]), a0);
    a1 = __ffma2_rn(f2p(x[k + 2], x[k + 3]), f2p(x[k + 2], x[k + 3]), a1);
  }
  return (a0.x + a1.x) + (a0.y + a1.y);
}
__device__ __forceinline__ float dot32(const float (&x)[32], const float (&y)[32]) {
  float2 a0 = f2p(0.f, 0.f), a1 = f2p(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    a0 = __ffma2_rn(f2p(x[k], x[k + 1]), f2p(y[k], y[k + 1]), a0);
    a1 = __ffma2_rn(f2p(x[k + 2], x[k + 3]), f2p(y[k + 2], y[k + 3]), a1);
  }
  return (a0.x + a1.x) + (a0.y + a1.y);
}
__device__ __forceinline__ void scale32(float (&x)[32], float s) {
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    const float2 v = __fmul2_rn(f2p(x[k], x[k + 1]), f2p(s, s));
    x[k] = v.x;
    x[k + 1] = v.y;
  }
}
// g <- (g - pr x) * inv   (the cosine-normalisation Jacobian, attention.cpp:421-437)
__device__ __forceinline__ void jacobian32(float (&g)[32], const float (&x)[32], float pr,
                                           float inv) {
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    const float2 v =
        __fmul2_rn(__ffma2_rn(f2p(x[k], x[k + 1]), f2p(-pr, -pr), f2p(g[k], g[k + 1])), f2p(inv, inv));
    g[k] = v.x;
    g[k + 1] = v.y;
  }
}
// Zero a row unless f (bit mask, NaN-safe: padded rows are never multiplied).
__device__ __forceinline__ void keep_if(float (&x)[32], bool f) {
  const uint32_t m = f ? 0xFFFFFFFFu : 0u;
#pragma unroll
  for (int k = 0; k < 32; ++k) x[k] = __uint_as_float(__float_as_uint(x[k]) & m);
}
// 3xTF32 split of a row: h = x with the low 13 mantissa bits cleared (exact
// in tf32), l = x - h (exact in fp32; |l| < 2^-10 |x|, the tensor core's own
// truncation of l costs < 2^-20 |x|).  Optionally NaN-safe masked to zero.
__device__ __forceinline__ void split32(const float (&x)[32], float (&h)[32], float (&l)[32],
                                        uint32_t mask = 0xFFFFFFFFu) {
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    const float h0 = __uint_as_float(__float_as_uint(x[k]) & (0xFFFFE000u & mask));
    const float h1 = __uint_as_float(__float_as_uint(x[k + 1]) & (0xFFFFE000u & mask));
    const float2 lv = __ffma2_rn(f2p(h0, h1), f2p(-1.f, -1.f), f2p(x[k], x[k + 1]));
    h[k] = h0;
    h[k + 1] = h1;
    l[k] = __uint_as_float(__float_as_uint(lv.x) & mask);
    l[k + 1] = __uint_as_float(__float_as_uint(lv.y) & mask);
  }
}
// lo = x - trunc_tf32(x) only: tcgen05 kind::tf32 truncates fp32 operands
// (measured, scripts/dev/tf32_round.cu), so an untouched fp32 tile already is
// its own hi part and only lo has to be written.
__device__ __forceinline__ void lo32(const float (&x)[32], float (&l)[32]) {
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    const float h0 = __uint_as_float(__float_as_uint(x[k]) & 0xFFFFE000u);
    const float h1 = __uint_as_float(__float_as_uint(x[k + 1]) & 0xFFFFE000u);
    const float2 lv = __ffma2_rn(f2p(h0, h1), f2p(-1.f, -1.f), f2p(x[k], x[k + 1]));
    l[k] = lv.x;
    l[k + 1] = lv.y;
  }
}
// Rows of a 32-byte-granule tile in "lane order": x[8q..8q+3] is the half of
// granule q the lane touches first (see load_row32), x[8q+4..8q+7] the other.
// Element-wise work (norms, scaling, hi/lo split) does not care about the order,
// so tiles that are only re-stored in the same layout skip the unswizzle selects.
__device__ __forceinline__ void load_row32_raw(const uint8_t* tile, int row, float (&x)[32]) {
  const uint32_t sw = (uint32_t)((row >> 2) & 1) << 4;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint8_t* g = tile + (uint32_t)row * 128u + ((uint32_t)(q ^ (row & 3)) << 5);
    const float4 a = *reinterpret_cast<const float4*>(g + sw);
    const float4 b = *reinterpret_cast<const float4*>(g + (sw ^ 16u));
    x[8 * q + 0] = a.x; x[8 * q + 1] = a.y; x[8 * q + 2] = a.z; x[8 * q + 3] = a.w;
    x[8 * q + 4] = b.x; x[8 * q + 5] = b.y; x[8 * q + 6] = b.z; x[8 * q + 7] = b.w;
  }
}
__device__ __forceinline__ void store_row32_raw(uint8_t* tile, int row, const float (&x)[32]) {
  const uint32_t sw = (uint32_t)((row >> 2) & 1) << 4;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint8_t* g = tile + (uint32_t)row * 128u + ((uint32_t)(q ^ (row & 3)) << 5);
    *reinterpret_cast<float4*>(g + sw) = make_float4(x[8 * q], x[8 * q + 1], x[8 * q + 2], x[8 * q + 3]);
    *reinterpret_cast<float4*>(g + (sw ^ 16u)) =
        make_float4(x[8 * q + 4], x[8 * q + 5], x[8 * q + 6], x[8 * q + 7]);
  }
}
// lane order -> natural column order (and back: the map is an involution)
__device__ __forceinline__ void unswap32(float (&x)[32], int row) {
  const bool s = (row >> 2) & 1;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float a = x[8 * q + e], b = x[8 * q + 4 + e];
      x[8 * q + e] = s ? b : a;
      x[8 * q + 4 + e] = s ? a : b;
    }
}
// Element (n, k) of a 32-row operand buffer (row n, column k).
__device__ __forceinline__ uint32_t elem_off(int n, int k) {
  return chunk_off(n, k >> 2) + (uint32_t)(k & 3) * 4u;
}

__device__ __forceinline__ bool flag_at(const uint32_t* fl, int r) {
  return (fl[r >> 5] >> (r & 31)) & 1u;
}

// ---- the mask warp ------------------------------------------------------------

// s = exp(-m ln n) and coef = -ln(n) s in fp64 (attention.cpp:304, :403, :408);
// out of line: one call per unit, keeps the fp64 libm expansion out of the
// instruction-cache working set of the hot loops.
__device__ __noinline__ void unit_scale(double m, int n, float* s_out, double* coef_out) {
  const double ln = log((double)n);
  const float s = (float)exp(-m * ln);
  *s_out = s;
  *coef_out = -ln * (double)s;
}

// Bitmask of valid rows + true_n + the fp64 scale constants of unit (b).
// `issued` (first unit only): arrived on once this warp's first valid-byte
// loads are issued, before their values are used — the producer holds its
// first TMA loads for it (see Bars::issued).
__device__ __forceinline__ void mask_unit(const OpParams& p, int64_t b, uint32_t* fl,
                                          UnitConst* uc, int lane, uint64_t* issued = nullptr) {
  const int N = (int)p.N;
  const int words = (N + 31) >> 5;
  int cnt = 0;
  const uint8_t* row = p.valid ? p.valid + b * p.msb : nullptr;
  for (int w0 = 0; w0 < words; w0 += 8) {
    uint8_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // 8 loads in flight before the first ballot
      const int r = (w0 + k) * 32 + lane;
      v[k] = (w0 + k < words && r < N) ? (row ? __ldg(row + r) : (uint8_t)1) : (uint8_t)0;
    }
    if (issued) {
      __syncwarp();
      if (lane == 0) mbar_arrive(issued);
      issued = nullptr;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t bits = __ballot_sync(0xffffffffu, v[k] != 0);
      if (w0 + k < words) {
        if (lane == 0) fl[w0 + k] = bits;
        cnt += __popc(bits);
      }
    }
  }
  if (lane == 0) {
    UnitConst c;
    c.tn = cnt;
    if (cnt > 0) {
      unit_scale(op_m(p), cnt, &c.s, &c.coef);
    } else {  // UsageError in the reference (attention.cpp:44): NaN outputs + status bit
      c.s = __int_as_float(0x7fc00000);
      c.coef = __longlong_as_double(0x7ff8000000000000ll);
      if (p.status) atomicOr(p.status, 1);
    }
    *uc = c;
  }
}

// ---- MMA issue helpers (one thread) ----------------------------------------------

// Reduction R += x^T y over the valid 8-row groups of a chunk (tiles in the
// 32-byte-granule swizzle): x's hi tile at xh, lo at xh + lbo; y's hi at yh,
// lo at yh + lbo.  D (M=64 x N=64) rows 0-31 are x_hi, 32-63 x_lo; columns
// 0-31 y_hi, 32-63 y_lo.  SBO = 512: 4-row groups of the 32B-granule atom.
__device__ __forceinline__ void issue_reduction(uint32_t d, uint32_t xh, uint32_t yh,
                                                uint32_t lbo, int ksteps, bool first) {
  const uint32_t id = idesc_tf32(64, 64, true, true);
  for (int kk = 0; kk < ksteps; ++kk)
    mma_tf32(d, sdesc(xh + 1024u * kk, lbo, 512u, 1u), sdesc(yh + 1024u * kk, lbo, 512u, 1u), id,
             (first && kk == 0) ? 0u : 1u);
}
// Row output D = A B with A = this chunk's 128 rows in TMEM (K-major: lane =
// row, hi at columns [ah, ah+32), lo at [ah+32, ah+64)) and B = a 32-row
// state operand in shared memory (hi at bh, lo at bl): 3xTF32 = 12 MMAs of
// M=128, N=32, K=8.  A from TMEM keeps these small-N MMAs off the shared-
// memory port (an SS MMA would re-read its 4 KB A tile for every 16-cycle
// instruction).
template <bool kBMN>
__device__ __forceinline__ void issue_rowout_ts(uint32_t d, uint32_t ah, uint32_t bh, uint32_t bl) {
  // B K-major (row n holds B[.][n], 16-byte granules): k-step = 32 bytes along the row;
  // B MN-major (row k holds B[k][.], 32-byte granules): k-step = 8 rows = 1 KB.
  const uint32_t id = idesc_tf32(128, 32, false, kBMN);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint64_t dh = kBMN ? sdesc(bh + 1024u * kk, 4096u, 512u, 1u) : sdesc(bh + 32u * kk, 16u, 1024u);
    const uint64_t dl = kBMN ? sdesc(bl + 1024u * kk, 4096u, 512u, 1u) : sdesc(bl + 32u * kk, 16u, 1024u);
    mma_tf32_ts(d, ah + 8 * kk, dh, id, kk > 0 ? 1u : 0u);
    mma_tf32_ts(d, ah + 8 * kk, dl, id, 1u);
    mma_tf32_ts(d, ah + 32 + 8 * kk, dh, id, 1u);
  }
}
// Same with A = a 128-row chunk in shared memory (K-major, 16-byte granules).
template <bool kBMN>
__device__ __forceinline__ void issue_rowout_ss(uint32_t d, uint32_t ah, uint32_t al, uint32_t bh,
                                                uint32_t bl) {
  const uint32_t id = idesc_tf32(128, 32, false, kBMN);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint64_t dh = kBMN ? sdesc(bh + 1024u * kk, 4096u, 512u, 1u) : sdesc(bh + 32u * kk, 16u, 1024u);
    const uint64_t dl = kBMN ? sdesc(bl + 1024u * kk, 4096u, 512u, 1u) : sdesc(bl + 32u * kk, 16u, 1024u);
    const uint64_t a_h = sdesc(ah + 32u * kk, 16u, 1024u), a_l = sdesc(al + 32u * kk, 16u, 1024u);
    mma_tf32(d, a_h, dh, id, kk > 0 ? 1u : 0u);
    mma_tf32(d, a_h, dl, id, 1u);
    mma_tf32(d, a_l, dh, id, 1u);
  }
}
__device__ __forceinline__ void tmem_ld_row(uint32_t taddr, float (&r)[32]) {
  tmem_ld32(taddr, r);
  tmem_wait_ld();
}
// Split a row into hi / lo and store both as TMEM A-operand columns of this
// thread's lane: hi at [col, col+32), lo at [col+32, col+64).
__device__ __forceinline__ void tmem_store_split(uint32_t taddr, const float (&x)[32],
                                                 uint32_t mask = 0xFFFFFFFFu) {
  float h[32], l[32];
  split32(x, h, l, mask);
  tmem_st32(taddr, h);
  tmem_st32(taddr + 32, l);
}

// ---- optional phase trace (debug builds: -DCOTTEN_TC_TRACE=1) ---------------------
// Per item (first kTraceItems of each CTA), clock64() stamps: splitter thread 0
// (slot 0): [0] before its waits, [1] stage landed and lo buffer free, [2] split
// published; epiloguer thread 0 (slot 1): [3] MMAs done, [5] outputs staged,
// [4] staged barrier arrived; MMA lane 0 (slot 2): [0] before its split wait,
// [1] after it, [2] after issuing.  Layout [cta][3][item][8].
#ifndef COTTEN_TC_TRACE
#define COTTEN_TC_TRACE 0
#endif
constexpr int kTraceItems = 64;
#if COTTEN_TC_TRACE
#define TC_TRACE(k)                                                                       \
  do {                                                                                    \
    if (t == 0 && p.workspace && it < kTraceItems)                                       \
      static_cast<long long*>(p.workspace)[((blockIdx.x * 3 + g) * kTraceItems + it) * 8 + (k)] = \
          clock64();                                                                      \
  } while (0)
#define TC_TRACE_MMA(k)                                                                   \
  do {                                                                                    \
    if (lane == 0 && p.workspace && it < kTraceItems)                                     \
      static_cast<long long*>(p.workspace)[((blockIdx.x * 3 + 2) * kTraceItems + it) * 8 + (k)] = \
          clock64();                                                                      \
  } while (0)
// CTA timeline in globaltimer ns (comparable across SMs): slot [cta][2][kTraceItems-1][k],
// k = 4 kernel entry, 5 setup done, 6 last item finished (epiloguer), 7 CTA exit.
#define TC_TRACE_CTA(k)                                                                   \
  do {                                                                                    \
    if (p.workspace) {                                                                    \
      unsigned long long gt_;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                              \
      static_cast<long long*>(p.workspace)[((blockIdx.x * 3 + 2) * kTraceItems + kTraceItems - 1) * 8 + (k)] = \
          (long long)gt_;                                                                 \
    }                                                                                     \
  } while (0)
// Start-up stamps (globaltimer ns) at [cta][2][kTraceItems-2][k]: 0 mask warp after
// its first loads are issued, 1 its flags published (fl_full), 2 producer's first TMA
// issued, 3 splitter passed fl_full, 4 splitter saw item 0 land.
#define TC_TRACE_T0(k)                                                                    \
  do {                                                                                    \
    if (p.workspace) {                                                                    \
      unsigned long long gt_;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                              \
      static_cast<long long*>(p.workspace)[((blockIdx.x * 3 + 2) * kTraceItems + kTraceItems - 2) * 8 + (k)] = \
          (long long)gt_;                                                                 \
    }                                                                                     \
  } while (0)
#else
#define TC_TRACE_T0(k) \
  do {                 \
  } while (0)
#define TC_TRACE_CTA(k) \
  do {                  \
  } while (0)
#define TC_TRACE(k) \
  do {              \
  } while (0)
#define TC_TRACE_MMA(k) \
  do {                  \
  } while (0)
#endif

// ---- warp roles, barriers -------------------------------------------------------

struct Bars {
  // ring slot = item % 3 for the TMA stage, the lo buffer and the TMEM buffer alike
  uint64_t raw_full[kRing], raw_empty[kRing];  // producer <-> splitter / MMA
  uint64_t split_full[kRing], mma_done[kRing];  // splitter -> MMA -> epiloguer
  uint64_t op_ready;                    // state operand (S or dA) written, per unit
  uint64_t acc_free;                    // epiloguer flushed the reduction accumulator
  uint64_t red_done;                    // bwd: a unit's G reduction MMAs complete (per unit)
  uint64_t fl_full[2], fl_empty[2];     // mask warp <-> workers (slot = unit & 1)
  uint64_t staged[kRing], lo_free[kRing];  // epiloguer -> store warp -> splitter
  // The first unit's small dependent loads (valid bytes; bwd: saved S) are
  // issued before the producer's first TMA loads: at a kernel start all 148
  // CTAs request three ring slots at once (~14 MB, ~2 us of HBM), and a mask
  // load queued behind them held the first split ~4 us at ML-1M (trace).
  uint64_t issued;
};
static_assert(sizeof(Bars) <= 256, "barrier area");

__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
}

// Barrier init + TMEM allocation (256 columns, one CTA per SM).
__device__ __forceinline__ uint32_t tc_setup(uint8_t* smem, Bars* br, uint32_t* tslot, int warp,
                                             int issued_count) {
  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023u) __trap();
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&br->raw_full[i], 1);
      mbar_init(&br->raw_empty[i], 1);
      mbar_init(&br->split_full[i], 4);
      mbar_init(&br->mma_done[i], 1);
      mbar_init(&br->staged[i], 4);
      mbar_init(&br->lo_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&br->fl_full[i], 1);
      mbar_init(&br->fl_empty[i], kWorkerWarps);
    }
    mbar_init(&br->op_ready, 1);
    mbar_init(&br->acc_free, 4);
    mbar_init(&br->red_done, 1);
    mbar_init(&br->issued, issued_count);
    d32::fence_barrier_init();
  }
  if (warp == kWarpMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        smem_u32(tslot)), "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  return *tslot;
}
// dm_total = fixed-order sum of dm_unit[0, units): the same partition and
// tree as dm_reduce_kernel (kernels_generic.cuh), run by the last CTA to
// finish, so the value is bit-identical to the separate launch it replaces.
__device__ __forceinline__ void last_cta_dm_total(const OpParams& p, int units, uint8_t* smem_word) {
  volatile unsigned* flag = reinterpret_cast<volatile unsigned*>(smem_word);
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(p.grid_done, 1u);
    *flag = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!*flag) return;
  __threadfence();
  double* red = reinterpret_cast<double*>(smem_word + 8);
  if (threadIdx.x < 256) {
    double part = 0.0;
    const int64_t per = (units + 255) / 256;
    const int64_t lo = threadIdx.x * per, hi = min64(units, lo + per);
    for (int64_t u = lo; u < hi; ++u) part += __ldcg(p.dm_unit + u);  // contiguous, in order
    part = warp_sum(part);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    *p.dm_total = t;
    *p.grid_done = 0u;  // ready for the next launch
  }
}
// Programmatic dependent launch: the setup above (barrier init, TMEM
// allocation) runs while the previous kernel in the stream drains; every role
// waits for that kernel's memory before its first global access.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void tc_teardown(uint32_t tmem, int warp) {
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  }
}

// The mask warp: one unit at a time, up to two units ahead of the workers.
__device__ __forceinline__ void mask_loop(const OpParams& p, uint8_t* smem, Bars* br, int lane) {
  UnitConst* ucs = reinterpret_cast<UnitConst*>(smem + kOffMisc);
  const int units = (int)(p.B * p.H), H = (int)p.H;
  int j = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
    const int sl = j & 1;
    mbar_wait(&br->fl_empty[sl], ((j >> 1) & 1) ^ 1);
    if (lane == 0 && j == 0) TC_TRACE_T0(0);
    mask_unit(p, u / H, reinterpret_cast<uint32_t*>(smem + kOffFlags + sl * (kMaxN / 8)),
              &ucs[sl], lane, j == 0 ? &br->issued : nullptr);
    __syncwarp();
    if (lane == 0) mbar_arrive(&br->fl_full[sl]);
    if (lane == 0 && j == 0) TC_TRACE_T0(1);
  }
}

// ---- reduction epilogue (S or G) --------------------------------------------------
// The M=64 accumulator (row m at lane (m%16) + 32(m/16); rows 0-31 x_hi, 32-63
// x_lo; columns 0-31 y_hi, 32-63 y_lo) is folded into R = sum of the four
// products, spread over the whole group: thread t gets row a = t/4, columns
// [8(t%4), 8(t%4)+8).  scratch: 8 KB of free smem (two 32-row partial tiles).
__device__ __forceinline__ void reduce_rows8(uint32_t tmem, uint8_t* scratch, int wq, int lane,
                                             int g, int t, float (&r8)[8],
                                             const uint8_t* run = nullptr) {
  float a[32], c[32];
  const uint32_t ta = tmem + ((uint32_t)(32 * wq) << 16);
  tmem_ld32(ta, a);
  tmem_ld32(ta + 32, c);
  tmem_wait_ld();
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 32; ++k) a[k] += c[k];  // x.. y_hi + x.. y_lo
    store_row(scratch + (wq >> 1) * 4096, 16 * (wq & 1) + lane, a);
  }
  group_sync(g);
  const int ra = t >> 2, q = t & 3;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float4 u = *reinterpret_cast<const float4*>(scratch + chunk_off(ra, 2 * q + h));
    const float4 v = *reinterpret_cast<const float4*>(scratch + 4096 + chunk_off(ra, 2 * q + h));
    r8[4 * h + 0] = u.x + v.x;
    r8[4 * h + 1] = u.y + v.y;
    r8[4 * h + 2] = u.z + v.z;
    r8[4 * h + 3] = u.w + v.w;
    if (run) {  // + the flushed partial sums of earlier chunks (same tile layout)
      const float4 x = *reinterpret_cast<const float4*>(run + chunk_off(ra, 2 * q + h));
      const float4 y = *reinterpret_cast<const float4*>(run + 4096 + chunk_off(ra, 2 * q + h));
      r8[4 * h + 0] += x.x + y.x;
      r8[4 * h + 1] += x.y + y.y;
      r8[4 * h + 2] += x.z + y.z;
      r8[4 * h + 3] += x.w + y.w;
    }
  }
  if (run) group_sync(g);  // the running sum is read before its area is reused
}
// Flush the reduction accumulator into the running sum (two 32-row tiles:
// x_hi rows, x_lo rows; each lane < 16 owns one row, so no synchronisation).
__device__ __forceinline__ void flush_acc(uint32_t tmem, uint8_t* run, int wq, int lane,
                                          bool first) {
  float a[32], c[32];
  const uint32_t ta = tmem + ((uint32_t)(32 * wq) << 16);
  tmem_ld32(ta, a);
  tmem_ld32(ta + 32, c);
  tmem_wait_ld();
  if (lane < 16) {
    uint8_t* tile = run + (wq >> 1) * 4096;
    const int row = 16 * (wq & 1) + lane;
#pragma unroll
    for (int k = 0; k < 32; ++k) a[k] += c[k];
    if (!first) {
      load_row(tile, row, c);
#pragma unroll
      for (int k = 0; k < 32; ++k) a[k] += c[k];
    }
    store_row(tile, row, a);
  }
}
// 8 columns [8q, 8q+8) of row a as hi / lo into a K-major (16-byte granule)
// and / or an MN-major (32-byte granule) state operand.
__device__ __forceinline__ void split8(const float (&x)[8], float (&h)[8], float (&l)[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    h[k] = tf32_hi(x[k]);
    l[k] = tf32_lo(x[k], h[k]);
  }
}
__device__ __forceinline__ void store8_k(uint8_t* op, int a, int q, const float (&x)[8]) {
  *reinterpret_cast<float4*>(op + chunk_off(a, 2 * q)) = make_float4(x[0], x[1], x[2], x[3]);
  *reinterpret_cast<float4*>(op + chunk_off(a, 2 * q + 1)) = make_float4(x[4], x[5], x[6], x[7]);
}
__device__ __forceinline__ void store8_mn(uint8_t* op, int a, int q, const float (&x)[8]) {
  uint8_t* gp = op + (uint32_t)a * 128u + ((uint32_t)(q ^ (a & 3)) << 5);
  *reinterpret_cast<float4*>(gp) = make_float4(x[0], x[1], x[2], x[3]);
  *reinterpret_cast<float4*>(gp + 16) = make_float4(x[4], x[5], x[6], x[7]);
}

// hi / lo split of a row into two register arrays.
__device__ __forceinline__ void split_regs(const float (&x)[32], float (&h)[32], float (&l)[32]) {
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    h[k] = tf32_hi(x[k]);
    l[k] = tf32_lo(x[k], h[k]);
  }
}

// Arrive on the group's "staged" barrier (one arrival per warp): the chunk's
// outputs are in its raw stage (or it has none) and the MMAs that read the
// stage are complete, so the store warp may store it and recycle the stage.
__device__ __forceinline__ void arrive_staged(Bars* br, int b, int lane) {
  fence_proxy_async();
  __syncwarp();
  if (lane == 0) mbar_arrive(&br->staged[b]);
}
// single-column TMEM store / load (a per-row scalar handed from splitter to epiloguer)
__device__ __forceinline__ void tmem_st1(uint32_t taddr, float v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr),
               "r"(__float_as_uint(v))
               : "memory");
}
__device__ __forceinline__ float tmem_ld1(uint32_t taddr) {
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
  return __uint_as_float(v);
}

// ======================================================================================
// Forward
// ======================================================================================
__global__ void __launch_bounds__(kThreads, 1) cos_fwd_tc_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap to,
    const OpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = (int)p.N, H = (int)p.H;
  const int units = (int)(p.B * p.H);
  const int C = (N + kRows - 1) / kRows;
  // pass 2 (Q) only when O or the Q norms are wanted (an S-only forward
  // feeds a backward that was given no saved state)
  const int P = (p.out != nullptr || p.saved_norms != nullptr) ? 2 : 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Bars* br = reinterpret_cast<Bars*>(smem + kOffBar);
  UnitConst* ucs = reinterpret_cast<UnitConst*>(smem + kOffMisc);
  uint8_t* ops = smem + kOffOps;
  if (threadIdx.x == 0) TC_TRACE_CTA(4);
  const uint32_t tmem =
      tc_setup(smem, br, reinterpret_cast<uint32_t*>(smem + kOffMisc + 32), warp, 1);
  // Before the dependency resolves: warm L2 with this CTA's first three items and its
  // first two units' valid bytes.  A prefetch is only a hint (if the preceding kernel
  // still writes these lines, the loads after pdl_wait read its data from L2); it
  // overlaps the first HBM round trip (~2 us at a cold start, trace) with that
  // kernel's tail.
  if (COTTEN_WARM_L2 && warp == kWarpProducer && lane == 0) {
    for (int it = 0; it < kRing; ++it) {
      ItemPos f;
      if (!item_pos(it, P, C, units, H, f)) break;
      if (f.ps == 0) {
        tma_prefetch_4d(&tk, 0, f.c * kRows, f.h, f.b);
        tma_prefetch_4d(&tv, 0, f.c * kRows, f.h, f.b);
      } else {
        tma_prefetch_4d(&tq, 0, f.c * kRows, f.h, f.b);
      }
    }
    for (int u = blockIdx.x; p.valid && u < units && u < (int)blockIdx.x + 2 * (int)gridDim.x; u += gridDim.x)
      prefetch_l2_lines(p.valid + (int64_t)(u / H) * p.msb, N);
  }
  pdl_wait();
  const KernelStamp stamp_(p);
  pdl_launch_dependents();
  if (threadIdx.x == 0) TC_TRACE_CTA(5);

  if (warp == kWarpProducer) {  // ===== TMA: (K, V) chunks then Q chunks =====
    if (lane == 0) {
      d32::prefetch_map(&tk);
      d32::prefetch_map(&tv);
      d32::prefetch_map(&tq);
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        for (int ps = 0; ps < P; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot3(it);
            if (COTTEN_ISSUED_GATE && it == 0) mbar_wait(&br->issued, 0);  // mask loads go first
            ItemPos f;
            if (p.l2_ahead && item_pos(it + p.l2_ahead, P, C, units, H, f)) {
              if (f.ps == 0) {
                tma_prefetch_4d(&tk, 0, f.c * kRows, f.h, f.b);
                tma_prefetch_4d(&tv, 0, f.c * kRows, f.h, f.b);
              } else {
                tma_prefetch_4d(&tq, 0, f.c * kRows, f.h, f.b);
              }
            }
            mbar_wait(&br->raw_empty[st], par3(it) ^ 1u);
            uint8_t* dst = smem + kOffRaw + st * kStage;
            if (ps == 0) {
              mbar_expect_tx(&br->raw_full[st], 2 * kTile);
              tma_load_4d(dst, &tk, 0, c * kRows, h, b, &br->raw_full[st]);
              tma_load_4d(dst + kTile, &tv, 0, c * kRows, h, b, &br->raw_full[st]);
              if (it == 0) TC_TRACE_T0(2);
            } else {
              mbar_expect_tx(&br->raw_full[st], kTile);
              tma_load_4d(dst, &tq, 0, c * kRows, h, b, &br->raw_full[st]);
            }
          }
      }
    }
  } else if (warp == kWarpMma) {  // ===== MMA issuer (whole warp, one elected lane issues) =====
    int it = 0, j = 0, nflush = 0;
    const uint32_t base = smem_u32(smem);
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      for (int ps = 0; ps < P; ++ps)
        for (int c = 0; c < C; ++c, ++it) {
          const int st = slot3(it), bf = st;
          TC_TRACE_MMA(0);
          mbar_wait(&br->split_full[bf], par3(it));
          if (ps == 0 && c == 0 && P == 1 && j > 0)  // previous S read before it is overwritten
            mbar_wait(&br->op_ready, (j - 1) & 1);
          if (ps == 0 && c > 0 && c % kFlush == 0) mbar_wait(&br->acc_free, (nflush++) & 1);
          if (ps == 1 && c == 0) mbar_wait(&br->op_ready, j & 1);
          tc_fence_after();
          TC_TRACE_MMA(1);
          const uint32_t X = base + kOffRaw + st * kStage;
          const uint32_t Y = base + kOffLo + bf * kStage;
          if (elect_one()) {
            if (ps == 0) {  // S += K~^T V (attention.cpp:345-353)
              const int rows = min(kRows, N - c * kRows);
              issue_reduction(tmem, X, X + kTile, Y - X, (rows + 7) >> 3, c % kFlush == 0);
            } else {  // O = Q~ S (attention.cpp:379-387), B = S rows (MN-major)
              const uint32_t D = tmem + kFwdBuf0 + kFwdBufCols * bf;
              issue_rowout_ts<true>(D, D + 32, base + kOffOps, base + kOffOps + kOpBytes);
            }
            TC_TRACE_MMA(2);
            // pass 2 reads Q~ from TMEM only: the splitter released its raw stage
            if (ps == 0 || !COTTEN_EARLY_RAW_RELEASE) mma_commit(&br->raw_empty[st]);
            mma_commit(&br->mma_done[bf]);
          }
          __syncwarp();
        }
    }
  } else if (warp == kWarpMask) {
    mask_loop(p, smem, br, lane);
  } else if (warp == kWarpStore) {  // ===== TMA stores of staged outputs; lo-buffer recycling =====
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        for (int ps = 0; ps < P; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int bf = slot3(it);
            mbar_wait(&br->staged[bf], par3(it));
            if (ps == 1 && p.out) {
              tma_store_4d(&to, smem + kOffLo + bf * kStage, 0, c * kRows, h, b);
              bulk_wait_read0();
            }
            mbar_arrive(&br->lo_free[bf]);
          }
      }
      store_tail();
    }
  } else {
    // ===== workers: group 0 splits every chunk, group 1 runs every epilogue;
    //       thread t owns row t of the chunk (= TMEM lane t) in both =====
    const int g = warp >> 2, wq = warp & 3, t = threadIdx.x & 127;
    const float eps = (float)p.eps;
    float* norms_all = static_cast<float*>(p.saved_norms);
    float* gS_all = static_cast<float*>(p.saved_S);
    const uint32_t lane_base = (uint32_t)(32 * wq) << 16;
    int it = 0, j = 0, n_tr = 0;
    (void)n_tr;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int sl = j & 1;
      const uint32_t* fl = reinterpret_cast<const uint32_t*>(smem + kOffFlags + sl * (kMaxN / 8));
      float* norms = norms_all ? norms_all + (int64_t)u * 2 * N : nullptr;
      mbar_wait(&br->fl_full[sl], (j >> 1) & 1);
      const UnitConst uc = ucs[sl];
      for (int k = 0; k < P * C; ++k, ++it) {  // the unit's chunks: pass 1, then pass 2
          const int ps = k >= C, c = ps ? k - C : k;
          const int st = slot3(it), bf = st;
          const int r = c * kRows + t;
          uint8_t* X = smem + kOffRaw + st * kStage;
          uint8_t* Y = smem + kOffLo + bf * kStage;
          const uint32_t D = tmem + kFwdBuf0 + kFwdBufCols * bf + lane_base;
          if (g == 0) {  // ---------------- splitter ----------------
            TC_TRACE(0);
            if (it == 0 && t == 0) TC_TRACE_T0(3);
            mbar_wait(&br->raw_full[st], par3(it));
            mbar_wait(&br->lo_free[bf], par3(it) ^ 1u);
            TC_TRACE(1);
            if (it == 0 && t == 0) TC_TRACE_T0(4);
            if (ps == 0) {  // K~ (masked, attention.cpp:334-343) and V, 32-byte-granule tiles
              float kx[32], vx[32], hh[32], ll[32];
              load_row32_raw(X, t, kx);  // lane order: only re-stored in the same layout
              load_row32_raw(X + kTile, t, vx);
              const bool f = r < N && flag_at(fl, r);
              const float ss = sumsq(kx) + eps;
              const float iv = rsqrtf(ss);
              scale32(kx, iv);
              if (norms && r < N) norms[N + r] = f ? ss * iv : 1.0f;  // :336, :343
              split32(kx, hh, ll, f ? 0xFFFFFFFFu : 0u);  // padded rows: exact zeros, NaN-safe
              store_row32_raw(X, t, hh);
              store_row32_raw(Y, t, ll);
              lo32(vx, ll);  // V: the TMA tile itself is the hi operand
              store_row32_raw(Y + kTile, t, ll);
            } else {  // Q~ for every row (attention.cpp:366-377), TMEM A operand of O = Q~ S
              float qx[32];
              load_row(X, t, qx);
              const float ss = sumsq(qx) + eps;  // (every loaded value consumed here)
              // the raw Q tile is read only here (the MMA takes Q~ from TMEM): release the
              // stage now, not after the MMA, so the producer's next load starts earlier
              if (COTTEN_EARLY_RAW_RELEASE) {
                fence_proxy_async();
                group_sync(g);
                if (t == 0) mbar_arrive(&br->raw_empty[st]);
              }
              const float iv = rsqrtf(ss);
              scale32(qx, iv);
              if (norms && r < N) norms[r] = ss * iv;
              tmem_store_split(D + 32, qx);
              tmem_wait_st();
              tc_fence_before();
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&br->split_full[bf]);
            TC_TRACE(2);
          } else {  // ---------------- epiloguer ----------------
            mbar_wait(&br->mma_done[bf], par3(it));
            tc_fence_after();
            TC_TRACE(3);
            if (ps == 0) {
              // a pass-1 item stages nothing and its MMAs are done: release the slot
              // before the flush / S-epilogue, which work in TMEM and the operand
              // area only (the splitter may refill the slot meanwhile)
              TC_TRACE(5);
              arrive_staged(br, bf, lane);
              TC_TRACE(4);
              uint8_t* run = ops + 2 * kOpBytes;  // 8 KB the forward does not otherwise use
              uint8_t* scr = ops + 4 * kOpBytes;  // and 8 KB more: the S-epilogue's scratch
              if (c != C - 1 && c % kFlush == kFlush - 1) {  // long N: flush the accumulator
                flush_acc(tmem, run, wq, lane, c == kFlush - 1);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&br->acc_free);
              }
              if (c == C - 1) {  // S complete: saved S + the MN-major B operand of O = Q~ S
                float s8[8], h8[8], l8[8];
                reduce_rows8(tmem, scr, wq, lane, g, t, s8, C > kFlush ? run : nullptr);
                const int a = t >> 2, q = t & 3;
                if (gS_all) {  // coalesced: a warp writes 8 whole rows of S
                  float4* gs = reinterpret_cast<float4*>(gS_all + (int64_t)u * 1024 + a * 32 + 8 * q);
                  gs[0] = make_float4(s8[0], s8[1], s8[2], s8[3]);
                  gs[1] = make_float4(s8[4], s8[5], s8[6], s8[7]);
                }
                split8(s8, h8, l8);
                store8_mn(ops, a, q, h8);
                store8_mn(ops + kOpBytes, a, q, l8);
                fence_proxy_async();
                tc_fence_before();
                group_sync(g);
                if (t == 0) mbar_arrive(&br->op_ready);
              }
            } else {  // O rows = s (Q~ S) (attention.cpp:379-387), staged in the lo buffer
              float acc[32];
              tmem_ld_row(D, acc);
              tc_fence_before();
              scale32(acc, uc.s);
              store_row(Y, t, acc);
              TC_TRACE(5);
              arrive_staged(br, bf, lane);
              TC_TRACE(4);
            }
            ++n_tr;
          }
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&br->fl_empty[sl]);
    }
  }
  if (threadIdx.x == 128) TC_TRACE_CTA(6);  // epiloguer thread 0: its last item is done
  tc_teardown(tmem, warp);
  if (threadIdx.x == 0) TC_TRACE_CTA(7);
}

// ======================================================================================
// Backward
// ======================================================================================
__global__ void __launch_bounds__(kThreads, 1) cos_bwd_tc_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
    const __grid_constant__ CUtensorMap tdq, const __grid_constant__ CUtensorMap tdk,
    const __grid_constant__ CUtensorMap tdv, const OpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = (int)p.N, H = (int)p.H;
  const int units = (int)(p.B * p.H);
  const int C = (N + kRows - 1) / kRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Bars* br = reinterpret_cast<Bars*>(smem + kOffBar);
  UnitConst* ucs = reinterpret_cast<UnitConst*>(smem + kOffMisc);
  double* dm_x = reinterpret_cast<double*>(smem + kOffMisc + 40);
  uint8_t* ops = smem + kOffOps;
  if (threadIdx.x == 0) TC_TRACE_CTA(4);
  const uint32_t tmem =
      tc_setup(smem, br, reinterpret_cast<uint32_t*>(smem + kOffMisc + 32), warp, 1 + 4);
  // Warm L2 before the dependency resolves (see the forward): the first three items,
  // the first two units' valid bytes and the first unit's saved S.
  if (COTTEN_WARM_L2 && warp == kWarpProducer && lane == 0) {
    for (int it = 0; it < kRing; ++it) {
      ItemPos f;
      if (!item_pos(it, 2, C, units, H, f)) break;
      tma_prefetch_4d(f.ps == 0 ? &tq : &tk, 0, f.c * kRows, f.h, f.b);
      tma_prefetch_4d(f.ps == 0 ? &tdo : &tv, 0, f.c * kRows, f.h, f.b);
    }
    for (int u = blockIdx.x; p.valid && u < units && u < (int)blockIdx.x + 2 * (int)gridDim.x; u += gridDim.x)
      prefetch_l2_lines(p.valid + (int64_t)(u / H) * p.msb, N);
    bulk_prefetch_l2(static_cast<const float*>(p.saved_S) + (int64_t)blockIdx.x * 1024, 4096);
  }
  pdl_wait();
  const KernelStamp stamp_(p);
  pdl_launch_dependents();
  if (threadIdx.x == 0) TC_TRACE_CTA(5);

  if (warp == kWarpProducer) {  // ===== TMA: (Q, dO) chunks, then (K, V) chunks =====
    if (lane == 0) {
      d32::prefetch_map(&tq);
      d32::prefetch_map(&tdo);
      d32::prefetch_map(&tk);
      d32::prefetch_map(&tv);
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        for (int ps = 0; ps < 2; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot3(it);
            if (COTTEN_ISSUED_GATE && it == 0) mbar_wait(&br->issued, 0);  // mask, S loads go first
            ItemPos f;
            if (p.l2_ahead && item_pos(it + p.l2_ahead, 2, C, units, H, f)) {
              tma_prefetch_4d(f.ps == 0 ? &tq : &tk, 0, f.c * kRows, f.h, f.b);
              tma_prefetch_4d(f.ps == 0 ? &tdo : &tv, 0, f.c * kRows, f.h, f.b);
            }
            mbar_wait(&br->raw_empty[st], par3(it) ^ 1u);
            uint8_t* dst = smem + kOffRaw + st * kStage;
            mbar_expect_tx(&br->raw_full[st], 2 * kTile);
            tma_load_4d(dst, ps == 0 ? &tq : &tk, 0, c * kRows, h, b, &br->raw_full[st]);
            tma_load_4d(dst + kTile, ps == 0 ? &tdo : &tv, 0, c * kRows, h, b, &br->raw_full[st]);
            if (it == 0) TC_TRACE_T0(2);
          }
      }
    }
  } else if (warp == kWarpMma) {  // ===== MMA issuer (whole warp, one elected lane issues) =====
    int it = 0, j = 0, nflush = 0;
    const uint32_t base = smem_u32(smem);
    const uint32_t opS = base + kOffOps, opA = opS + 2 * kOpBytes, opAt = opS + 4 * kOpBytes;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      for (int ps = 0; ps < 2; ++ps)
        for (int c = 0; c < C; ++c, ++it) {
          const int st = slot3(it), bf = st;
          TC_TRACE_MMA(0);
          mbar_wait(&br->split_full[bf], par3(it));
          if (ps == 1 && c == 0) mbar_wait(&br->op_ready, j & 1);
          if (ps == 0 && c > 0 && c % kFlush == 0) mbar_wait(&br->acc_free, (nflush++) & 1);
          tc_fence_after();
          TC_TRACE_MMA(1);
          const uint32_t X = base + kOffRaw + st * kStage;
          const uint32_t Y = base + kOffLo + bf * kStage;
          const uint32_t D = tmem + kBwdBuf0 + kBwdBufCols * bf;
          if (elect_one()) {
            if (ps == 0) {
              // G += Q~^T dO (attention.cpp:405)
              const int rows = min(kRows, N - c * kRows);
              issue_reduction(tmem, X, X + kTile, Y - X, (rows + 7) >> 3, c % kFlush == 0);
              // G is complete: the epiloguer starts the G-epilogue (the path to the
              // pass-2 MMAs) while the dQ~ MMAs below still run
              if (c == C - 1) mma_commit(&br->red_done);
              // dQ~ (unscaled) = dO S^T (:410-411): A = dO hi/lo in TMEM, B row n = S row n
              issue_rowout_ts<false>(D, D + 32, opS, opS + kOpBytes);
            } else {
              // dV = K~ dA (:416): A = K~ hi/lo in TMEM, B = dA rows as an MN-major operand
              issue_rowout_ts<true>(D, D + 64, opAt, opAt + kOpBytes);
              // dK~ = V dA^T (:415): A = V hi (TMA stage) / lo (lo buffer), B row n = dA row n
              issue_rowout_ss<false>(D + 32, X + kTile, Y + kTile, opA, opA + kOpBytes);
            }
            TC_TRACE_MMA(2);
            mma_commit(&br->raw_empty[st]);
            mma_commit(&br->mma_done[bf]);
          }
          __syncwarp();
        }
    }
  } else if (warp == kWarpMask) {
    mask_loop(p, smem, br, lane);
  } else if (warp == kWarpStore) {  // ===== TMA stores of staged outputs; lo-buffer recycling =====
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        for (int ps = 0; ps < 2; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int bf = slot3(it);
            uint8_t* Y = smem + kOffLo + bf * kStage;
            mbar_wait(&br->staged[bf], par3(it));
            if (ps == 0) {
              tma_store_4d(&tdq, Y, 0, c * kRows, h, b);
            } else {
              tma_store_4d(&tdk, Y, 0, c * kRows, h, b);
              tma_store_4d(&tdv, Y + kTile, 0, c * kRows, h, b);
            }
            bulk_wait_read0();
            mbar_arrive(&br->lo_free[bf]);
          }
      }
      store_tail();
    }
  } else {
    // ===== workers: group 0 splits every chunk, group 1 runs every epilogue =====
    const int g = warp >> 2, wq = warp & 3, t = threadIdx.x & 127;
    const float eps = (float)p.eps;
    const float* gS_all = static_cast<const float*>(p.saved_S);
    const uint32_t lane_base = (uint32_t)(32 * wq) << 16;
    // saved S of the next unit, prefetched a unit ahead by the splitter
    float4 snext[2];
    auto fetch_S = [&](int u) {
      if (u < units) {
        const float4* gs = reinterpret_cast<const float4*>(gS_all + (int64_t)u * 1024);
        snext[0] = __ldg(gs + t);
        snext[1] = __ldg(gs + t + 128);
      }
    };
    if (g == 0) {
      fetch_S(blockIdx.x);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&br->issued);
    }
    const float qnan = __int_as_float(0x7fc00000);
    int it = 0, j = 0, n_tr = 0;
    (void)n_tr;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int sl = j & 1;
      const uint32_t* fl = reinterpret_cast<const uint32_t*>(smem + kOffFlags + sl * (kMaxN / 8));
      mbar_wait(&br->fl_full[sl], (j >> 1) & 1);
      const UnitConst uc = ucs[sl];
      for (int k = 0; k < 2 * C; ++k, ++it) {  // the unit's chunks: pass 1, then pass 2
          const int ps = k >= C, c = ps ? k - C : k;
          const int st = slot3(it), bf = st;
          const int r = c * kRows + t;
          uint8_t* X = smem + kOffRaw + st * kStage;
          uint8_t* Y = smem + kOffLo + bf * kStage;
          const uint32_t D = tmem + kBwdBuf0 + kBwdBufCols * bf + lane_base;
          const uint32_t tinv = tmem + kBwdInv + bf + lane_base;
          if (g == 0) {  // ---------------- splitter ----------------
            TC_TRACE(0);
            if (it == 0 && t == 0) TC_TRACE_T0(3);
            mbar_wait(&br->raw_full[st], par3(it));
            mbar_wait(&br->lo_free[bf], par3(it) ^ 1u);
            TC_TRACE(1);
            if (it == 0 && t == 0) TC_TRACE_T0(4);
            if (ps == 0) {
              // Q~ every row (:366-377, used again in :421-428); rows past N are exact
              // zeros in G even for eps = 0.  Tiles use the 32-byte-granule swizzle.
              float xr[32], hh[32], ll[32];
              load_row32_raw(X, t, xr);
              const float inv = rsqrtf(sumsq(xr) + eps);
              scale32(xr, r < N ? inv : 0.f);
              split32(xr, hh, ll);
              TC_TRACE(3);
              store_row32_raw(X, t, hh);
              store_row32_raw(Y, t, ll);
              unswap32(xr, t);  // natural order: the dQ Jacobian pairs it with TMEM columns
              tmem_st32(D + 96, xr);  // q~ and inv for the epiloguer's dQ Jacobian
              tmem_st1(tinv, inv);
              TC_TRACE(4);
              load_row32_raw(X + kTile, t, hh);  // dO: the TMA tile itself is the hi operand
              lo32(hh, ll);
              store_row32_raw(Y + kTile, t, ll);
              unswap32(hh, t);
              unswap32(ll, t);
              TC_TRACE(5);
              tmem_st32(D + 32, hh);  // dO as the TMEM A operand of dQ~ = dO S^T
              tmem_st32(D + 64, ll);
              if (c == 0) {  // S rows (row n = S row n) for dQ~ = dO S^T
                // the previous unit's G-epilogue (dm) and dQ~ MMAs have read its S rows
                // (op_ready follows both); matters for C == 1, already true for C >= 2
                if (j > 0) mbar_wait(&br->op_ready, (j - 1) & 1);
#pragma unroll
                for (int e2 = 0; e2 < 2; ++e2) {
                  const int e = t + 128 * e2;
                  const int n = e >> 3, q4 = e & 7;
                  const float4 v = snext[e2];
                  const float4 hq =
                      make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
                  *reinterpret_cast<float4*>(ops + chunk_off(n, q4)) = hq;
                  *reinterpret_cast<float4*>(ops + kOpBytes + chunk_off(n, q4)) =
                      make_float4(tf32_lo(v.x, hq.x), tf32_lo(v.y, hq.y), tf32_lo(v.z, hq.z),
                                  tf32_lo(v.w, hq.w));
                }
                fetch_S(u + gridDim.x);
              }
            } else {  // K~ masked (TMEM A operand of dV = K~ dA) and V (smem A of dK~ = V dA^T)
              float kx[32];
              load_row(X, t, kx);
              const bool f = r < N && flag_at(fl, r);
              const float inv = rsqrtf(sumsq(kx) + eps);
              scale32(kx, inv);  // padded rows may hold anything: masked, never multiplied in
              tmem_store_split(D + 64, kx, f ? 0xFFFFFFFFu : 0u);
              tmem_st1(tinv, inv);
              load_row(X + kTile, t, kx);  // V: the TMA tile itself is the hi operand
              float vl[32];
              lo32(kx, vl);
              store_row(Y + kTile, t, vl);
            }
            tmem_wait_st();
            tc_fence_before();
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&br->split_full[bf]);
            TC_TRACE(2);
          } else {  // ---------------- epiloguer ----------------
            uint8_t* run = ops + 2 * kOpBytes;  // the dA operands' area, free until the G-epilogue
            if (ps == 0 && c == C - 1) {
              // G-epilogue first: it gates the pass-2 MMAs, the dQ epilogue does not
              mbar_wait(&br->red_done, j & 1);
              tc_fence_after();
              // G complete: dm (:408), dA = s G (:412-413) as both state operands
              float g8[8], h8[8], l8[8];
              reduce_rows8(tmem, Y + kTile, wq, lane, g, t, g8, C > kFlush ? run : nullptr);
              const int a = t >> 2, q = t & 3;
              double dot = 0.0;
#pragma unroll
              for (int hh2 = 0; hh2 < 2; ++hh2) {  // <G, S> (S row a = K-major operand row a)
                const float4 sh = *reinterpret_cast<const float4*>(ops + chunk_off(a, 2 * q + hh2));
                const float4 sl4 =
                    *reinterpret_cast<const float4*>(ops + kOpBytes + chunk_off(a, 2 * q + hh2));
                float d = g8[4 * hh2] * (sh.x + sl4.x);
                d = fmaf(g8[4 * hh2 + 1], sh.y + sl4.y, d);
                d = fmaf(g8[4 * hh2 + 2], sh.z + sl4.z, d);
                d = fmaf(g8[4 * hh2 + 3], sh.w + sl4.w, d);
                dot += (double)d;
              }
#pragma unroll
              for (int k = 0; k < 8; ++k) g8[k] *= uc.s;  // dA row a, columns 8q..8q+7
              split8(g8, h8, l8);
              store8_k(ops + 2 * kOpBytes, a, q, h8);  // K-major B of dK~ = V dA^T
              store8_k(ops + 3 * kOpBytes, a, q, l8);
              store8_mn(ops + 4 * kOpBytes, a, q, h8);  // MN-major B of dV = K~ dA
              store8_mn(ops + 5 * kOpBytes, a, q, l8);
              // fixed-order dm: warp tree, then the 4 warps of the group in order
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
              if (lane == 0) dm_x[wq] = dot;
              fence_proxy_async();
              tc_fence_before();
              group_sync(g);
              if (t == 0) {  // dm partials read before op_ready lets the next G-epilogue run
                const double dsum = ((dm_x[0] + dm_x[1]) + dm_x[2]) + dm_x[3];
                if (p.dm_unit) p.dm_unit[u] = uc.coef * dsum;
                mbar_arrive(&br->op_ready);
              }
            }
            mbar_wait(&br->mma_done[bf], par3(it));
            tc_fence_after();
            TC_TRACE(3);
            if (ps == 0 && c != C - 1 && c % kFlush == kFlush - 1) {  // long N: flush G
              flush_acc(tmem, run, wq, lane, c == kFlush - 1);
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&br->acc_free);
            }
            if (ps == 0) {
              // dQ_i = (g - (g.q~_i) q~_i) / nq_i, g = s dO S^T (:410-411, :421-428)
              float gq[32], xq[32];
              tmem_ld32(D, gq);
              tmem_ld32(D + 96, xq);
              const float inv = tmem_ld1(tinv);
              tmem_wait_ld();
              scale32(gq, uc.s);
              jacobian32(gq, xq, dot32(gq, xq), inv);
              store_row(Y, t, gq);  // staged in the lo buffer (free: the MMAs are done)
              tc_fence_before();
            } else {
              // dV_i = v_i ? (K~ dA)_i : 0 (:416, :439); dK_i = v_i ? (g - (g.k~)k~)/nk : 0 (:430-437)
              const bool f = r < N && flag_at(fl, r);
              const bool nan_out = uc.tn == 0;  // UsageError in the reference: NaN + status bit
              float kx[32], gk[32];
              float inv;
              {  // k~ = hi + lo exactly (valid rows); staged loads keep the register peak low
                float kl[32];
                tmem_ld32(D + 64, kx);
                tmem_ld32(D + 96, kl);
                inv = tmem_ld1(tinv);
                tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < 32; k += 2) {
                  const float2 v = __fadd2_rn(f2p(kx[k], kx[k + 1]), f2p(kl[k], kl[k + 1]));
                  kx[k] = v.x;
                  kx[k + 1] = v.y;
                }
              }
              tmem_ld32(D + 32, gk);
              tmem_wait_ld();
              jacobian32(gk, kx, dot32(gk, kx), inv);
              keep_if(gk, f);  // padded rows: exact zeros (:437)
              if (nan_out) {
#pragma unroll
                for (int k = 0; k < 32; ++k) gk[k] = qnan;
              }
              store_row(Y, t, gk);
              tmem_ld32(D, gk);  // dV
              tmem_wait_ld();
              tc_fence_before();
              keep_if(gk, f);  // (:439)
              if (nan_out) {
#pragma unroll
                for (int k = 0; k < 32; ++k) gk[k] = qnan;
              }
              store_row(Y + kTile, t, gk);
            }
            TC_TRACE(5);
            arrive_staged(br, bf, lane);
            TC_TRACE(4);
            ++n_tr;
          }
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&br->fl_empty[sl]);
    }
  }
  if (threadIdx.x == 128) {
    TC_TRACE_CTA(6);  // epiloguer thread 0: its last item is done
    if (p.dm_total) __threadfence();  // this thread wrote the CTA's dm_unit entries
  }
  tc_teardown(tmem, warp);
  if (p.dm_total) last_cta_dm_total(p, units, smem + kOffRaw);
  if (threadIdx.x == 0) TC_TRACE_CTA(7);
}

}  // namespace tc

// ---- host side ----------------------------------------------------------------------

// 4-D map over (D, N, H, B) with a (32, 128, 1, 1) box and 128-byte swizzle
// (loads zero-fill rows >= N; stores clip them).
// MN-major reduction operands are loaded with 32-byte granules (the UMMA
// SWIZZLE_128B_BASE32B layout); K-major operands and stores use 16-byte ones.
inline bool make_chunk_map(CUtensorMap* map, const void* base, const OpParams& p,
                           bool granule32 = false) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)p.D, (cuuint64_t)p.N, (cuuint64_t)p.H, (cuuint64_t)p.B};
  cuuint64_t strides[3] = {(cuuint64_t)p.sn * 4, (cuuint64_t)p.sh * 4, (cuuint64_t)p.sb * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)tc::kRows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             granule32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Sequences of <= 64 rows would leave half of every 128-row chunk empty; the
// FP32-pipe kernels (kernels_d32.cuh) serve them until units are packed.
#ifndef COTTEN_TC_MIN_N
#define COTTEN_TC_MIN_N 65
#endif
constexpr int64_t kTcMinN = COTTEN_TC_MIN_N;

inline bool tc_layout_ok(const OpParams& p, std::initializer_list<const void*> ptrs) {
  if (p.D != 32 || p.N < kTcMinN || p.N > tc::kMaxN) return false;
  if ((p.sn * 4) % 16 || (p.sh * 4) % 16 || (p.sb * 4) % 16) return false;
  if (p.B * p.H > (1ll << 31) - 1) return false;
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<uintptr_t>(q) & 15)) return false;
  return encode_fn() != nullptr;
}

template <typename T>
inline bool tc_fwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, float>::value) {
    return false;
  } else {
    return tc_layout_ok(p, {p.q, p.k, p.v, p.out});
  }
}
template <typename T>
inline bool tc_bwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, float>::value) {
    return false;
  } else {
    return p.saved_S != nullptr && tc_layout_ok(p, {p.q, p.k, p.v, p.dout, p.dq, p.dk, p.dv});
  }
}

// Phase-trace plumbing (trace builds only): a device buffer per launch, dumped
// to $COTTEN_TRACE_DIR/<fwd|bwd>.bin after the kernel.
inline void* tc_trace_begin(int grid) {
#if COTTEN_TC_TRACE
  static void* buf = nullptr;
  const size_t bytes = (size_t)grid * 3 * tc::kTraceItems * 8 * sizeof(long long);
  if (!buf) cudaMalloc(&buf, (size_t)1024 * 3 * tc::kTraceItems * 8 * sizeof(long long));
  cudaMemset(buf, 0, bytes);
  return buf;
#else
  (void)grid;
  return nullptr;
#endif
}
inline void tc_trace_end(void* buf, int grid, const char* tag, cudaStream_t st) {
#if COTTEN_TC_TRACE
  const char* dir = getenv("COTTEN_TRACE_DIR");
  if (!dir || !buf) return;
  const size_t n = (size_t)grid * 3 * tc::kTraceItems * 8;
  std::vector<long long> h(n);
  cudaStreamSynchronize(st);
  cudaMemcpy(h.data(), buf, n * sizeof(long long), cudaMemcpyDeviceToHost);
  std::string path = std::string(dir) + "/" + tag + ".bin";
  if (FILE* f = fopen(path.c_str(), "wb")) {
    fwrite(h.data(), sizeof(long long), n, f);
    fclose(f);
  }
#else
  (void)buf; (void)grid; (void)tag; (void)st;
#endif
}

// One CTA per SM, programmatic stream serialization (PDL) enabled.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tc::kThreads);
  cfg.dynamicSmemBytes = tc::kSmemBytes;
  cfg.stream = st;
  static const bool pdl = getenv("COTTEN_NO_PDL") == nullptr;  // A/B switch
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// L2 prefetch distance of the tcgen05 producers (items); COTTEN_L2_AHEAD
// overrides it (0 = off) for A/B runs.
// L2 prefetch distance (items) of the tcgen05 producers: COTTEN_L2_AHEAD if
// set, else 4 items for a forward whose units span >= 8 chunks and 0
// otherwise.  Measured (profiles/r02g_tcb_trace/l2_prefetch_ab.txt): the
// forward gains at long N (N = 4096 d_h 32: 0.85 -> 0.92; bf16 d_h 64:
// 0.50 -> 0.54), short units lose (ML-1M 0.42 -> 0.40) and every backward
// loses (its ring already holds two tensors per item).
inline int l2_ahead_items(bool forward = false, int chunks = 0) {
  static const int env = [] {
    const char* e = getenv("COTTEN_L2_AHEAD");
    return e ? atoi(e) : -1;
  }();
  if (env >= 0) return env;
  return forward && chunks >= 8 ? 4 : 0;
}

inline int launch_tc_fwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mo;
  if (!make_chunk_map(&mq, p.q, p) || !make_chunk_map(&mk, p.k, p, true) ||
      !make_chunk_map(&mv, p.v, p, true) || !make_chunk_map(&mo, p.out ? p.out : p.q, p))
    return -1;
  const int units = (int)(p.B * p.H);
  if (cudaFuncSetAttribute(tc::cos_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tc::kSmemBytes) != cudaSuccess)
    return -1;
  const int grid = std::min(units, sm_count());
  OpParams q = p;
  q.l2_ahead = l2_ahead_items(true, (int)((p.N + tc::kRows - 1) / tc::kRows));
  q.workspace = tc_trace_begin(grid);
  if (launch_pdl(tc::cos_fwd_tc_kernel, grid, st, mq, mk, mv, mo, q) != cudaSuccess) return -1;
  tc_trace_end(q.workspace, grid, "fwd", st);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

inline int launch_tc_bwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mg, mdq, mdk, mdv;
  if (!make_chunk_map(&mq, p.q, p, true) || !make_chunk_map(&mk, p.k, p) ||
      !make_chunk_map(&mv, p.v, p) || !make_chunk_map(&mg, p.dout, p, true) ||
      !make_chunk_map(&mdq, p.dq, p) || !make_chunk_map(&mdk, p.dk, p) ||
      !make_chunk_map(&mdv, p.dv, p))
    return -1;
  const int units = (int)(p.B * p.H);
  if (cudaFuncSetAttribute(tc::cos_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tc::kSmemBytes) != cudaSuccess)
    return -1;
  const int grid = std::min(units, sm_count());
  OpParams q = p;
  q.l2_ahead = l2_ahead_items();
  q.workspace = tc_trace_begin(grid);
  if (launch_pdl(tc::cos_bwd_tc_kernel, grid, st, mq, mk, mv, mg, mdq, mdk, mdv, q) != cudaSuccess)
    return -1;
  tc_trace_end(q.workspace, grid, "bwd", st);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace cotten
