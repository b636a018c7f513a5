// Tensor-core (tcgen05 kind::f16) cosine-attention kernels for bf16 inputs,
// head_dim 64, any seq_len up to 16384 — BASELINE config #5's bf16 points
// (north star: "tcgen05/TMEM tiles for the two small contractions ... at
// d_head >= 64"; the FP32-pipe kernels_rt.cuh is the A/B alternative).
//
// bf16 data in HBM, fp32 arithmetic everywhere; every value computed in
// fp32 that enters an MMA — the normalised rows q~ / k~ and the d_h x d_h
// state (S, dA = s G) — is a bf16 hi / lo pair (x = hi + lo to ~2^-17), and
// the MMAs accumulate hi*hi + hi*lo + lo*hi in fp32 TMEM ("bf16x3"; V and dO
// are bf16 already, so their products need hi only).  A single bf16 rounding
// of q~ / k~ is not enough: at N = 1, O = (q~.k~) v cancels and the 2^-9
// rounding grows to ~2e-2 (measured), over the 1e-2 bar.  The lo half of
// q~ / k~ overwrites the raw row in the TMA stage (each splitter thread owns
// its row), so no extra shared memory is needed; the epiloguer rebuilds
// q~ / k~ = hi + lo in fp32 for the row Jacobians, with 1/norm handed over in
// a TMEM column.
//
// Same persistent warp-role pipeline as the fp32 kernels (kernels_tc.cuh):
// 128-row chunks, one TMA box (64 bf16 x 128 rows = 16 KB, SWIZZLE_128B) per
// tensor per chunk, a 3-slot ring; per slot a raw stage (X, Y) and one
// "normalised" tile Z (q~ or k~ in bf16) that later stages the chunk's
// outputs for the TMA store.
//   forward   pass 1 (K, V):  Z|X = k~ hi|lo (masked);  S += (Z + X)^T Y    (M = N = 64, K = 16 rows)
//             pass 2 (Q):     Z|X = q~ hi|lo;           O = s (Z + X) S     (M = 128, N = 64, K = 64)
//   backward  pass 1 (Q, dO): Z|X = q~ hi|lo (r < N);   G += (Z + X)^T Y,  dQ~ = s Y S^T
//             pass 2 (K, V):  Z|X = k~ hi|lo (masked);  dV = (Z + X) dA,  dK~ = Y dA^T  (dA = s G)
// (attention.cpp:297-395, :397-441).  Operand conventions (measured in
// scripts/dev/mma_probe_bf16.cu): a 128-B-row SW128 tile is both the
// MN-major operand of a reduction (rows = K) and the K-major operand of a
// row output (rows = M); the 64 x 64 state tiles (S or dA rows, bf16) are the
// MN-major B of O = Q~ S / dV = K~ dA and the K-major B of dQ~ = dO S^T /
// dK~ = V dA^T alike.
//
// Paired rows (kPair, head_dim 32): a contiguous [N][32] bf16 unit (N even)
// is read as [N/2][64] — packed row p = rows 2p | 2p+1, one 128-B row — so
// the same 128-B tiles, TMA boxes and MMAs serve d_h = 32 (attention.cpp has
// no head-dim restriction).  Each half of a packed row is normalised, masked
// and differentiated as its own row; the 64 x 64 reduction R' = X'^T Y' holds
// R = R'00 + R'11 on its diagonal blocks (the off-diagonal blocks pair row 2p
// with 2p+1 and are discarded), and the state operand is blockdiag(S, S) /
// blockdiag(dA, dA), so every row output [x_2p | x_2p+1] B' = [x_2p S | x_2p+1 S].
// The tensor pipe does twice the useful work, which it has to spare; the
// alternative (64-B rows) would halve every TMA box and MMA K-step.
//
// Warp roles (512 threads): 0-7 splitter (two threads per chunk row, 32
// columns each: a single splitter warp per SMSP was the latency-bound stage,
// measured), 8-11 epiloguer (thread t = TMEM lane t, rows processed in two
// 32-column halves to stay within 128 registers), 12 TMA producer, 13 MMA
// issuer, 14 mask warp, 15 store warp (TMA stores, then frees the slot).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels_tc.cuh"

namespace cotten {
namespace tcb {

using d32::mbar_arrive;
using d32::mbar_expect_tx;
using d32::mbar_init;
using d32::mbar_wait;
using d32::smem_u32;
using d32::tma_load_4d;
using tc::bulk_wait0;
using tc::bulk_wait_read0;
using tc::elect_one;
using tc::fence_proxy_async;
using tc::mma_commit;
using tc::tc_fence_after;
using tc::tc_fence_before;
using tc::tma_store_4d;
using tc::tmem_ld32;
using tc::tmem_wait_ld;
using tc::UnitConst;

constexpr int kD = 64;
constexpr int kRows = 128;
constexpr uint32_t kTile = 16384;  // 128 rows x 128 B
constexpr int kRing = 3;
constexpr int kMaxN = 16384;
constexpr int kFlush = 4;  // S / G accumulator flushed every 4 chunks (<= 32 MMAs per chain)
constexpr int kSplitWarps = 8, kEpiWarps = 4;
constexpr int kWarpEpi0 = kSplitWarps;
constexpr int kWarpProducer = 12, kWarpMma = 13, kWarpMask = 14, kWarpStore = 15;
constexpr int kThreads = 16 * 32;

// shared memory: per slot X, Y (raw TMA tiles) and Z (normalised / staging)
constexpr uint32_t kSlot = 3 * kTile;
constexpr uint32_t kOffRing = 0;
constexpr uint32_t kStateTile = 64 * 128;  // 64 x 64 bf16 rows
constexpr uint32_t kOffOps = kOffRing + kRing * kSlot;   // S hi, S lo, dA hi, dA lo
constexpr uint32_t kOffRun = kOffOps + 4 * kStateTile;   // fp32 running sum, 64 x 64
constexpr uint32_t kOffFlags = kOffRun + 64 * 64 * 4;    // 2 x 2 KB bitmasks
constexpr uint32_t kOffInv = kOffFlags + 2 * (kMaxN / 8);  // per slot 256 x 1/norm (bwd)
constexpr uint32_t kOffScr = kOffInv + kRing * 2 * kRows * 4;  // paired rows: 32 x 32 fp32 hand-off
constexpr uint32_t kOffMisc = kOffScr + 32 * 32 * 4;
constexpr uint32_t kOffBar = kOffMisc + 128;
constexpr uint32_t kSmemBytes = kOffBar + 32 * 8;
static_assert(kSmemBytes <= 227 * 1024, "shared-memory budget");

// TMEM: [0, 64) the S / G accumulator (M = 64: row m at lane (m % 16) + 32 (m / 16));
// slot b at 64 + 128 b: [+0, +64) O | dQ~ | dV, [+64, +128) dK~.
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kBuf0 = 64;
constexpr uint32_t kBufCols = 128;

// Optional per-item trace (-DCOTTEN_TCB_TRACE=1): clock64 stamps of the first
// kTraceItems items of every CTA into p.workspace [cta][item][8]:
// 0 splitter waits raw, 1 raw landed, 2 split published, 3 MMA sees split,
// 4 MMAs issued, 5 epiloguer sees MMAs done, 6 outputs staged, 7 slot freed.
#ifndef COTTEN_TCB_TRACE
#define COTTEN_TCB_TRACE 0
#endif
constexpr int kTraceItems = 64;
#if COTTEN_TCB_TRACE
#define TCB_TRACE(k, cond)                                                                   \
  do {                                                                                       \
    if ((cond) && p.workspace && it < kTraceItems)                                           \
      static_cast<long long*>(p.workspace)[(blockIdx.x * kTraceItems + it) * 8 + (k)] = clock64(); \
  } while (0)
#else
#define TCB_TRACE(k, cond) \
  do {                     \
  } while (0)
#endif

__device__ __forceinline__ int slot3(int it) { return it % kRing; }
__device__ __forceinline__ uint32_t par3(int it) { return (uint32_t)(it / kRing) & 1u; }

struct Bars {
  uint64_t raw_full[kRing], slot_free[kRing], split_full[kRing], mma_done[kRing], staged[kRing];
  uint64_t op_ready, acc_free, red_done;
  uint64_t fl_full[2], fl_empty[2];
  uint64_t issued;  // the first unit's mask loads are out (kernels_tc.cuh Bars::issued)
};
static_assert(sizeof(Bars) <= 256, "barrier area");

// ---- bf16 rows of a 128-B SW128 tile (16-byte granule j of row r at j ^ (r & 7)) ----
__device__ __forceinline__ uint32_t goff(int row, int j) {
  return (uint32_t)row * 128u + ((uint32_t)(j ^ (row & 7)) << 4);
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void unpack8(const uint4 v, float* x) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
    x[2 * e] = f.x;
    x[2 * e + 1] = f.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* x) {
  return make_uint4(pack2(x[0], x[1]), pack2(x[2], x[3]), pack2(x[4], x[5]), pack2(x[6], x[7]));
}
// columns [32 h, 32 h + 32) of a row = granules 4h .. 4h + 3
__device__ __forceinline__ void load_half(const uint8_t* tile, int row, int h, float (&x)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) unpack8(*reinterpret_cast<const uint4*>(tile + goff(row, 4 * h + q)), x + 8 * q);
}
__device__ __forceinline__ void store_half(uint8_t* tile, int row, int h, const float (&x)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(tile + goff(row, 4 * h + q)) = pack8(x + 8 * q);
}
// x = hi + lo (bf16 each) for half h of a row
__device__ __forceinline__ void store_split_half(uint8_t* hi_tile, uint8_t* lo_tile, int row, int h,
                                                 const float (&x)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // one cvt.rn.bf16x2.f32 per pair; bf16 -> fp32 is a shift
      const float x0 = x[8 * q + 2 * e], x1 = x[8 * q + 2 * e + 1];
      hw[e] = pack2(x0, x1);
      lw[e] = pack2(x0 - __uint_as_float(hw[e] << 16), x1 - __uint_as_float(hw[e] & 0xFFFF0000u));
    }
    *reinterpret_cast<uint4*>(hi_tile + goff(row, 4 * h + q)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(lo_tile + goff(row, 4 * h + q)) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
}
__device__ __forceinline__ void load_split_half(const uint8_t* hi_tile, const uint8_t* lo_tile,
                                                int row, int h, float (&x)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float a[8], b[8];
    unpack8(*reinterpret_cast<const uint4*>(hi_tile + goff(row, 4 * h + q)), a);
    unpack8(*reinterpret_cast<const uint4*>(lo_tile + goff(row, 4 * h + q)), b);
#pragma unroll
    for (int e = 0; e < 8; ++e) x[8 * q + e] = a[e] + b[e];
  }
}
__device__ __forceinline__ float sumsq32(const float (&x)[32]) {
  float a = 0.f, b = 0.f, c = 0.f, d = 0.f;
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    a = fmaf(x[k], x[k], a);
    b = fmaf(x[k + 1], x[k + 1], b);
    c = fmaf(x[k + 2], x[k + 2], c);
    d = fmaf(x[k + 3], x[k + 3], d);
  }
  return (a + b) + (c + d);
}
__device__ __forceinline__ float dot32(const float (&x)[32], const float (&y)[32]) {
  float a = 0.f, b = 0.f, c = 0.f, d = 0.f;
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    a = fmaf(x[k], y[k], a);
    b = fmaf(x[k + 1], y[k + 1], b);
    c = fmaf(x[k + 2], y[k + 2], c);
    d = fmaf(x[k + 3], y[k + 3], d);
  }
  return (a + b) + (c + d);
}
// 32 accumulator columns of this thread's lane
__device__ __forceinline__ void tmem_ld_half(uint32_t taddr, float (&r)[32]) {
  tmem_ld32(taddr, r);
  tmem_wait_ld();
}

// ---- MMA issue ------------------------------------------------------------------
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);  // SWIZZLE_128B
}
__device__ __forceinline__ uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  // D fp32, A / B bf16
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// R (M = N = 64) += x^T y over `ksteps` 16-row groups of two MN-major tiles
__device__ __forceinline__ void issue_reduction(uint32_t d, uint32_t x, uint32_t y, int ksteps,
                                                bool first) {
  const uint32_t id = idesc_bf16(64, 64, true, true);
  for (int kk = 0; kk < ksteps; ++kk)
    mma_bf16(d, sdesc(x + 2048u * kk, kTile, 1024u), sdesc(y + 2048u * kk, kTile, 1024u), id,
             (first && kk == 0) ? 0u : 1u);
}
// D (128 x 64) = A (K-major chunk tile, K = 64 features) x B (state hi + lo):
// B MN-major (rows = k) for O = Q~ S, dV = K~ dA; K-major (rows = n) for
// dQ~ = dO S^T, dK~ = V dA^T.
template <bool kBMN>
__device__ __forceinline__ void issue_rowout(uint32_t d, uint32_t a, uint32_t bh, uint32_t bl) {
  const uint32_t id = idesc_bf16(128, 64, false, kBMN);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint64_t ad = sdesc(a + 32u * kk, 16u, 1024u);
    const uint64_t dh = kBMN ? sdesc(bh + 2048u * kk, kTile, 1024u) : sdesc(bh + 32u * kk, 16u, 1024u);
    const uint64_t dl = kBMN ? sdesc(bl + 2048u * kk, kTile, 1024u) : sdesc(bl + 32u * kk, 16u, 1024u);
    mma_bf16(d, ad, dh, id, kk > 0 ? 1u : 0u);
    mma_bf16(d, ad, dl, id, 1u);
  }
}

// Same with A = hi (ah) + lo (al): hi*hi + hi*lo + lo*hi (12 MMAs)
template <bool kBMN>
__device__ __forceinline__ void issue_rowout3(uint32_t d, uint32_t ah, uint32_t al, uint32_t bh,
                                              uint32_t bl) {
  const uint32_t id = idesc_bf16(128, 64, false, kBMN);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint64_t adh = sdesc(ah + 32u * kk, 16u, 1024u), adl = sdesc(al + 32u * kk, 16u, 1024u);
    const uint64_t dh = kBMN ? sdesc(bh + 2048u * kk, kTile, 1024u) : sdesc(bh + 32u * kk, 16u, 1024u);
    const uint64_t dl = kBMN ? sdesc(bl + 2048u * kk, kTile, 1024u) : sdesc(bl + 32u * kk, 16u, 1024u);
    mma_bf16(d, adh, dh, id, kk > 0 ? 1u : 0u);
    mma_bf16(d, adh, dl, id, 1u);
    mma_bf16(d, adl, dh, id, 1u);
  }
}
// ---- setup / mask warp ----------------------------------------------------------
__device__ __forceinline__ uint32_t setup(uint8_t* smem, Bars* br, uint32_t* tslot, int warp) {
  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023u) __trap();
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&br->raw_full[i], 1);
      mbar_init(&br->slot_free[i], 1);
      mbar_init(&br->split_full[i], kSplitWarps);
      mbar_init(&br->mma_done[i], 1);
      mbar_init(&br->staged[i], kEpiWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&br->fl_full[i], 1);
      mbar_init(&br->fl_empty[i], kSplitWarps + kEpiWarps);
    }
    mbar_init(&br->op_ready, 1);
    mbar_init(&br->acc_free, kEpiWarps);
    mbar_init(&br->red_done, 1);
    mbar_init(&br->issued, 1);
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
__device__ __forceinline__ void teardown(uint32_t tmem, int warp) {
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  }
}
__device__ __forceinline__ void mask_loop(const OpParams& p, uint8_t* smem, Bars* br, int lane) {
  UnitConst* ucs = reinterpret_cast<UnitConst*>(smem + kOffMisc);
  const int units = (int)(p.B * p.H), H = (int)p.H;
  int j = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
    const int sl = j & 1;
    mbar_wait(&br->fl_empty[sl], ((j >> 1) & 1) ^ 1);
    tc::mask_unit(p, u / H, reinterpret_cast<uint32_t*>(smem + kOffFlags + sl * (kMaxN / 8)),
                  &ucs[sl], lane, j == 0 ? &br->issued : nullptr);
    __syncwarp();
    if (lane == 0) mbar_arrive(&br->fl_full[sl]);
  }
}
// Half h of the M = 64 accumulator row of this thread (lanes 0-15 of each
// warp hold rows 16 wq + lane) plus the flushed running sum.  The running
// sum's row a = 16 wq + lane keeps float4 k at slot k ^ lane, so the 16
// lanes of a warp hit 16 different 16-byte slots (2 wavefronts, the minimum).
__device__ __forceinline__ void acc_half(uint32_t tmem, const float* run, int wq, int lane, int h,
                                         bool with_run, float (&r)[32]) {
  tmem_ld_half(tmem + ((uint32_t)(32 * wq) << 16) + 32u * h, r);
  if (with_run && lane < 16) {
    const float4* rr = reinterpret_cast<const float4*>(run + (16 * wq + lane) * 64);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 v = rr[(8 * h + k) ^ lane];
      r[4 * k] += v.x;
      r[4 * k + 1] += v.y;
      r[4 * k + 2] += v.z;
      r[4 * k + 3] += v.w;
    }
  }
}
__device__ __forceinline__ void flush_acc(uint32_t tmem, float* run, int wq, int lane, bool first) {
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    float r[32];
    acc_half(tmem, run, wq, lane, h, !first, r);
    if (lane < 16) {
      float4* rr = reinterpret_cast<float4*>(run + (16 * wq + lane) * 64);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        rr[(8 * h + k) ^ lane] = make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
    }
  }
}
// Half h = lane / 16 (columns 32 h ..) of accumulator row 16 wq + lane % 16 for
// all 32 lanes at once (tcgen05.ld.16x32bx2), plus the flushed running sum: the
// per-unit S / G epilogue of the d_h = 64 kernels runs on all 128 threads.
__device__ __forceinline__ void acc_pair(uint32_t tmem, const float* run, int wq, int lane,
                                         bool with_run, float (&r)[32]) {
  uint32_t* u = reinterpret_cast<uint32_t*>(r);
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], 32;"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
        "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
        "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
        "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(tmem + ((uint32_t)(32 * wq) << 16)));
  tmem_wait_ld();
  if (with_run) {
    const int l = lane & 15, h = lane >> 4;
    const float4* rr = reinterpret_cast<const float4*>(run + (16 * wq + l) * 64);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 v = rr[(8 * h + k) ^ l];
      r[4 * k] += v.x;
      r[4 * k + 1] += v.y;
      r[4 * k + 2] += v.z;
      r[4 * k + 3] += v.w;
    }
  }
}
// <x, hi + lo> over half h of row a of a state tile pair
__device__ __forceinline__ float dot_state_half(const uint8_t* hi, const uint8_t* lo, int a, int h,
                                                const float (&x)[32]) {
  float s[32];
  load_split_half(hi, lo, a, h, s);
  return dot32(x, s);
}
__device__ __forceinline__ void arrive_staged(Bars* br, int b, int lane) {
  fence_proxy_async();
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(&br->staged[b]);
}
__device__ __forceinline__ void epi_sync() {  // the 4 epiloguer warps
  asm volatile("bar.sync 2, 128;" ::: "memory");
}

// Splitter: two threads per chunk row; the row's squared norm is the sum of
// the pair's halves (lanes 2i, 2i + 1 of the same warp).
struct SplitRow {
  int row, h;
  float x[32];
  float ss;  // |row|^2 (both halves)
};
// (kPair: each half is a row of its own, so no partner sum.)
template <bool kPair>
__device__ __forceinline__ void split_load(const uint8_t* X, int t, SplitRow& s) {
  s.row = t >> 1;
  s.h = t & 1;
  load_half(X, s.row, s.h, s.x);
  const float part = sumsq32(s.x);
  s.ss = kPair ? part : part + __shfl_xor_sync(0xffffffffu, part, 1);
}

// ---- paired rows (d_h = 32) --------------------------------------------------------
// R = R'00 + R'11 of the finished 64 x 64 accumulator (+ running sum): warps
// 2-3 (rows 32-63, columns 32-63) hand their rows to warps 0-1 through `scr`
// (row stride 128 B, float4 k of row a at slot k ^ (a & 7): 2 wavefronts per
// 16-lane access); on return lanes < 16 of warps 0-1 hold R row 16 wq + lane.
__device__ __forceinline__ void pair_combine(uint32_t tmem, const float* run, float* scr, int wq,
                                             int lane, bool with_run, float (&r)[32]) {
  acc_half(tmem, run, wq, lane, wq >= 2 ? 1 : 0, with_run, r);
  const int a = 16 * (wq & 1) + lane;
  if (wq >= 2 && lane < 16) {
    float4* d = reinterpret_cast<float4*>(scr + a * 32);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      d[k ^ (a & 7)] = make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
  }
  epi_sync();
  if (wq < 2 && lane < 16) {
    const float4* d = reinterpret_cast<const float4*>(scr + a * 32);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 v = d[k ^ (a & 7)];
      r[4 * k] += v.x;
      r[4 * k + 1] += v.y;
      r[4 * k + 2] += v.z;
      r[4 * k + 3] += v.w;
    }
  }
}
// Row a (< 32) of a 32 x 32 state as rows a and a + 32 of blockdiag(X, X) (bf16 hi / lo).
__device__ __forceinline__ void store_blockdiag(uint8_t* hi, uint8_t* lo, int a, const float (&x)[32]) {
  float z[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) z[e] = 0.f;
  store_split_half(hi, lo, a, 0, x);
  store_split_half(hi, lo, a, 1, z);
  store_split_half(hi, lo, a + 32, 0, z);
  store_split_half(hi, lo, a + 32, 1, x);
}

// ======================================================================================
// Forward
// ======================================================================================
template <bool kPair>
__global__ void __launch_bounds__(kThreads, 1) cos_fwd_tcb_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap to,
    const OpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = (int)p.N, H = (int)p.H;
  const int NP = kPair ? (N + 1) >> 1 : N;  // tile rows (packed rows when kPair)
  const int units = (int)(p.B * p.H);
  const int C = (NP + kRows - 1) / kRows;
  const int P = (p.out != nullptr || p.saved_norms != nullptr) ? 2 : 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Bars* br = reinterpret_cast<Bars*>(smem + kOffBar);
  UnitConst* ucs = reinterpret_cast<UnitConst*>(smem + kOffMisc);
  uint8_t* ops = smem + kOffOps;
  float* run = reinterpret_cast<float*>(smem + kOffRun);
  const uint32_t tmem = setup(smem, br, reinterpret_cast<uint32_t*>(smem + kOffMisc + 32), warp);
  tc::pdl_wait();
  const KernelStamp stamp_(p);
  tc::pdl_launch_dependents();

  if (warp == kWarpProducer) {
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
            tc::ItemPos f;
            if (p.l2_ahead && tc::item_pos(it + p.l2_ahead, P, C, units, H, f)) {
              if (f.ps == 0) {
                tc::tma_prefetch_4d(&tk, 0, f.c * kRows, f.h, f.b);
                tc::tma_prefetch_4d(&tv, 0, f.c * kRows, f.h, f.b);
              } else {
                tc::tma_prefetch_4d(&tq, 0, f.c * kRows, f.h, f.b);
              }
            }
            mbar_wait(&br->slot_free[st], par3(it) ^ 1u);
            uint8_t* X = smem + kOffRing + st * kSlot;
            if (ps == 0) {
              mbar_expect_tx(&br->raw_full[st], 2 * kTile);
              tma_load_4d(X, &tk, 0, c * kRows, h, b, &br->raw_full[st]);
              tma_load_4d(X + kTile, &tv, 0, c * kRows, h, b, &br->raw_full[st]);
            } else {
              mbar_expect_tx(&br->raw_full[st], kTile);
              tma_load_4d(X, &tq, 0, c * kRows, h, b, &br->raw_full[st]);
            }
          }
      }
    }
  } else if (warp == kWarpMma) {
    int it = 0, j = 0, nflush = 0;
    const uint32_t base = smem_u32(smem);
    const uint32_t opS = base + kOffOps;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      for (int ps = 0; ps < P; ++ps)
        for (int c = 0; c < C; ++c, ++it) {
          const int st = slot3(it);
          mbar_wait(&br->split_full[st], par3(it));
          TCB_TRACE(3, lane == 0);
          if (ps == 0 && c == 0 && P == 1 && j > 0) mbar_wait(&br->op_ready, (j - 1) & 1);
          if (ps == 0 && c > 0 && c % kFlush == 0) mbar_wait(&br->acc_free, (nflush++) & 1);
          if (ps == 1 && c == 0) mbar_wait(&br->op_ready, j & 1);
          tc_fence_after();
          const uint32_t X = base + kOffRing + st * kSlot, Z = X + 2 * kTile;
          if (elect_one()) {
            if (ps == 0) {  // S += K~^T V (attention.cpp:345-353), K~ = hi (Z) + lo (X)
              const int ks = (min(kRows, NP - c * kRows) + 15) >> 4;
              issue_reduction(tmem, Z, X + kTile, ks, c % kFlush == 0);
              issue_reduction(tmem, X, X + kTile, ks, false);
            } else {  // O = Q~ S (:379-387)
              issue_rowout3<true>(tmem + kBuf0 + kBufCols * st, Z, X, opS, opS + kStateTile);
            }
            mma_commit(&br->mma_done[st]);
          }
          TCB_TRACE(4, lane == 0);
          __syncwarp();
        }
    }
  } else if (warp == kWarpMask) {
    mask_loop(p, smem, br, lane);
  } else if (warp == kWarpStore) {
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        for (int ps = 0; ps < P; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot3(it);
            mbar_wait(&br->staged[st], par3(it));
            if (ps == 1 && p.out) {
              tma_store_4d(&to, smem + kOffRing + st * kSlot + 2 * kTile, 0, c * kRows, h, b);
              bulk_wait_read0();
            }
            mbar_arrive(&br->slot_free[st]);
            TCB_TRACE(7, true);
          }
      }
      tc::store_tail();
    }
  } else {
    const bool splitter = warp < kWarpEpi0;
    const int wq = warp & 3;
    const int t = splitter ? (int)threadIdx.x : (int)threadIdx.x - 32 * kWarpEpi0;
    const float eps = (float)p.eps;
    float* norms_all = static_cast<float*>(p.saved_norms);
    float* gS_all = static_cast<float*>(p.saved_S);
    const uint32_t lane_base = (uint32_t)(32 * wq) << 16;
    int it = 0, j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int sl = j & 1;
      const uint32_t* fl = reinterpret_cast<const uint32_t*>(smem + kOffFlags + sl * (kMaxN / 8));
      float* norms = norms_all ? norms_all + (int64_t)u * 2 * N : nullptr;
      mbar_wait(&br->fl_full[sl], (j >> 1) & 1);
      const UnitConst uc = ucs[sl];
      for (int k = 0; k < P * C; ++k, ++it) {
        const int ps = k >= C, c = ps ? k - C : k;
        const int st = slot3(it);
        uint8_t* X = smem + kOffRing + st * kSlot;
        uint8_t* Z = X + 2 * kTile;
        if (splitter) {  // ---------------- splitter (2 threads per row) ----------------
          TCB_TRACE(0, threadIdx.x == 0);
          mbar_wait(&br->raw_full[st], par3(it));
          TCB_TRACE(1, threadIdx.x == 0);
          SplitRow s;
          split_load<kPair>(X, t, s);
          // sequence row of this half (kPair: packed row s.row holds rows 2 s.row, 2 s.row + 1)
          const int r = kPair ? 2 * c * kRows + t : c * kRows + s.row;
          const bool wr = norms && r < N && (kPair || s.h == 0);
          const float iv = rsqrtf(s.ss + eps);
          if (ps == 0) {  // k~ masked (attention.cpp:334-343)
            const bool f = r < N && tc::flag_at(fl, r);
            if (wr) norms[N + r] = f ? (s.ss + eps) * iv : 1.0f;
#pragma unroll
            for (int e = 0; e < 32; ++e) s.x[e] = f ? s.x[e] * iv : 0.f;  // NaN-safe zeros
          } else {  // q~ every row (:366-377)
            if (wr) norms[r] = (s.ss + eps) * iv;
#pragma unroll
            for (int e = 0; e < 32; ++e) s.x[e] *= iv;
          }
          store_split_half(Z, X, s.row, s.h, s.x);  // lo over this thread's own raw half row
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&br->split_full[st]);
          TCB_TRACE(2, threadIdx.x == 0);
        } else {  // ---------------- epiloguer ----------------
          mbar_wait(&br->mma_done[st], par3(it));
          TCB_TRACE(5, t == 0);
          tc_fence_after();
          if (ps == 0) {
            // a pass-1 item stages nothing and its MMAs are done: release the slot
            // before the flush / S-epilogue (TMEM, the running sum and the operand
            // area only), so the splitter can refill it meanwhile
            arrive_staged(br, st, lane);
            if (c != C - 1 && c % kFlush == kFlush - 1) {  // long N: flush the accumulator
              flush_acc(tmem, run, wq, lane, c == kFlush - 1);
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&br->acc_free);
            }
            if (kPair && c == C - 1) {  // S = S'00 + S'11; operand blockdiag(S, S)
              float sv[32];
              pair_combine(tmem, run, reinterpret_cast<float*>(smem + kOffScr), wq, lane, C > kFlush, sv);
              if (wq < 2 && lane < 16) {
                const int a = 16 * wq + lane;
                if (gS_all) {
                  float4* gs = reinterpret_cast<float4*>(gS_all + (int64_t)u * 1024 + a * 32);
#pragma unroll
                  for (int e = 0; e < 8; ++e)
                    gs[e] = make_float4(sv[4 * e], sv[4 * e + 1], sv[4 * e + 2], sv[4 * e + 3]);
                }
                store_blockdiag(ops, ops + kStateTile, a, sv);
              }
              fence_proxy_async();
              tc_fence_before();
              epi_sync();
              if (t == 0) mbar_arrive(&br->op_ready);
            } else if (c == C - 1) {  // S complete: saved S + the bf16 hi / lo state operand
              const int a = 16 * wq + (lane & 15), h = lane >> 4;  // all 128 threads
              float sv[32];
              acc_pair(tmem, run, wq, lane, C > kFlush, sv);
              if (gS_all) {
                float4* gs = reinterpret_cast<float4*>(gS_all + (int64_t)u * 4096 + a * 64 + 32 * h);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  gs[e] = make_float4(sv[4 * e], sv[4 * e + 1], sv[4 * e + 2], sv[4 * e + 3]);
              }
              store_split_half(ops, ops + kStateTile, a, h, sv);
              fence_proxy_async();
              tc_fence_before();
              epi_sync();
              if (t == 0) mbar_arrive(&br->op_ready);
            }
          } else {  // O rows = s (Q~ S), staged in Z (its MMAs are done)
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
              float o[32];
              tmem_ld_half(tmem + kBuf0 + kBufCols * st + lane_base + 32u * h, o);
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] *= uc.s;
              store_half(Z, t, h, o);
            }
            arrive_staged(br, st, lane);
          }
          TCB_TRACE(6, t == 0);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&br->fl_empty[sl]);
    }
  }
  teardown(tmem, warp);
}

// ======================================================================================
// Backward
// ======================================================================================
template <bool kPair>
__global__ void __launch_bounds__(kThreads, 1) cos_bwd_tcb_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
    const __grid_constant__ CUtensorMap tdq, const __grid_constant__ CUtensorMap tdk,
    const __grid_constant__ CUtensorMap tdv, const OpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = (int)p.N, H = (int)p.H;
  const int NP = kPair ? (N + 1) >> 1 : N;  // tile rows (packed rows when kPair)
  const int units = (int)(p.B * p.H);
  const int C = (NP + kRows - 1) / kRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Bars* br = reinterpret_cast<Bars*>(smem + kOffBar);
  UnitConst* ucs = reinterpret_cast<UnitConst*>(smem + kOffMisc);
  double* dm_x = reinterpret_cast<double*>(smem + kOffMisc + 40);
  uint8_t* ops = smem + kOffOps;
  float* run = reinterpret_cast<float*>(smem + kOffRun);
  float* invs = reinterpret_cast<float*>(smem + kOffInv);
  const uint32_t tmem = setup(smem, br, reinterpret_cast<uint32_t*>(smem + kOffMisc + 32), warp);
  tc::pdl_wait();
  const KernelStamp stamp_(p);
  tc::pdl_launch_dependents();

  if (warp == kWarpProducer) {
    if (lane == 0) {
      d32::prefetch_map(&tq);
      d32::prefetch_map(&tdo);
      d32::prefetch_map(&tk);
      d32::prefetch_map(&tv);
      int it = 0;
      const int64_t sbytes = (int64_t)p.D * p.D * 4;  // one unit's saved S
      if (blockIdx.x < units) tc::bulk_prefetch_l2(static_cast<const uint8_t*>(p.saved_S) + blockIdx.x * sbytes, (uint32_t)sbytes);
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        // the splitter loads the next unit's S at its first chunk: have it in L2
        if (u + (int)gridDim.x < units)
          tc::bulk_prefetch_l2(static_cast<const uint8_t*>(p.saved_S) + (u + gridDim.x) * sbytes, (uint32_t)sbytes);
        for (int ps = 0; ps < 2; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot3(it);
            if (COTTEN_ISSUED_GATE && it == 0) mbar_wait(&br->issued, 0);  // mask loads go first
            tc::ItemPos f;
            if (p.l2_ahead && tc::item_pos(it + p.l2_ahead, 2, C, units, H, f)) {
              tc::tma_prefetch_4d(f.ps == 0 ? &tq : &tk, 0, f.c * kRows, f.h, f.b);
              tc::tma_prefetch_4d(f.ps == 0 ? &tdo : &tv, 0, f.c * kRows, f.h, f.b);
            }
            mbar_wait(&br->slot_free[st], par3(it) ^ 1u);
            uint8_t* X = smem + kOffRing + st * kSlot;
            mbar_expect_tx(&br->raw_full[st], 2 * kTile);
            tma_load_4d(X, ps == 0 ? &tq : &tk, 0, c * kRows, h, b, &br->raw_full[st]);
            tma_load_4d(X + kTile, ps == 0 ? &tdo : &tv, 0, c * kRows, h, b, &br->raw_full[st]);
          }
      }
    }
  } else if (warp == kWarpMma) {
    int it = 0, j = 0, nflush = 0;
    const uint32_t base = smem_u32(smem);
    const uint32_t opS = base + kOffOps, opA = opS + 2 * kStateTile;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      for (int ps = 0; ps < 2; ++ps)
        for (int c = 0; c < C; ++c, ++it) {
          const int st = slot3(it);
          mbar_wait(&br->split_full[st], par3(it));
          TCB_TRACE(3, lane == 0);
          if (ps == 1 && c == 0) mbar_wait(&br->op_ready, j & 1);
          if (ps == 0 && c > 0 && c % kFlush == 0) mbar_wait(&br->acc_free, (nflush++) & 1);
          tc_fence_after();
          const uint32_t X = base + kOffRing + st * kSlot, Y = X + kTile, Z = X + 2 * kTile;
          const uint32_t D = tmem + kBuf0 + kBufCols * st;
          if (elect_one()) {
            if (ps == 0) {
              // G += Q~^T dO (attention.cpp:405), Q~ = hi (Z) + lo (X)
              const int ks = (min(kRows, NP - c * kRows) + 15) >> 4;
              issue_reduction(tmem, Z, Y, ks, c % kFlush == 0);
              issue_reduction(tmem, X, Y, ks, false);
              // dQ~ (unscaled) = dO S^T (:410-411): A = dO (K-major), B row n = S row n
              issue_rowout<false>(D, Y, opS, opS + kStateTile);
              // G complete (and every MMA that reads this unit's S rows: the
              // splitter may overwrite them once the G-epilogue has run)
              if (c == C - 1) mma_commit(&br->red_done);
            } else {
              issue_rowout3<true>(D, Z, X, opA, opA + kStateTile);     // dV = K~ dA (:416)
              issue_rowout<false>(D + 64, Y, opA, opA + kStateTile);   // dK~ = V dA^T (:415)
            }
            mma_commit(&br->mma_done[st]);
          }
          TCB_TRACE(4, lane == 0);
          __syncwarp();
        }
    }
  } else if (warp == kWarpMask) {
    mask_loop(p, smem, br, lane);
  } else if (warp == kWarpStore) {
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        for (int ps = 0; ps < 2; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot3(it);
            uint8_t* X = smem + kOffRing + st * kSlot;
            mbar_wait(&br->staged[st], par3(it));
            if (ps == 0) {
              tma_store_4d(&tdq, X + 2 * kTile, 0, c * kRows, h, b);
            } else {
              tma_store_4d(&tdv, X + 2 * kTile, 0, c * kRows, h, b);
              tma_store_4d(&tdk, X + kTile, 0, c * kRows, h, b);
            }
            bulk_wait_read0();
            mbar_arrive(&br->slot_free[st]);
            TCB_TRACE(7, true);
          }
      }
      tc::store_tail();
    }
  } else {
    const bool splitter = warp < kWarpEpi0;
    const int wq = warp & 3;
    const int t = splitter ? (int)threadIdx.x : (int)threadIdx.x - 32 * kWarpEpi0;
    const float eps = (float)p.eps;
    const float* gS_all = static_cast<const float*>(p.saved_S);
    const uint32_t lane_base = (uint32_t)(32 * wq) << 16;
    const float qnan = __int_as_float(0x7fc00000);
    int it = 0, j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int sl = j & 1;
      const uint32_t* fl = reinterpret_cast<const uint32_t*>(smem + kOffFlags + sl * (kMaxN / 8));
      mbar_wait(&br->fl_full[sl], (j >> 1) & 1);
      const UnitConst uc = ucs[sl];
      for (int k = 0; k < 2 * C; ++k, ++it) {
        const int ps = k >= C, c = ps ? k - C : k;
        const int st = slot3(it);
        uint8_t* X = smem + kOffRing + st * kSlot;
        uint8_t* Y = X + kTile;
        uint8_t* Z = X + 2 * kTile;
        float* inv_st = invs + st * 2 * kRows;
        if (splitter) {  // ---------------- splitter (2 threads per row) ----------------
          if (ps == 0 && c == 0) {
            // this unit's S (saved by the forward) as bf16 hi / lo rows; the previous
            // unit's dQ~ MMAs and G-epilogue (dm) have read its S (op_ready)
            if (j > 0) mbar_wait(&br->op_ready, (j - 1) & 1);
            const int a = t >> 2, q4 = t & 3;  // row a, granules 2 q4, 2 q4 + 1
            // kPair: blockdiag(S, S) — granules 0-3 of rows 0-31 and 4-7 of rows 32-63 hold S
            const bool live = !kPair || (q4 >> 1) == (a >> 5);
            const float4* gs = reinterpret_cast<const float4*>(
                kPair ? gS_all + (int64_t)u * 1024 + (a & 31) * 32 + 16 * (q4 & 1)
                      : gS_all + (int64_t)u * 4096 + a * 64 + 16 * q4);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
              const float4 v0 = live ? __ldg(gs + 2 * q) : z4, v1 = live ? __ldg(gs + 2 * q + 1) : z4;
              const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
              float hi[8], lo[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                hi[e] = __bfloat162float(__float2bfloat16_rn(vv[e]));
                lo[e] = vv[e] - hi[e];
              }
              const uint32_t o = goff(a, 2 * q4 + q);
              *reinterpret_cast<uint4*>(ops + o) = pack8(hi);
              *reinterpret_cast<uint4*>(ops + kStateTile + o) = pack8(lo);
            }
          }
          TCB_TRACE(0, threadIdx.x == 0);
          mbar_wait(&br->raw_full[st], par3(it));
          TCB_TRACE(1, threadIdx.x == 0);
          SplitRow s;
          split_load<kPair>(X, t, s);
          const int r = kPair ? 2 * c * kRows + t : c * kRows + s.row;
          const float iv = rsqrtf(s.ss + eps);
          if (ps == 0) {  // q~ (rows past N: exact zeros in G even for eps = 0)
            const float sc = r < N ? iv : 0.f;
#pragma unroll
            for (int e = 0; e < 32; ++e) s.x[e] *= sc;
          } else {  // k~ masked (padded rows never multiplied in)
            const bool f = r < N && tc::flag_at(fl, r);
#pragma unroll
            for (int e = 0; e < 32; ++e) s.x[e] = f ? s.x[e] * iv : 0.f;
          }
          store_split_half(Z, X, s.row, s.h, s.x);
          if (kPair)
            inv_st[t] = iv;  // 1/norm of row 2 s.row + s.h for the epiloguer's Jacobian
          else if (s.h == 0)
            inv_st[s.row] = iv;
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&br->split_full[st]);
          TCB_TRACE(2, threadIdx.x == 0);
        } else {  // ---------------- epiloguer ----------------
          if (ps == 0 && c == C - 1) {
            // G complete: dm = -ln(n) s <G, S> (:408), dA = s G (:412-413)
            mbar_wait(&br->red_done, j & 1);
            tc_fence_after();
            float dotf = 0.f;
            if (kPair) {  // G = G'00 + G'11; dA operand blockdiag(s G, s G)
              float gr[32];
              pair_combine(tmem, run, reinterpret_cast<float*>(smem + kOffScr), wq, lane, C > kFlush, gr);
              if (wq < 2 && lane < 16) {
                const int a = 16 * wq + lane;
                dotf = dot_state_half(ops, ops + kStateTile, a, 0, gr);  // S row a = op row a, half 0
#pragma unroll
                for (int e = 0; e < 32; ++e) gr[e] *= uc.s;
                store_blockdiag(ops + 2 * kStateTile, ops + 3 * kStateTile, a, gr);
              }
            } else {  // all 128 threads: row a, columns 32 h ..
              const int a = 16 * wq + (lane & 15), h = lane >> 4;
              float gr[32];
              acc_pair(tmem, run, wq, lane, C > kFlush, gr);
              dotf = dot_state_half(ops, ops + kStateTile, a, h, gr);
#pragma unroll
              for (int e = 0; e < 32; ++e) gr[e] *= uc.s;
              store_split_half(ops + 2 * kStateTile, ops + 3 * kStateTile, a, h, gr);
            }
            double dot = (double)dotf;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            if (lane == 0) dm_x[wq] = dot;
            fence_proxy_async();
            tc_fence_before();
            epi_sync();
            if (t == 0) {
              const double dsum = ((dm_x[0] + dm_x[1]) + dm_x[2]) + dm_x[3];
              if (p.dm_unit) p.dm_unit[u] = uc.coef * dsum;
              mbar_arrive(&br->op_ready);
            }
          }
          mbar_wait(&br->mma_done[st], par3(it));
          TCB_TRACE(5, t == 0);
          tc_fence_after();
          if (ps == 0 && c != C - 1 && c % kFlush == kFlush - 1) {  // long N: flush G
            flush_acc(tmem, run, wq, lane, c == kFlush - 1);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&br->acc_free);
          }
          // per half h: its sequence row, 1/norm and g . x~ (kPair: each half is a row;
          // otherwise both halves are one row)
          const int r0 = kPair ? 2 * (c * kRows + t) : c * kRows + t;
          const float iv0 = kPair ? inv_st[2 * t] : inv_st[t];
          const float iv1 = kPair ? inv_st[2 * t + 1] : iv0;
          const uint32_t Dg = tmem + kBuf0 + kBufCols * st + lane_base + (ps == 0 ? 0u : 64u);
          // pr = g . x~ (x~ = hi + lo rebuilt in fp32; g = dQ~ or dK~)
          float pr0 = 0.f, pr1 = 0.f;
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            float g[32], x[32];
            tmem_ld_half(Dg + 32u * h, g);
            load_split_half(Z, X, t, h, x);
            (h == 0 ? pr0 : pr1) = dot32(g, x);
          }
          if (!kPair) pr1 = pr0 = pr0 + pr1;
          if (ps == 0) {
            // dQ_i = (g - (g.q~_i) q~_i) / nq_i, g = s dO S^T (:410-411, :421-428); staged in Z
            // (half h reads and then overwrites only its own granules of row t)
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
              float g[32], x[32];
              tmem_ld_half(Dg + 32u * h, g);
              load_split_half(Z, X, t, h, x);
              const float pr = h ? pr1 : pr0, iv = h ? iv1 : iv0;
#pragma unroll
              for (int e = 0; e < 32; ++e) g[e] = (uc.s * g[e] - uc.s * pr * x[e]) * iv;
              store_half(Z, t, h, g);
            }
          } else {
            const bool f0 = r0 < N && tc::flag_at(fl, r0);
            const bool f1 = kPair ? (r0 + 1 < N && tc::flag_at(fl, r0 + 1)) : f0;
            const bool nan_out = uc.tn == 0;
            // dK_i = v_i ? (g - (g.k~)k~) / nk : 0 (:430-437), staged in Y (V is done)
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
              float g[32], x[32];
              tmem_ld_half(Dg + 32u * h, g);
              load_split_half(Z, X, t, h, x);
              const float pr = h ? pr1 : pr0, iv = h ? iv1 : iv0;
              const bool f = h ? f1 : f0;
#pragma unroll
              for (int e = 0; e < 32; ++e) g[e] = nan_out ? qnan : (f ? (g[e] - pr * x[e]) * iv : 0.f);
              store_half(Y, t, h, g);
            }
            // dV_i = v_i ? (K~ dA)_i : 0 (:416, :439), staged in Z (K~ is done)
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
              float g[32];
              tmem_ld_half(tmem + kBuf0 + kBufCols * st + lane_base + 32u * h, g);
              const bool f = h ? f1 : f0;
#pragma unroll
              for (int e = 0; e < 32; ++e) g[e] = nan_out ? qnan : (f ? g[e] : 0.f);
              store_half(Z, t, h, g);
            }
          }
          arrive_staged(br, st, lane);
          TCB_TRACE(6, t == 0);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&br->fl_empty[sl]);
    }
  }
  if (threadIdx.x == 32 * kWarpEpi0 && p.dm_total) __threadfence();
  teardown(tmem, warp);
  if (p.dm_total) tc::last_cta_dm_total(p, units, smem + kOffRing);
}

}  // namespace tcb

// ---- host side ----------------------------------------------------------------------

// 4-D bf16 map over (D, N, H, B), box (64, 128, 1, 1), 128-byte swizzle; for
// paired rows (d_h = 32, contiguous rows, N even) over (64, N / 2, H, B).
inline bool tcb_pair(const OpParams& p) { return p.D == 32; }
inline bool make_bf16_chunk_map(CUtensorMap* map, const void* base, const OpParams& p) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const bool pair = tcb_pair(p);
  cuuint64_t dims[4] = {64, (cuuint64_t)(pair ? p.N / 2 : p.N), (cuuint64_t)p.H, (cuuint64_t)p.B};
  cuuint64_t strides[3] = {(cuuint64_t)p.sn * 2 * (pair ? 2 : 1), (cuuint64_t)p.sh * 2,
                           (cuuint64_t)p.sb * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)tcb::kRows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline bool tcb_layout_ok(const OpParams& p, std::initializer_list<const void*> ptrs) {
  if (p.N < 1 || p.N > tcb::kMaxN) return false;
  if (p.D == 32) {  // paired rows: [N][32] read as [N/2][64]
    if (p.sn != 32 || (p.N & 1) || getenv("COTTEN_NO_TCB_PAIR")) return false;
  } else if (p.D != 64) {
    return false;
  }
  if ((p.sn * 2) % 16 || (p.sh * 2) % 16 || (p.sb * 2) % 16) return false;
  if (p.B * p.H > (1ll << 31) - 1) return false;
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<uintptr_t>(q) & 15)) return false;
  return encode_fn() != nullptr && getenv("COTTEN_NO_TCB") == nullptr;
}
template <typename T>
inline bool tcb_fwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, __nv_bfloat16>::value) {
    return false;
  } else {
    return tcb_layout_ok(p, {p.q, p.k, p.v, p.out});
  }
}
template <typename T>
inline bool tcb_bwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, __nv_bfloat16>::value) {
    return false;
  } else {
    return p.saved_S != nullptr && tcb_layout_ok(p, {p.q, p.k, p.v, p.dout, p.dq, p.dk, p.dv});
  }
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_tcb_pdl(void (*kern)(KArgs...), int grid, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tcb::kThreads);
  cfg.dynamicSmemBytes = tcb::kSmemBytes;
  cfg.stream = st;
  static const bool pdl = getenv("COTTEN_NO_PDL") == nullptr;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

inline void* tcb_trace_begin(int grid) {
#if COTTEN_TCB_TRACE
  static void* buf = nullptr;
  if (!buf) cudaMalloc(&buf, (size_t)1024 * tcb::kTraceItems * 8 * sizeof(long long));
  cudaMemset(buf, 0, (size_t)grid * tcb::kTraceItems * 8 * sizeof(long long));
  return buf;
#else
  (void)grid;
  return nullptr;
#endif
}
inline void tcb_trace_end(void* buf, int grid, const char* tag, cudaStream_t st) {
#if COTTEN_TCB_TRACE
  const char* dir = getenv("COTTEN_TRACE_DIR");
  if (!dir || !buf) return;
  const size_t n = (size_t)grid * tcb::kTraceItems * 8;
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

inline int launch_tcb_fwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mo;
  if (!make_bf16_chunk_map(&mq, p.q, p) || !make_bf16_chunk_map(&mk, p.k, p) ||
      !make_bf16_chunk_map(&mv, p.v, p) || !make_bf16_chunk_map(&mo, p.out ? p.out : p.q, p))
    return -1;
  auto kern = tcb_pair(p) ? tcb::cos_fwd_tcb_kernel<true> : tcb::cos_fwd_tcb_kernel<false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tcb::kSmemBytes) != cudaSuccess)
    return -1;
  const int grid = std::min((int)(p.B * p.H), sm_count());
  OpParams q = p;
  q.l2_ahead = l2_ahead_items(true, (int)(((tcb_pair(p) ? p.N / 2 : p.N) + tcb::kRows - 1) / tcb::kRows));
  q.workspace = tcb_trace_begin(grid);
  if (launch_tcb_pdl(kern, grid, st, mq, mk, mv, mo, q) != cudaSuccess) return -1;
  tcb_trace_end(q.workspace, grid, "tcb_fwd", st);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}
inline int launch_tcb_bwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mg, mdq, mdk, mdv;
  if (!make_bf16_chunk_map(&mq, p.q, p) || !make_bf16_chunk_map(&mk, p.k, p) ||
      !make_bf16_chunk_map(&mv, p.v, p) || !make_bf16_chunk_map(&mg, p.dout, p) ||
      !make_bf16_chunk_map(&mdq, p.dq, p) || !make_bf16_chunk_map(&mdk, p.dk, p) ||
      !make_bf16_chunk_map(&mdv, p.dv, p))
    return -1;
  auto kern = tcb_pair(p) ? tcb::cos_bwd_tcb_kernel<true> : tcb::cos_bwd_tcb_kernel<false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tcb::kSmemBytes) != cudaSuccess)
    return -1;
  const int grid = std::min((int)(p.B * p.H), sm_count());
  OpParams q = p;
  q.l2_ahead = l2_ahead_items();
  q.workspace = tcb_trace_begin(grid);
  if (launch_tcb_pdl(kern, grid, st, mq, mk, mv, mg, mdq, mdk, mdv, q) != cudaSuccess)
    return -1;
  tcb_trace_end(q.workspace, grid, "tcb_bwd", st);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace cotten
