// Tensor-core (tcgen05 kind::f16) cosine-attention kernels for fp32 inputs,
// head_dim 64, any seq_len up to 16384 — BASELINE config #5's fp32 d_h = 64
// points (north star: "tcgen05/TMEM tiles for the two small contractions ...
// at d_head >= 64"; kernels_rt.cuh is the FP32-pipe A/B partner).
//
// Precision: every fp32 operand x (the normalised rows q~ / k~, the raw V and
// dO, the d x d state S or dA = s G) is split into three bf16 parts
// x = b0 + b1 + b2 (b0 = bf16(x), b1 = bf16(x - b0), b2 = bf16(x - b0 - b1):
// 24 significant bits, the fp32 mantissa), and the MMAs accumulate the six
// products b0 b0' + b0 b1' + b1 b0' + b0 b2' + b2 b0' + b1 b1' in fp32 TMEM;
// the dropped terms are ~2^-24 relative, inside the 1e-5 bar with the fp32
// pipe's margin.  3xTF32 (the d_h = 32 kernels' split) needs 4 x 32 KB of
// fp32 operand tiles per 128-row reduction chunk at d_h = 64 and does not fit
// a 3-deep ring in 227 KB; three bf16 parts of a 64-row chunk are 24 KB per
// tensor and are written over the raw fp32 tile in place (two of them).
//
// 64-row chunks, so every MMA is M = 64 (D row m at TMEM lane (m % 16) +
// 32 (m / 16), measured in scripts/dev/mma_probe_m64.cu):
//   forward   pass 1 (K, V):  S += K~^T V                    (reduction, M = N = 64, K = 16 rows)
//             pass 2 (Q):     O  = s Q~ S                    (row output, M = N = 64, K = 64)
//   backward  pass 1 (Q, dO): G += Q~^T dO,  dQ~ = s dO S^T
//             pass 2 (K, V):  dV = K~ dA,    dK~ = V dA^T    (dA = s G)
// (attention.cpp:297-395, :397-441).  All operands come from shared memory
// (SS MMAs): the bf16 part tiles are 64 rows x 128 B, 128-byte swizzle, and
// one such tile is both the MN-major operand of a reduction and the K-major
// operand of a row output (scripts/dev/mma_probe_bf16.cu), so S and dA are
// stored once each (as three parts).
//
// Ring slot (48 KB): X raw fp32 (two SW128 boxes of 32 columns x 64 rows)
// becomes parts 0 | 1 in place, Y likewise, plus X part 2 and Y part 2.
// Outputs are staged as fp32 boxes over X or Y once the item's MMAs are done.
//
// Head-merged mode (kMerge, fp32 d_h = 32, even H, N <= 64 — the Beauty /
// Steam shape, where a 128-row chunk of the d_h = 32 kernels is 61 % padding):
// heads 2j and 2j + 1 of one sequence ride in the two 32-column boxes of a
// 64-column row (box hb is loaded from head 2j + hb), so one 64-row chunk
// carries both heads' 50 rows.  They share the mask and true_n; each half is
// normalised and differentiated as its own row; the reduction's diagonal
// blocks are S_2j and S_2j+1 (the off-diagonal blocks pair the two heads and
// are discarded), and the state operand is blockdiag(S_2j, S_2j+1).
//
// Warp roles (512 threads): 0-7 splitter (four threads per row, 16 columns
// each; the in-place part writes follow a __syncwarp, since a row's four
// threads share a warp), 8-11 epiloguer (two threads per row: the M = 64
// accumulator's 16 lanes per subpartition are read by 32 threads with
// tcgen05.ld.16x32bx2, thread l >= 16 taking columns 32-63 of lane l - 16;
// scripts/dev/tmem_ld_probe.cu), 12 TMA producer, 13 MMA issuer, 14 mask
// warp, 15 store warp.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels_tcb.cuh"

namespace cotten {
namespace tcf {

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
using tcb::goff;
using tcb::idesc_bf16;
using tcb::mma_bf16;
using tcb::pack2;
using tcb::sdesc;
using tcb::unpack8;

constexpr int kD = 64;
constexpr int kRows = 64;
constexpr uint32_t kBox = 8192;    // 64 rows x 128 B: one fp32 box (32 columns) or one bf16 part
constexpr uint32_t kRaw = 2 * kBox;
constexpr int kRing = 3;
constexpr int kMaxN = 16384;
constexpr int kFlush = 8;  // S / G accumulator flushed every 8 chunks (512 rows, <= 192 MMAs)
constexpr int kSplitWarps = 8, kEpiWarps = 4;
constexpr int kWarpEpi0 = kSplitWarps;
constexpr int kWarpProducer = 12, kWarpMma = 13, kWarpMask = 14, kWarpStore = 15;
constexpr int kThreads = 16 * 32;

// slot: X (raw -> parts 0 | 1) at +0, Y at +16K, X part 2 at +32K, Y part 2 at +40K
constexpr uint32_t kSlot = 2 * kRaw + 2 * kBox;
constexpr uint32_t kOffRing = 0;
constexpr uint32_t kOffOps = kOffRing + kRing * kSlot;   // S parts 0-2, dA parts 0-2
constexpr uint32_t kOffRun = kOffOps + 6 * kBox;         // fp32 running sum, 64 x 64
constexpr uint32_t kOffFlags = kOffRun + 64 * 64 * 4;    // 2 x 2 KB bitmasks
constexpr uint32_t kOffInv = kOffFlags + 2 * (kMaxN / 8);  // per slot 64 x 2 x 1/norm (bwd)
constexpr uint32_t kOffMisc = kOffInv + kRing * 2 * kRows * 4;
constexpr uint32_t kOffBar = kOffMisc + 128;
constexpr uint32_t kSmemBytes = kOffBar + 32 * 8;
static_assert(kSmemBytes <= 227 * 1024, "shared-memory budget");
static_assert((kOffOps % 1024) == 0 && (kOffRun % 1024) == 0, "SW128 tiles are 1024-B aligned");

// TMEM: [0, 64) the S / G accumulator (M = 64); slot b at 64 + 128 b:
// [+0, +64) O | dQ~ | dV, [+64, +128) dK~.
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kBuf0 = 64;
constexpr uint32_t kBufCols = 128;

__device__ __forceinline__ int slot3(int it) { return it % kRing; }
__device__ __forceinline__ uint32_t par3(int it) { return (uint32_t)(it / kRing) & 1u; }

// Unit u of the persistent schedule: sequence b, first head h, and g = b H + h,
// the first head's index in saved_S / dm_unit / saved_norms.  kMerge: a unit
// is the head pair (h, h + 1).
struct UnitPos {
  int b, h, g;
};
template <bool kMerge>
__device__ __forceinline__ UnitPos unit_pos(int u, int H) {
  const int Hs = kMerge ? H >> 1 : H;
  UnitPos o;
  o.b = u / Hs;
  o.h = (u - o.b * Hs) * (kMerge ? 2 : 1);
  o.g = o.b * H + o.h;
  return o;
}
// TMA coordinates (column, head) of 32-column box hb of unit position q
template <bool kMerge>
__device__ __forceinline__ int box_col(int hb) { return kMerge ? 0 : 32 * hb; }
template <bool kMerge>
__device__ __forceinline__ int box_head(const UnitPos& q, int hb) { return kMerge ? q.h + hb : q.h; }

struct Bars {
  uint64_t raw_full[kRing], slot_free[kRing], split_full[kRing], mma_done[kRing], staged[kRing];
  uint64_t op_ready, acc_free, red_done;
  uint64_t fl_full[2], fl_empty[2];
  uint64_t issued;  // the first unit's mask loads are out (kernels_tc.cuh Bars::issued)
};
static_assert(sizeof(Bars) <= 256, "barrier area");

// ---- three-part bf16 split ----------------------------------------------------------
__device__ __forceinline__ uint32_t bf2_bits(__nv_bfloat162 h) { return *reinterpret_cast<uint32_t*>(&h); }
// (x0, x1) -> three packed bf16x2 words: one cvt.rn.bf16x2.f32 per part, the
// unpacking back to fp32 is a shift / mask (bf16 is the top half of an fp32).
__device__ __forceinline__ void split3_pair(float x0, float x1, uint32_t& w0, uint32_t& w1, uint32_t& w2) {
  w0 = bf2_bits(__floats2bfloat162_rn(x0, x1));
  const float r0 = x0 - __uint_as_float(w0 << 16), r1 = x1 - __uint_as_float(w0 & 0xFFFF0000u);  // exact
  w1 = bf2_bits(__floats2bfloat162_rn(r0, r1));
  w2 = bf2_bits(__floats2bfloat162_rn(r0 - __uint_as_float(w1 << 16), r1 - __uint_as_float(w1 & 0xFFFF0000u)));
}
// 8 values -> parts 0-2 at granule j of row `row` of three part tiles
__device__ __forceinline__ void store_parts8(uint8_t* p0, uint8_t* p1, uint8_t* p2, int row, int j,
                                             const float* x) {
  uint32_t a[4], b[4], c[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) split3_pair(x[2 * e], x[2 * e + 1], a[e], b[e], c[e]);
  const uint32_t o = goff(row, j);
  *reinterpret_cast<uint4*>(p0 + o) = make_uint4(a[0], a[1], a[2], a[3]);
  *reinterpret_cast<uint4*>(p1 + o) = make_uint4(b[0], b[1], b[2], b[3]);
  *reinterpret_cast<uint4*>(p2 + o) = make_uint4(c[0], c[1], c[2], c[3]);
}
// parts 0-2 at granule j of row `row` rebuilt in fp32 (b0 + b1 + b2 = x exactly)
__device__ __forceinline__ void load_parts8(const uint8_t* p0, const uint8_t* p1, const uint8_t* p2,
                                            int row, int j, float* x) {
  float a[8], b[8], c[8];
  const uint32_t o = goff(row, j);
  unpack8(*reinterpret_cast<const uint4*>(p0 + o), a);
  unpack8(*reinterpret_cast<const uint4*>(p1 + o), b);
  unpack8(*reinterpret_cast<const uint4*>(p2 + o), c);
#pragma unroll
  for (int e = 0; e < 8; ++e) x[e] = (a[e] + b[e]) + c[e];
}
// fp32 tile row (two boxes): 4-float granule k of box h
__device__ __forceinline__ float4 ld_f4(const uint8_t* tile, int row, int h, int k) {
  return *reinterpret_cast<const float4*>(tile + h * kBox + goff(row, k));
}
__device__ __forceinline__ void st_f4(uint8_t* tile, int row, int h, int k, float4 v) {
  *reinterpret_cast<float4*>(tile + h * kBox + goff(row, k)) = v;
}

// 32 columns of the M = 64 row of this thread's pair: lanes < 16 read columns
// [c, c + 32) of lane 32 wq + l, lanes >= 16 columns [c + 32, c + 64) of lane
// 32 wq + l - 16 (tcgen05.ld.16x32bx2, half-split offset 32 columns).
__device__ __forceinline__ void tmem_ld_pair(uint32_t taddr, float (&r)[32]) {
  uint32_t* u = reinterpret_cast<uint32_t*>(r);
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], 32;"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
        "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
        "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
        "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(taddr));
  tmem_wait_ld();
}

// ---- MMA issue (one thread) -------------------------------------------------------
// The six products (i, j) of x = sum_i x_i and y = sum_j y_j kept by the split:
// (0,0) (0,1) (1,0) (0,2) (2,0) (1,1).
// R (M = N = 64) += x^T y over `ksteps` 16-row groups; x, y = three MN-major part tiles each
__device__ __forceinline__ void issue_reduction(uint32_t d, const uint32_t (&x)[3],
                                                const uint32_t (&y)[3], int ksteps, bool first) {
  const uint32_t id = idesc_bf16(64, 64, true, true);
  for (int kk = 0; kk < ksteps; ++kk)
#pragma unroll
    for (int pr = 0; pr < 6; ++pr) {
      const int i = pr == 0 ? 0 : pr == 1 ? 0 : pr == 2 ? 1 : pr == 3 ? 0 : pr == 4 ? 2 : 1;
      const int j = pr == 0 ? 0 : pr == 1 ? 1 : pr == 2 ? 0 : pr == 3 ? 2 : pr == 4 ? 0 : 1;
      mma_bf16(d, sdesc(x[i] + 2048u * kk, kBox, 1024u), sdesc(y[j] + 2048u * kk, kBox, 1024u), id,
               (first && kk == 0 && pr == 0) ? 0u : 1u);
    }
}
// D (64 x 64) = A (64-row chunk, K-major, K = 64 features) x B (state parts):
// B MN-major (rows = k) for O = Q~ S, dV = K~ dA; K-major (rows = n) for
// dQ~ = dO S^T, dK~ = V dA^T.
template <bool kBMN>
__device__ __forceinline__ void issue_rowout(uint32_t d, const uint32_t (&a)[3], const uint32_t (&b)[3]) {
  const uint32_t id = idesc_bf16(64, 64, false, kBMN);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int pr = 0; pr < 6; ++pr) {
      const int i = pr == 0 ? 0 : pr == 1 ? 0 : pr == 2 ? 1 : pr == 3 ? 0 : pr == 4 ? 2 : 1;
      const int j = pr == 0 ? 0 : pr == 1 ? 1 : pr == 2 ? 0 : pr == 3 ? 2 : pr == 4 ? 0 : 1;
      const uint64_t ad = sdesc(a[i] + 32u * kk, 16u, 1024u);
      const uint64_t bd = kBMN ? sdesc(b[j] + 2048u * kk, kBox, 1024u) : sdesc(b[j] + 32u * kk, 16u, 1024u);
      mma_bf16(d, ad, bd, id, (kk == 0 && pr == 0) ? 0u : 1u);
    }
}

// ---- setup / mask warp ------------------------------------------------------------
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
template <bool kMerge>
__device__ __forceinline__ void mask_loop(const OpParams& p, uint8_t* smem, Bars* br, int lane) {
  UnitConst* ucs = reinterpret_cast<UnitConst*>(smem + kOffMisc);
  const int H = (int)p.H, Hs = kMerge ? H >> 1 : H;
  const int units = (int)p.B * Hs;
  int j = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
    const int sl = j & 1;
    mbar_wait(&br->fl_empty[sl], ((j >> 1) & 1) ^ 1);
    tc::mask_unit(p, u / Hs, reinterpret_cast<uint32_t*>(smem + kOffFlags + sl * (kMaxN / 8)),
                  &ucs[sl], lane, j == 0 ? &br->issued : nullptr);
    __syncwarp();
    if (lane == 0) mbar_arrive(&br->fl_full[sl]);
  }
}
__device__ __forceinline__ void epi_sync() {  // the 4 epiloguer warps
  asm volatile("bar.sync 2, 128;" ::: "memory");
}
__device__ __forceinline__ void arrive_staged(Bars* br, int b, int lane) {
  fence_proxy_async();
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(&br->staged[b]);
}
// Half h of accumulator row a = 16 wq + lane (lanes < 16) + the flushed running
// sum (row a's float4 k at slot k ^ lane: 16 lanes hit 16 different slots).
__device__ __forceinline__ void acc_half(uint32_t tmem, const float* run, int wq, int lane, int h,
                                         bool with_run, float (&r)[32]) {
  tmem_ld32(tmem + ((uint32_t)(32 * wq) << 16) + 32u * h, r);
  tmem_wait_ld();
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
// Half h = lane / 16 (columns 32 h ..) of accumulator row 16 wq + lane % 16 for
// all 32 lanes at once (tcgen05.ld.16x32bx2), plus the flushed running sum:
// the per-unit S / G epilogue runs on all 128 epiloguer threads.
__device__ __forceinline__ void acc_pair(uint32_t tmem, const float* run, int wq, int lane,
                                         bool with_run, float (&r)[32]) {
  tmem_ld_pair(tmem + ((uint32_t)(32 * wq) << 16), r);
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
// Half h (32 columns) of row a of a state as its three part tiles.
__device__ __forceinline__ void store_state_half(uint8_t* ops3, int a, int h, const float (&x)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) store_parts8(ops3, ops3 + kBox, ops3 + 2 * kBox, a, 4 * h + q, x + 8 * q);
}

// Splitter: four threads per chunk row (16 columns each: fp32 box q / 2,
// granules 4 (q % 2) .. +3); the row's squared norm is the sum over the quad.
// Threads q = 2, 3 walk their granules starting at the third: an LDS.128 is
// served 8 lanes (two rows) per wavefront, and in natural order lanes q and
// q + 2 of a row would hit the same bank group of the two boxes (2-way
// conflicts, measured); rotated, the 8 lanes cover all 8 bank groups.  x[]
// then holds columns 8-15 before 0-7 for q >= 2 (split_store undoes it).
struct SplitRow {
  int row, q;
  float x[16];
  float ss;  // |row|^2
};
template <bool kMerge = false>
__device__ __forceinline__ void split_load(const uint8_t* X, int t, SplitRow& s, bool norm) {
  s.row = t >> 2;
  s.q = t & 3;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 v = ld_f4(X, s.row, s.q >> 1, 4 * (s.q & 1) + ((k + 2 * (s.q >> 1)) & 3));
    s.x[4 * k] = v.x;
    s.x[4 * k + 1] = v.y;
    s.x[4 * k + 2] = v.z;
    s.x[4 * k + 3] = v.w;
  }
  if (norm) {
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int e = 0; e < 16; e += 2) {
      a = fmaf(s.x[e], s.x[e], a);
      b = fmaf(s.x[e + 1], s.x[e + 1], b);
    }
    float part = a + b;
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    // kMerge: threads q = 0, 1 hold head h's row, q = 2, 3 head h + 1's
    s.ss = kMerge ? part : part + __shfl_xor_sync(0xffffffffu, part, 2);
  }
}
// The split row's 16 values as parts over its own raw tile: part 0 over box 0,
// part 1 over box 1 (granules 2q, 2q + 1 of the 128-B bf16 row), part 2 into
// P2.  Call after a __syncwarp that follows every split_load of the warp.
__device__ __forceinline__ void split_store(uint8_t* X, uint8_t* P2, const SplitRow& s) {
  const int sw = s.q >> 1;  // rotated load order (split_load)
  store_parts8(X, X + kBox, P2, s.row, 2 * s.q + sw, s.x);
  store_parts8(X, X + kBox, P2, s.row, 2 * s.q + 1 - sw, s.x + 8);
}

// ======================================================================================
// Forward
// ======================================================================================
template <bool kMerge>
__global__ void __launch_bounds__(kThreads, 1) cos_fwd_tcf_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap to,
    const OpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = (int)p.N, H = (int)p.H;
  const int units = (int)p.B * (kMerge ? H >> 1 : H);
  const int C = (N + kRows - 1) / kRows;
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
        const UnitPos up = unit_pos<kMerge>(u, H);
        for (int ps = 0; ps < P; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot3(it);
            if (COTTEN_ISSUED_GATE && it == 0) mbar_wait(&br->issued, 0);  // mask loads go first
            tc::ItemPos f;
            if (!kMerge && p.l2_ahead && tc::item_pos(it + p.l2_ahead, P, C, units, H, f))
              for (int hb = 0; hb < 2; ++hb) {  // L2 prefetch of a later item (long N)
                tc::tma_prefetch_4d(f.ps == 0 ? &tk : &tq, 32 * hb, f.c * kRows, f.h, f.b);
                if (f.ps == 0) tc::tma_prefetch_4d(&tv, 32 * hb, f.c * kRows, f.h, f.b);
              }
            mbar_wait(&br->slot_free[st], par3(it) ^ 1u);
            uint8_t* X = smem + kOffRing + st * kSlot;
            if (ps == 0) {
              mbar_expect_tx(&br->raw_full[st], 2 * kRaw);
              for (int hb = 0; hb < 2; ++hb) {
                tma_load_4d(X + hb * kBox, &tk, box_col<kMerge>(hb), c * kRows, box_head<kMerge>(up, hb), up.b,
                            &br->raw_full[st]);
                tma_load_4d(X + kRaw + hb * kBox, &tv, box_col<kMerge>(hb), c * kRows, box_head<kMerge>(up, hb),
                            up.b, &br->raw_full[st]);
              }
            } else {
              mbar_expect_tx(&br->raw_full[st], kRaw);
              for (int hb = 0; hb < 2; ++hb)
                tma_load_4d(X + hb * kBox, &tq, box_col<kMerge>(hb), c * kRows, box_head<kMerge>(up, hb), up.b,
                            &br->raw_full[st]);
            }
          }
      }
    }
  } else if (warp == kWarpMma) {
    int it = 0, j = 0, nflush = 0;
    const uint32_t base = smem_u32(smem);
    const uint32_t opS[3] = {base + kOffOps, base + kOffOps + kBox, base + kOffOps + 2 * kBox};
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      for (int ps = 0; ps < P; ++ps)
        for (int c = 0; c < C; ++c, ++it) {
          const int st = slot3(it);
          mbar_wait(&br->split_full[st], par3(it));
          if (ps == 0 && c == 0 && P == 1 && j > 0) mbar_wait(&br->op_ready, (j - 1) & 1);
          if (ps == 0 && c > 0 && c % kFlush == 0) mbar_wait(&br->acc_free, (nflush++) & 1);
          if (ps == 1 && c == 0) mbar_wait(&br->op_ready, j & 1);
          tc_fence_after();
          const uint32_t X = base + kOffRing + st * kSlot;
          const uint32_t xp[3] = {X, X + kBox, X + 2 * kRaw};
          const uint32_t yp[3] = {X + kRaw, X + kRaw + kBox, X + 2 * kRaw + kBox};
          if (elect_one()) {
            if (ps == 0) {  // S += K~^T V (attention.cpp:345-353)
              const int ks = (min(kRows, N - c * kRows) + 15) >> 4;
              issue_reduction(tmem, xp, yp, ks, c % kFlush == 0);
            } else {  // O = Q~ S (:379-387)
              issue_rowout<true>(tmem + kBuf0 + kBufCols * st, xp, opS);
            }
            mma_commit(&br->mma_done[st]);
          }
          __syncwarp();
        }
    }
  } else if (warp == kWarpMask) {
    mask_loop<kMerge>(p, smem, br, lane);
  } else if (warp == kWarpStore) {
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const UnitPos up = unit_pos<kMerge>(u, H);
        for (int ps = 0; ps < P; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot3(it);
            mbar_wait(&br->staged[st], par3(it));
            if (ps == 1 && p.out) {  // O staged over Y (free in pass 2)
              uint8_t* Y = smem + kOffRing + st * kSlot + kRaw;
              tma_store_4d(&to, Y, box_col<kMerge>(0), c * kRows, box_head<kMerge>(up, 0), up.b);
              tma_store_4d(&to, Y + kBox, box_col<kMerge>(1), c * kRows, box_head<kMerge>(up, 1), up.b);
              bulk_wait_read0();
            }
            mbar_arrive(&br->slot_free[st]);
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
      const UnitPos up = unit_pos<kMerge>(u, H);
      mbar_wait(&br->fl_full[sl], (j >> 1) & 1);
      const UnitConst uc = ucs[sl];
      for (int k = 0; k < P * C; ++k, ++it) {
        const int ps = k >= C, c = ps ? k - C : k;
        const int st = slot3(it);
        uint8_t* X = smem + kOffRing + st * kSlot;
        uint8_t* Y = X + kRaw;
        if (splitter) {  // ---------------- splitter (4 threads per row) ----------------
          mbar_wait(&br->raw_full[st], par3(it));
          SplitRow s;
          split_load<kMerge>(X, t, s, true);
          const int r = c * kRows + s.row;
          const float iv = rsqrtf(s.ss + eps);
          // this thread's head (kMerge: q = 2, 3 hold the second head) and its saved norms
          float* norms = norms_all && r < N && (s.q & (kMerge ? 1 : 3)) == 0
                             ? norms_all + (int64_t)(up.g + (kMerge ? s.q >> 1 : 0)) * 2 * N
                             : nullptr;
          if (ps == 0) {  // k~ masked (attention.cpp:334-343), V as it is
            const bool f = r < N && tc::flag_at(fl, r);
            if (norms) norms[N + r] = f ? (s.ss + eps) * iv : 1.0f;
#pragma unroll
            for (int e = 0; e < 16; ++e) s.x[e] = f ? s.x[e] * iv : 0.f;  // NaN-safe zeros
            SplitRow v;
            split_load(Y, t, v, false);
            __syncwarp();
            split_store(X, X + 2 * kRaw, s);
            split_store(Y, X + 2 * kRaw + kBox, v);
          } else {  // q~ every row (:366-377)
            if (norms) norms[r] = (s.ss + eps) * iv;
#pragma unroll
            for (int e = 0; e < 16; ++e) s.x[e] *= iv;
            __syncwarp();
            split_store(X, X + 2 * kRaw, s);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&br->split_full[st]);
        } else {  // ---------------- epiloguer (2 threads per row) ----------------
          mbar_wait(&br->mma_done[st], par3(it));
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
            if (c == C - 1) {  // S complete: saved S + its three part tiles (all 128 threads)
              const int a = 16 * wq + (lane & 15), h = lane >> 4;  // row a, columns 32 h ..
              float sv[32];
              acc_pair(tmem, run, wq, lane, C > kFlush, sv);
              if (kMerge) {  // the two heads' S: diagonal blocks, operand blockdiag
                const bool live = h == (a >> 5);  // rows 0-31: first head (columns 0-31), 32-63: second
                if (live && gS_all) {
                  float4* gs = reinterpret_cast<float4*>(gS_all + (int64_t)(up.g + h) * 1024 + (a & 31) * 32);
#pragma unroll
                  for (int e = 0; e < 8; ++e)
                    gs[e] = make_float4(sv[4 * e], sv[4 * e + 1], sv[4 * e + 2], sv[4 * e + 3]);
                }
                if (!live) {
#pragma unroll
                  for (int e = 0; e < 32; ++e) sv[e] = 0.f;
                }
              } else if (gS_all) {
                float4* gs = reinterpret_cast<float4*>(gS_all + (int64_t)u * 4096 + a * 64 + 32 * h);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  gs[e] = make_float4(sv[4 * e], sv[4 * e + 1], sv[4 * e + 2], sv[4 * e + 3]);
              }
              store_state_half(ops, a, h, sv);
            }
            if (c == C - 1) {
              fence_proxy_async();
              tc_fence_before();
              epi_sync();
              if (t == 0) mbar_arrive(&br->op_ready);
            }
          } else {  // O rows = s (Q~ S), staged over Y as two fp32 boxes
            const int row = 16 * wq + (lane & 15), h = lane >> 4;
            float o[32];
            tmem_ld_pair(tmem + kBuf0 + kBufCols * st + lane_base, o);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              st_f4(Y, row, h, k, make_float4(o[4 * k] * uc.s, o[4 * k + 1] * uc.s, o[4 * k + 2] * uc.s,
                                              o[4 * k + 3] * uc.s));
            arrive_staged(br, st, lane);
          }
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
template <bool kMerge>
__global__ void __launch_bounds__(kThreads, 1) cos_bwd_tcf_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
    const __grid_constant__ CUtensorMap tdq, const __grid_constant__ CUtensorMap tdk,
    const __grid_constant__ CUtensorMap tdv, const OpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = (int)p.N, H = (int)p.H;
  const int units = (int)p.B * (kMerge ? H >> 1 : H);
  const int C = (N + kRows - 1) / kRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Bars* br = reinterpret_cast<Bars*>(smem + kOffBar);
  UnitConst* ucs = reinterpret_cast<UnitConst*>(smem + kOffMisc);
  double* dm_x = reinterpret_cast<double*>(smem + kOffMisc + 40);
  uint8_t* ops = smem + kOffOps;  // S parts at +0, dA parts at +3 kBox
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
      // one unit's saved S (kMerge: the two heads' S, contiguous)
      const uint32_t sbytes = (uint32_t)(kMerge ? 2 * 32 * 32 * 4 : 64 * 64 * 4);
      const uint8_t* gS = static_cast<const uint8_t*>(p.saved_S);
      if (blockIdx.x < units) tc::bulk_prefetch_l2(gS + (int64_t)unit_pos<kMerge>(blockIdx.x, H).g * (kMerge ? 4096 : 16384), sbytes);
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const UnitPos up = unit_pos<kMerge>(u, H);
        // the splitter loads the next unit's S at its first chunk: have it in L2
        if (u + (int)gridDim.x < units)
          tc::bulk_prefetch_l2(gS + (int64_t)unit_pos<kMerge>(u + gridDim.x, H).g * (kMerge ? 4096 : 16384), sbytes);
        for (int ps = 0; ps < 2; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot3(it);
            if (COTTEN_ISSUED_GATE && it == 0) mbar_wait(&br->issued, 0);  // mask loads go first
            mbar_wait(&br->slot_free[st], par3(it) ^ 1u);
            uint8_t* X = smem + kOffRing + st * kSlot;
            mbar_expect_tx(&br->raw_full[st], 2 * kRaw);
            for (int hb = 0; hb < 2; ++hb) {
              tma_load_4d(X + hb * kBox, ps == 0 ? &tq : &tk, box_col<kMerge>(hb), c * kRows,
                          box_head<kMerge>(up, hb), up.b, &br->raw_full[st]);
              tma_load_4d(X + kRaw + hb * kBox, ps == 0 ? &tdo : &tv, box_col<kMerge>(hb), c * kRows,
                          box_head<kMerge>(up, hb), up.b, &br->raw_full[st]);
            }
          }
      }
    }
  } else if (warp == kWarpMma) {
    int it = 0, j = 0, nflush = 0;
    const uint32_t base = smem_u32(smem);
    const uint32_t opS[3] = {base + kOffOps, base + kOffOps + kBox, base + kOffOps + 2 * kBox};
    const uint32_t opA[3] = {base + kOffOps + 3 * kBox, base + kOffOps + 4 * kBox,
                             base + kOffOps + 5 * kBox};
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      for (int ps = 0; ps < 2; ++ps)
        for (int c = 0; c < C; ++c, ++it) {
          const int st = slot3(it);
          mbar_wait(&br->split_full[st], par3(it));
          if (ps == 1 && c == 0) mbar_wait(&br->op_ready, j & 1);
          if (ps == 0 && c > 0 && c % kFlush == 0) mbar_wait(&br->acc_free, (nflush++) & 1);
          tc_fence_after();
          const uint32_t X = base + kOffRing + st * kSlot;
          const uint32_t xp[3] = {X, X + kBox, X + 2 * kRaw};
          const uint32_t yp[3] = {X + kRaw, X + kRaw + kBox, X + 2 * kRaw + kBox};
          const uint32_t D = tmem + kBuf0 + kBufCols * st;
          if (elect_one()) {
            if (ps == 0) {
              // G += Q~^T dO (attention.cpp:405)
              const int ks = (min(kRows, N - c * kRows) + 15) >> 4;
              issue_reduction(tmem, xp, yp, ks, c % kFlush == 0);
              // dQ~ (unscaled) = dO S^T (:410-411): A = dO, B row n = S row n
              issue_rowout<false>(D, yp, opS);
              // G complete, and every MMA that reads this unit's S parts
              if (c == C - 1) mma_commit(&br->red_done);
            } else {
              issue_rowout<true>(D, xp, opA);        // dV = K~ dA (:416)
              issue_rowout<false>(D + 64, yp, opA);  // dK~ = V dA^T (:415)
            }
            mma_commit(&br->mma_done[st]);
          }
          __syncwarp();
        }
    }
  } else if (warp == kWarpMask) {
    mask_loop<kMerge>(p, smem, br, lane);
  } else if (warp == kWarpStore) {
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const UnitPos up = unit_pos<kMerge>(u, H);
        for (int ps = 0; ps < 2; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot3(it);
            uint8_t* X = smem + kOffRing + st * kSlot;
            mbar_wait(&br->staged[st], par3(it));
            for (int hb = 0; hb < 2; ++hb) {
              const int bc = box_col<kMerge>(hb), bh = box_head<kMerge>(up, hb);
              if (ps == 0) {
                tma_store_4d(&tdq, X + hb * kBox, bc, c * kRows, bh, up.b);
              } else {
                tma_store_4d(&tdk, X + hb * kBox, bc, c * kRows, bh, up.b);
                tma_store_4d(&tdv, X + kRaw + hb * kBox, bc, c * kRows, bh, up.b);
              }
            }
            bulk_wait_read0();
            mbar_arrive(&br->slot_free[st]);
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
      const UnitPos up = unit_pos<kMerge>(u, H);
      mbar_wait(&br->fl_full[sl], (j >> 1) & 1);
      const UnitConst uc = ucs[sl];
      for (int k = 0; k < 2 * C; ++k, ++it) {
        const int ps = k >= C, c = ps ? k - C : k;
        const int st = slot3(it);
        uint8_t* X = smem + kOffRing + st * kSlot;
        uint8_t* Y = X + kRaw;
        uint8_t* X2 = X + 2 * kRaw;
        uint8_t* Y2 = X2 + kBox;
        float* inv_st = invs + st * 2 * kRows;  // [row][half] (kMerge: one per head)
        if (splitter) {  // ---------------- splitter (4 threads per row) ----------------
          if (ps == 0 && c == 0) {
            // this unit's S (saved by the forward) as three part tiles; the previous
            // unit's dQ~ MMAs and G-epilogue (dm) have read its S (op_ready)
            if (j > 0) mbar_wait(&br->op_ready, (j - 1) & 1);
            const int a = t >> 2, q4 = t & 3;  // row a, columns 16 q4 .. 16 q4 + 15
            // kMerge: blockdiag(S_h, S_h+1) — columns 0-31 of rows 0-31 and 32-63 of rows 32-63
            const bool live = !kMerge || (q4 >> 1) == (a >> 5);
            const float4* gs = reinterpret_cast<const float4*>(
                kMerge ? gS_all + (int64_t)(up.g + (a >> 5)) * 1024 + (a & 31) * 32 + 16 * (q4 & 1)
                       : gS_all + (int64_t)u * 4096 + a * 64 + 16 * q4);
            float vv[16];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float4 v = live ? __ldg(gs + e) : make_float4(0.f, 0.f, 0.f, 0.f);
              vv[4 * e] = v.x;
              vv[4 * e + 1] = v.y;
              vv[4 * e + 2] = v.z;
              vv[4 * e + 3] = v.w;
            }
            store_parts8(ops, ops + kBox, ops + 2 * kBox, a, 2 * q4, vv);
            store_parts8(ops, ops + kBox, ops + 2 * kBox, a, 2 * q4 + 1, vv + 8);
          }
          mbar_wait(&br->raw_full[st], par3(it));
          SplitRow s, y;
          split_load<kMerge>(X, t, s, true);
          split_load(Y, t, y, false);
          const int r = c * kRows + s.row;
          const float iv = rsqrtf(s.ss + eps);
          if (ps == 0) {  // q~ (rows past N: exact zeros in G even for eps = 0)
            const float sc = r < N ? iv : 0.f;
#pragma unroll
            for (int e = 0; e < 16; ++e) s.x[e] *= sc;
          } else {  // k~ masked (padded rows never multiplied in)
            const bool f = r < N && tc::flag_at(fl, r);
#pragma unroll
            for (int e = 0; e < 16; ++e) s.x[e] = f ? s.x[e] * iv : 0.f;
          }
          if ((s.q & (kMerge ? 1 : 3)) == 0) inv_st[2 * s.row + (s.q >> 1)] = iv;  // for the Jacobian
          __syncwarp();
          split_store(X, X2, s);
          split_store(Y, Y2, y);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&br->split_full[st]);
        } else {  // ---------------- epiloguer (2 threads per row) ----------------
          if (ps == 0 && c == C - 1) {
            // G complete: dm = -ln(n) s <G, S> (:408), dA = s G (:412-413)
            mbar_wait(&br->red_done, j & 1);
            tc_fence_after();
            float dotf = 0.f;
            {
              // all 128 threads: row a, columns 32 h ..; kMerge: only the diagonal
              // blocks (rows 0-31 x columns 0-31: the first head's G, rows 32-63 x
              // columns 32-63: the second's); the operand is blockdiag(s G_h, s G_h+1)
              const int a = 16 * wq + (lane & 15), h = lane >> 4;
              const bool live = !kMerge || h == (a >> 5);
              float gr[32];
              acc_pair(tmem, run, wq, lane, C > kFlush, gr);
              if (!live) {
#pragma unroll
                for (int e = 0; e < 32; ++e) gr[e] = 0.f;
              }
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float sv[8];
                load_parts8(ops, ops + kBox, ops + 2 * kBox, a, 4 * h + q, sv);
#pragma unroll
                for (int e = 0; e < 8; ++e) dotf = fmaf(gr[8 * q + e], sv[e], dotf);
              }
#pragma unroll
              for (int e = 0; e < 32; ++e) gr[e] *= uc.s;
              store_state_half(ops + 3 * kBox, a, h, gr);
            }
            double dot = (double)dotf;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            if (lane == 0) dm_x[wq] = dot;
            fence_proxy_async();
            tc_fence_before();
            epi_sync();
            if (t == 0) {
              if (kMerge) {  // one dm per head: warps 0-1 hold the first head's rows
                if (p.dm_unit) {
                  p.dm_unit[up.g] = uc.coef * (dm_x[0] + dm_x[1]);
                  p.dm_unit[up.g + 1] = uc.coef * (dm_x[2] + dm_x[3]);
                }
              } else {
                const double dsum = ((dm_x[0] + dm_x[1]) + dm_x[2]) + dm_x[3];
                if (p.dm_unit) p.dm_unit[u] = uc.coef * dsum;
              }
              mbar_arrive(&br->op_ready);
            }
          }
          mbar_wait(&br->mma_done[st], par3(it));
          tc_fence_after();
          if (ps == 0 && c != C - 1 && c % kFlush == kFlush - 1) {  // long N: flush G
            flush_acc(tmem, run, wq, lane, c == kFlush - 1);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&br->acc_free);
          }
          const int row = 16 * wq + (lane & 15), h = lane >> 4;
          const int r = c * kRows + row;
          const float iv = inv_st[2 * row + (kMerge ? h : 0)];
          const uint32_t D = tmem + kBuf0 + kBufCols * st + lane_base;
          // g = dQ~ or dK~ (this thread's 32 columns), x~ = the part tiles rebuilt
          float g[32], x[32];
          tmem_ld_pair(D + (ps == 0 ? 0u : 64u), g);
#pragma unroll
          for (int q = 0; q < 4; ++q) load_parts8(X, X + kBox, X2, row, 4 * h + q, x + 8 * q);
          float pr = 0.f;
#pragma unroll
          for (int e = 0; e < 32; ++e) pr = fmaf(g[e], x[e], pr);
          const float pr_other = __shfl_xor_sync(0xffffffffu, pr, 16);  // the row's other half
          if (!kMerge) pr += pr_other;  // kMerge: each half is its own head's row
          __syncwarp();  // both halves have read the parts of X before they are overwritten
          if (ps == 0) {
            // dQ_i = (g - (g.q~_i) q~_i) / nq_i, g = s dO S^T (:410-411, :421-428); staged over X
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              float4 v;
              v.x = (uc.s * g[4 * k] - uc.s * pr * x[4 * k]) * iv;
              v.y = (uc.s * g[4 * k + 1] - uc.s * pr * x[4 * k + 1]) * iv;
              v.z = (uc.s * g[4 * k + 2] - uc.s * pr * x[4 * k + 2]) * iv;
              v.w = (uc.s * g[4 * k + 3] - uc.s * pr * x[4 * k + 3]) * iv;
              st_f4(X, row, h, k, v);
            }
          } else {
            const bool f = r < N && tc::flag_at(fl, r);
            const bool nan_out = uc.tn == 0;
            // dK_i = v_i ? (g - (g.k~)k~) / nk : 0 (:430-437), staged over X
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              float4 v;
              v.x = nan_out ? qnan : (f ? (g[4 * k] - pr * x[4 * k]) * iv : 0.f);
              v.y = nan_out ? qnan : (f ? (g[4 * k + 1] - pr * x[4 * k + 1]) * iv : 0.f);
              v.z = nan_out ? qnan : (f ? (g[4 * k + 2] - pr * x[4 * k + 2]) * iv : 0.f);
              v.w = nan_out ? qnan : (f ? (g[4 * k + 3] - pr * x[4 * k + 3]) * iv : 0.f);
              st_f4(X, row, h, k, v);
            }
            // dV_i = v_i ? (K~ dA)_i : 0 (:416, :439), staged over Y (V's parts are done)
            tmem_ld_pair(D, g);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              float4 v;
              v.x = nan_out ? qnan : (f ? g[4 * k] : 0.f);
              v.y = nan_out ? qnan : (f ? g[4 * k + 1] : 0.f);
              v.z = nan_out ? qnan : (f ? g[4 * k + 2] : 0.f);
              v.w = nan_out ? qnan : (f ? g[4 * k + 3] : 0.f);
              st_f4(Y, row, h, k, v);
            }
          }
          arrive_staged(br, st, lane);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&br->fl_empty[sl]);
    }
  }
  if (threadIdx.x == 32 * kWarpEpi0 && p.dm_total) __threadfence();
  teardown(tmem, warp);
  if (p.dm_total) tc::last_cta_dm_total(p, (int)(p.B * p.H), smem + kOffRing);
}

}  // namespace tcf

// ---- host side ----------------------------------------------------------------------

// 4-D fp32 map over (D, N, H, B), box (32, 64, 1, 1), 128-byte swizzle
// (d_h = 64: two boxes per row; head-merged d_h = 32: one box per head).
inline bool tcf_merge(const OpParams& p) { return p.D == 32; }
inline bool make_tcf_map(CUtensorMap* map, const void* base, const OpParams& p) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)p.D, (cuuint64_t)p.N, (cuuint64_t)p.H, (cuuint64_t)p.B};
  cuuint64_t strides[3] = {(cuuint64_t)p.sn * 4, (cuuint64_t)p.sh * 4, (cuuint64_t)p.sb * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)tcf::kRows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
inline bool tcf_layout_ok(const OpParams& p, std::initializer_list<const void*> ptrs) {
  if (p.N < 1 || p.N > tcf::kMaxN) return false;
  if (p.D == 32) {  // head-merged: short sequences (one 64-row chunk holds both heads' rows)
    if (p.N > tcf::kRows || (p.H & 1) || getenv("COTTEN_NO_TCF_MERGE")) return false;
  } else if (p.D != 64) {
    return false;
  }
  if ((p.sn * 4) % 16 || (p.sh * 4) % 16 || (p.sb * 4) % 16) return false;
  if (p.B * p.H > (1ll << 31) - 1) return false;
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<uintptr_t>(q) & 15)) return false;
  return encode_fn() != nullptr && getenv("COTTEN_NO_TCF") == nullptr;
}
template <typename T>
inline bool tcf_fwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, float>::value) {
    return false;
  } else {
    return tcf_layout_ok(p, {p.q, p.k, p.v, p.out});
  }
}
template <typename T>
inline bool tcf_bwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, float>::value) {
    return false;
  } else {
    return p.saved_S != nullptr && tcf_layout_ok(p, {p.q, p.k, p.v, p.dout, p.dq, p.dk, p.dv});
  }
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_tcf_pdl(void (*kern)(KArgs...), int grid, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tcf::kThreads);
  cfg.dynamicSmemBytes = tcf::kSmemBytes;
  cfg.stream = st;
  static const bool pdl = getenv("COTTEN_NO_PDL") == nullptr;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
inline int launch_tcf_fwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mo;
  if (!make_tcf_map(&mq, p.q, p) || !make_tcf_map(&mk, p.k, p) || !make_tcf_map(&mv, p.v, p) ||
      !make_tcf_map(&mo, p.out ? p.out : p.q, p))
    return -1;
  auto kern = tcf_merge(p) ? tcf::cos_fwd_tcf_kernel<true> : tcf::cos_fwd_tcf_kernel<false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tcf::kSmemBytes) !=
      cudaSuccess)
    return -1;
  const int grid = std::min((int)(p.B * p.H / (tcf_merge(p) ? 2 : 1)), sm_count());
  OpParams q = p;
  q.l2_ahead = l2_ahead_items(true, (int)((p.N + tcf::kRows - 1) / tcf::kRows));
  if (launch_tcf_pdl(kern, grid, st, mq, mk, mv, mo, q) != cudaSuccess) return -1;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}
inline int launch_tcf_bwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mg, mdq, mdk, mdv;
  if (!make_tcf_map(&mq, p.q, p) || !make_tcf_map(&mk, p.k, p) || !make_tcf_map(&mv, p.v, p) ||
      !make_tcf_map(&mg, p.dout, p) || !make_tcf_map(&mdq, p.dq, p) || !make_tcf_map(&mdk, p.dk, p) ||
      !make_tcf_map(&mdv, p.dv, p))
    return -1;
  auto kern = tcf_merge(p) ? tcf::cos_bwd_tcf_kernel<true> : tcf::cos_bwd_tcf_kernel<false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tcf::kSmemBytes) !=
      cudaSuccess)
    return -1;
  const int grid = std::min((int)(p.B * p.H / (tcf_merge(p) ? 2 : 1)), sm_count());
  if (launch_tcf_pdl(kern, grid, st, mq, mk, mv, mg, mdq, mdk, mdv, p) != cudaSuccess)
    return -1;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace cotten
