// Tensor-core (tcgen05 kind::f16) cosine-attention kernels for bf16 inputs,
// head_dim 128, any seq_len up to 16384 — BASELINE config #5's bf16 d_h = 128
// points, which the FP32-pipe kernels (kernels_rt.cuh, the A/B partner) serve
// at 0.05-0.06 of HBM.
//
// Arithmetic as kernels_tcb.cuh (bf16 in HBM, fp32 everywhere else): the
// normalised rows q~ / k~ and the 128 x 128 state (S, dA = s G) enter the MMAs
// as bf16 hi / lo pairs, V and dO as they are; products hi*hi + hi*lo + lo*hi
// (or hi + lo against a bf16 operand) accumulate in fp32 TMEM.
//
// Why the d_h = 64 design does not carry over: a 128 x 128 state is 64 KB as
// hi / lo and its fp32 running sum another 64 KB, and 128-row chunks of two
// 256-B-row tensors are 96 KB per ring slot.  So here:
//  * 64-row chunks: a row tile is 64 rows x 256 B = two SW128 half-tiles
//    (features 0-63 | 64-127, 8 KB each); a ring slot holds X, Y (raw) and Z
//    (q~ / k~ hi, later the staging of the chunk's outputs): 48 KB, 3 slots.
//  * Reductions are M = N = 128 (TMEM lane = state row), K = 16 rows per MMA;
//    row outputs are M = 64 (row m at TMEM lane (m % 16) + 32 (m / 16)),
//    N = 128, K = 128 (descriptors measured in scripts/dev/mma_probe_d128.cu).
//  * The fp32 running sum of S / G lives in TMEM (flushed every 8 chunks by
//    tcgen05.ld / st), not in shared memory.
//  * One 64 KB state area: S in the forward; in the backward S during pass 1,
//    then dA = s G written over it in place by the G-epilogue (each thread
//    reads S and writes dA at the same positions), and the next unit's S only
//    after the last MMA reading dA has completed (ops_free).
//  * TMEM: [0, 128) S / G accumulator, [128, 256) running sum, two 128-column
//    output buffers [256, 384) and [384, 512) taken in turn by the row-output
//    jobs (O; dQ~), each released by the epiloguer (out_free).  The backward's
//    pass 2 (dV and dK~ per item) also borrows the accumulator and running-sum
//    columns, idle until the next unit's G: its items alternate between the
//    buffer pairs (out 0, out 1) and (acc, run), so the MMAs of one item run
//    while the epiloguer drains the previous one.
// Shared memory 213 KB; 512 threads: 0-7 splitter (four threads per row, 32
// columns each, granule order rotated for threads 2-3 so that an 8-lane
// LDS.128 phase covers all 8 bank groups), 8-11 epiloguer, 12 TMA producer,
// 13 MMA issuer, 14 mask warp, 15 store warp.
//   forward   pass 1 (K, V):  S += (Z + X)^T Y                      (attention.cpp:345-353)
//             pass 2 (Q):     O = s (Z + X) S                       (:379-387)
//   backward  pass 1 (Q, dO): G += (Z + X)^T Y,  dQ~ = s Y S^T      (:405, :410-411)
//             pass 2 (K, V):  dV = (Z + X) dA,   dK~ = Y dA^T       (:412-416)
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels_tcf.cuh"

namespace cotten {
namespace tch {

using d32::mbar_arrive;
using d32::mbar_expect_tx;
using d32::mbar_init;
using d32::mbar_wait;
using d32::smem_u32;
using d32::tma_load_4d;
using tc::bulk_wait_read0;
using tc::elect_one;
using tc::fence_proxy_async;
using tc::mma_commit;
using tc::tc_fence_after;
using tc::tc_fence_before;
using tc::tma_store_4d;
using tc::tmem_ld32;
using tc::tmem_st32;
using tc::tmem_wait_ld;
using tc::tmem_wait_st;
using tc::UnitConst;
using tcb::dot32;
using tcb::goff;
using tcb::idesc_bf16;
using tcb::load_split_half;
using tcb::mma_bf16;
using tcb::pack2;
using tcb::sdesc;
using tcb::store_half;
using tcb::store_split_half;
using tcb::unpack8;
using tcf::tmem_ld_pair;

constexpr int kD = 128;
constexpr int kRows = 64;
constexpr uint32_t kHalf = 8192;                 // 64 rows x 128 B (one TMA box of 64 bf16)
constexpr uint32_t kTile = 2 * kHalf;            // a 64-row chunk of one tensor
constexpr uint32_t kStateHalf = 16384;           // 128 state rows x 128 B
constexpr uint32_t kStateTile = 2 * kStateHalf;  // 128 x 128 bf16
constexpr int kRing = 3;
constexpr int kMaxN = 16384;
constexpr int kFlush = 8;  // S / G accumulator flushed into the running sum every 8 chunks (512 rows)
constexpr int kSplitWarps = 8, kEpiWarps = 4;
constexpr int kWarpEpi0 = kSplitWarps;
constexpr int kWarpProducer = 12, kWarpMma = 13, kWarpMask = 14, kWarpStore = 15;
constexpr int kThreads = 16 * 32;

constexpr uint32_t kSlot = 3 * kTile;  // X, Y raw; Z = q~ / k~ hi, then the outputs
constexpr uint32_t kOffRing = 0;
constexpr uint32_t kOffOps = kOffRing + kRing * kSlot;     // state hi | lo
constexpr uint32_t kOffFlags = kOffOps + 2 * kStateTile;   // 2 x 2 KB bitmasks
constexpr uint32_t kOffInv = kOffFlags + 2 * (kMaxN / 8);  // per slot 64 x 1/norm (bwd)
constexpr uint32_t kOffMisc = kOffInv + kRing * kRows * 4;
constexpr uint32_t kOffBar = kOffMisc + 128;
constexpr uint32_t kSmemBytes = kOffBar + 32 * 8;
static_assert(kSmemBytes <= 227 * 1024, "shared-memory budget");
static_assert((kOffOps % 1024) == 0, "SW128 tiles are 1024-B aligned");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAcc = 0, kRun = 128, kOut0 = 256, kOutCols = 128;

__device__ __forceinline__ int slot3(int it) { return it % kRing; }
__device__ __forceinline__ uint32_t par3(int it) { return (uint32_t)(it / kRing) & 1u; }

struct Bars {
  uint64_t raw_full[kRing], slot_free[kRing], split_full[kRing], mma_done[kRing], staged[kRing];
  uint64_t out_free[4];  // out 0, out 1, acc, run as output buffers
  uint64_t op_ready, acc_free, red_done, ops_free;
  uint64_t fl_full[2], fl_empty[2];
  uint64_t issued;
};
static_assert(sizeof(Bars) <= 256, "barrier area");

// ---- MMA issue (one thread) -------------------------------------------------------
// R (M = N = 128) += x^T y over `ksteps` 16-row groups of two MN-major row tiles
__device__ __forceinline__ void issue_red(uint32_t d, uint32_t x, uint32_t y, int ksteps, bool first) {
  const uint32_t id = idesc_bf16(128, 128, true, true);
  for (int kk = 0; kk < ksteps; ++kk)
    mma_bf16(d, sdesc(x + 2048u * kk, kHalf, 1024u), sdesc(y + 2048u * kk, kHalf, 1024u), id,
             (first && kk == 0) ? 0u : 1u);
}
// B operand of a row output for K-step kk: MN-major (rows = k: O = Q~ S,
// dV = K~ dA) or K-major (rows = n: dQ~ = dO S^T, dK~ = V dA^T)
template <bool kBMN>
__device__ __forceinline__ uint64_t state_desc(uint32_t b, int kk) {
  return kBMN ? sdesc(b + 2048u * kk, kStateHalf, 1024u)
              : sdesc(b + (uint32_t)(kk >> 2) * kStateHalf + 32u * (kk & 3), 16u, 1024u);
}
__device__ __forceinline__ uint64_t row_desc(uint32_t a, int kk) {
  return sdesc(a + (uint32_t)(kk >> 2) * kHalf + 32u * (kk & 3), 16u, 1024u);
}
// D (64 x 128) = A (64-row tile, K-major, K = 128 features) x (state hi + lo)
template <bool kBMN>
__device__ __forceinline__ void issue_rowout(uint32_t d, uint32_t a, uint32_t bh, uint32_t bl) {
  const uint32_t id = idesc_bf16(64, 128, false, kBMN);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint64_t ad = row_desc(a, kk);
    mma_bf16(d, ad, state_desc<kBMN>(bh, kk), id, kk > 0 ? 1u : 0u);
    mma_bf16(d, ad, state_desc<kBMN>(bl, kk), id, 1u);
  }
}
// the same with A = hi (ah) + lo (al): hi*hi + hi*lo + lo*hi
template <bool kBMN>
__device__ __forceinline__ void issue_rowout3(uint32_t d, uint32_t ah, uint32_t al, uint32_t bh, uint32_t bl) {
  const uint32_t id = idesc_bf16(64, 128, false, kBMN);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint64_t adh = row_desc(ah, kk), adl = row_desc(al, kk);
    const uint64_t dh = state_desc<kBMN>(bh, kk), dl = state_desc<kBMN>(bl, kk);
    mma_bf16(d, adh, dh, id, kk > 0 ? 1u : 0u);
    mma_bf16(d, adh, dl, id, 1u);
    mma_bf16(d, adl, dh, id, 1u);
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
    for (int i = 0; i < 4; ++i) mbar_init(&br->out_free[i], kEpiWarps);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&br->fl_full[i], 1);
      mbar_init(&br->fl_empty[i], kSplitWarps + kEpiWarps);
    }
    mbar_init(&br->op_ready, 1);
    mbar_init(&br->acc_free, kEpiWarps);
    mbar_init(&br->red_done, 1);
    mbar_init(&br->ops_free, 1);
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
__device__ __forceinline__ void epi_sync() {  // the 4 epiloguer warps
  asm volatile("bar.sync 2, 128;" ::: "memory");
}
__device__ __forceinline__ void arrive_staged(Bars* br, int b, int lane) {
  fence_proxy_async();
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(&br->staged[b]);
}
// TMEM column of output buffer b (0, 1: the output columns; 2, 3: acc, run)
__device__ __forceinline__ uint32_t out_col(int b) { return b < 2 ? kOut0 + kOutCols * b : (b == 2 ? kAcc : kRun); }
// MMA side: wait until buffer b's previous use is drained (use parities in `par`)
__device__ __forceinline__ void take_out(Bars* br, uint32_t& par, int b) {
  mbar_wait(&br->out_free[b], ((par >> b) & 1u) ^ 1u);
  par ^= 1u << b;
}
__device__ __forceinline__ void release_out(Bars* br, int b, int lane) {
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(&br->out_free[b]);
}

// ---- accumulator (M = 128: thread t = TMEM lane t = state row t) --------------------
// 32-column block q of this thread's state row (+ the running sum)
__device__ __forceinline__ void acc_block(uint32_t tmem, uint32_t lane_base, int q, bool with_run,
                                          float (&r)[32]) {
  tmem_ld32(tmem + lane_base + kAcc + 32u * q, r);
  tmem_wait_ld();
  if (with_run) {
    float s[32];
    tmem_ld32(tmem + lane_base + kRun + 32u * q, s);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 32; ++e) r[e] += s[e];
  }
}
__device__ __forceinline__ void flush_acc(uint32_t tmem, uint32_t lane_base, bool first) {
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    float r[32];
    acc_block(tmem, lane_base, q, !first, r);
    tmem_st32(tmem + lane_base + kRun + 32u * q, r);
    tmem_wait_st();
  }
}
// state tiles: block q (columns 32 q ..) of row a is half-tile q / 2, granules 4 (q % 2) ..
__device__ __forceinline__ void store_state_block(uint8_t* hi, int a, int q, const float (&x)[32]) {
  store_split_half(hi + (q >> 1) * kStateHalf, hi + kStateTile + (q >> 1) * kStateHalf, a, q & 1, x);
}
__device__ __forceinline__ void load_state_block(const uint8_t* hi, int a, int q, float (&x)[32]) {
  load_split_half(hi + (q >> 1) * kStateHalf, hi + kStateTile + (q >> 1) * kStateHalf, a, q & 1, x);
}

// ---- splitter: four threads per chunk row, 32 columns each ------------------------
// Thread q of a row owns column block q (half-tile q / 2, granules 4 (q % 2) ..
// + 3).  Its four 16-B granules are visited in the order k' = (k + 2 (q / 2)) & 3,
// so that an 8-lane LDS / STS phase (two rows) covers the 8 bank groups; x[8 k ..]
// holds granule k' (split_store writes them back in the same order).
struct SplitRow {
  int row, q;
  float x[32];
  float ss;  // |row|^2
};
__device__ __forceinline__ uint32_t split_off(const SplitRow& s, int k) {
  return (uint32_t)(s.q >> 1) * kHalf + goff(s.row, 4 * (s.q & 1) + ((k + 2 * (s.q >> 1)) & 3));
}
__device__ __forceinline__ void split_load(const uint8_t* X, int t, SplitRow& s) {
  s.row = t >> 2;
  s.q = t & 3;
#pragma unroll
  for (int k = 0; k < 4; ++k) unpack8(*reinterpret_cast<const uint4*>(X + split_off(s, k)), s.x + 8 * k);
  float part = tcb::sumsq32(s.x);
  part += __shfl_xor_sync(0xffffffffu, part, 1);
  s.ss = part + __shfl_xor_sync(0xffffffffu, part, 2);
}
// hi into Z, lo over this thread's own raw granules of X
__device__ __forceinline__ void split_store(uint8_t* Z, uint8_t* X, const SplitRow& s) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float x0 = s.x[8 * k + 2 * e], x1 = s.x[8 * k + 2 * e + 1];
      hw[e] = pack2(x0, x1);
      lw[e] = pack2(x0 - __uint_as_float(hw[e] << 16), x1 - __uint_as_float(hw[e] & 0xFFFF0000u));
    }
    const uint32_t o = split_off(s, k);
    *reinterpret_cast<uint4*>(Z + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(X + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
}

// ---- row-output epilogue (M = 64): thread (row = 16 wq + lane % 16, h = lane / 16)
// holds column blocks h and h + 2 of its row (tcgen05.ld.16x32bx2 at columns 0 and 64)
__device__ __forceinline__ void out_block(uint32_t d, int hh, float (&g)[32]) { tmem_ld_pair(d + 64u * hh, g); }
// x~ = hi (Z) + lo (X) at block 2 hh + h of row `row`
__device__ __forceinline__ void row_block(const uint8_t* Z, const uint8_t* X, int row, int hh, int h,
                                          float (&x)[32]) {
  load_split_half(Z + hh * kHalf, X + hh * kHalf, row, h, x);
}

// ======================================================================================
// Forward
// ======================================================================================
__global__ void __launch_bounds__(kThreads, 1) cos_fwd_tch_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap to,
    const OpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = (int)p.N, H = (int)p.H;
  const int units = (int)(p.B * p.H);
  const int C = (N + kRows - 1) / kRows;
  const int P = (p.out != nullptr || p.saved_norms != nullptr) ? 2 : 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Bars* br = reinterpret_cast<Bars*>(smem + kOffBar);
  UnitConst* ucs = reinterpret_cast<UnitConst*>(smem + kOffMisc);
  uint8_t* ops = smem + kOffOps;
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
            tc::ItemPos f;
            if (p.l2_ahead && tc::item_pos(it + p.l2_ahead, P, C, units, H, f))
              for (int hb = 0; hb < 2; ++hb) {
                tc::tma_prefetch_4d(f.ps == 0 ? &tk : &tq, 64 * hb, f.c * kRows, f.h, f.b);
                if (f.ps == 0) tc::tma_prefetch_4d(&tv, 64 * hb, f.c * kRows, f.h, f.b);
              }
            mbar_wait(&br->slot_free[st], par3(it) ^ 1u);
            uint8_t* X = smem + kOffRing + st * kSlot;
            if (ps == 0) {
              mbar_expect_tx(&br->raw_full[st], 2 * kTile);
              for (int hb = 0; hb < 2; ++hb) {
                tma_load_4d(X + hb * kHalf, &tk, 64 * hb, c * kRows, h, b, &br->raw_full[st]);
                tma_load_4d(X + kTile + hb * kHalf, &tv, 64 * hb, c * kRows, h, b, &br->raw_full[st]);
              }
            } else {
              mbar_expect_tx(&br->raw_full[st], kTile);
              for (int hb = 0; hb < 2; ++hb)
                tma_load_4d(X + hb * kHalf, &tq, 64 * hb, c * kRows, h, b, &br->raw_full[st]);
            }
          }
      }
    }
  } else if (warp == kWarpMma) {
    int it = 0, j = 0, nflush = 0, ob = 0;
    const uint32_t base = smem_u32(smem);
    const uint32_t opS = base + kOffOps;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      for (int ps = 0; ps < P; ++ps)
        for (int c = 0; c < C; ++c, ++it) {
          const int st = slot3(it);
          mbar_wait(&br->split_full[st], par3(it));
          if (ps == 0 && c == 0 && P == 1 && j > 0) mbar_wait(&br->op_ready, (j - 1) & 1);
          if (ps == 0 && c > 0 && c % kFlush == 0) mbar_wait(&br->acc_free, (nflush++) & 1);
          if (ps == 1 && c == 0) mbar_wait(&br->op_ready, j & 1);
          if (ps == 1) mbar_wait(&br->out_free[ob & 1], ((ob >> 1) & 1) ^ 1u);
          tc_fence_after();
          const uint32_t X = base + kOffRing + st * kSlot, Y = X + kTile, Z = X + 2 * kTile;
          if (elect_one()) {
            if (ps == 0) {  // S += K~^T V (attention.cpp:345-353), K~ = hi (Z) + lo (X)
              const int ks = (min(kRows, N - c * kRows) + 15) >> 4;
              issue_red(tmem + kAcc, Z, Y, ks, c % kFlush == 0);
              issue_red(tmem + kAcc, X, Y, ks, false);
            } else {  // O = Q~ S (:379-387)
              issue_rowout3<true>(tmem + kOut0 + kOutCols * (ob & 1), Z, X, opS, opS + kStateTile);
            }
            mma_commit(&br->mma_done[st]);
          }
          __syncwarp();
          if (ps == 1) ++ob;
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
              uint8_t* Z = smem + kOffRing + st * kSlot + 2 * kTile;
              tma_store_4d(&to, Z, 0, c * kRows, h, b);
              tma_store_4d(&to, Z + kHalf, 64, c * kRows, h, b);
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
    int it = 0, j = 0, ob = 0;
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
        if (splitter) {  // ---------------- splitter ----------------
          mbar_wait(&br->raw_full[st], par3(it));
          SplitRow s;
          split_load(X, t, s);
          const int r = c * kRows + s.row;
          const bool wr = norms && r < N && s.q == 0;
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
          split_store(Z, X, s);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&br->split_full[st]);
        } else {  // ---------------- epiloguer ----------------
          mbar_wait(&br->mma_done[st], par3(it));
          tc_fence_after();
          if (ps == 0) {
            arrive_staged(br, st, lane);  // a pass-1 item stages nothing: free the slot now
            if (c != C - 1 && c % kFlush == kFlush - 1) {  // long N: flush the accumulator
              flush_acc(tmem, lane_base, c == kFlush - 1);
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&br->acc_free);
            }
            if (c == C - 1) {  // S complete: saved S + the bf16 hi / lo state operand
#pragma unroll 1
              for (int q = 0; q < 4; ++q) {
                float sv[32];
                acc_block(tmem, lane_base, q, C > kFlush, sv);
                if (gS_all) {
                  float4* gs = reinterpret_cast<float4*>(gS_all + (int64_t)u * (kD * kD) + t * kD + 32 * q);
#pragma unroll
                  for (int e = 0; e < 8; ++e)
                    gs[e] = make_float4(sv[4 * e], sv[4 * e + 1], sv[4 * e + 2], sv[4 * e + 3]);
                }
                store_state_block(ops, t, q, sv);
              }
              fence_proxy_async();
              tc_fence_before();
              epi_sync();
              if (t == 0) mbar_arrive(&br->op_ready);
            }
          } else {  // O rows = s (Q~ S), staged in Z (its MMAs are done)
            const int row = 16 * wq + (lane & 15), h = lane >> 4;
            const uint32_t D = tmem + kOut0 + kOutCols * (ob & 1) + lane_base;
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
              float o[32];
              out_block(D, hh, o);
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] *= uc.s;
              store_half(Z + hh * kHalf, row, h, o);
            }
            release_out(br, ob & 1, lane);
            ++ob;
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
__global__ void __launch_bounds__(kThreads, 1) cos_bwd_tch_kernel(
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
  uint8_t* ops = smem + kOffOps;  // S (pass 1), then dA (pass 2)
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
      const int64_t sbytes = (int64_t)kD * kD * 4;  // one unit's saved S
      const uint8_t* gS = static_cast<const uint8_t*>(p.saved_S);
      if (blockIdx.x < units) tc::bulk_prefetch_l2(gS + blockIdx.x * sbytes, (uint32_t)sbytes);
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        if (u + (int)gridDim.x < units)  // the splitter loads the next unit's S: have it in L2
          tc::bulk_prefetch_l2(gS + (u + gridDim.x) * sbytes, (uint32_t)sbytes);
        for (int ps = 0; ps < 2; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot3(it);
            mbar_wait(&br->slot_free[st], par3(it) ^ 1u);
            uint8_t* X = smem + kOffRing + st * kSlot;
            mbar_expect_tx(&br->raw_full[st], 2 * kTile);
            for (int hb = 0; hb < 2; ++hb) {
              tma_load_4d(X + hb * kHalf, ps == 0 ? &tq : &tk, 64 * hb, c * kRows, h, b, &br->raw_full[st]);
              tma_load_4d(X + kTile + hb * kHalf, ps == 0 ? &tdo : &tv, 64 * hb, c * kRows, h, b,
                          &br->raw_full[st]);
            }
          }
      }
    }
  } else if (warp == kWarpMma) {
    int it = 0, j = 0, nflush = 0, n1 = 0, n2 = 0;
    uint32_t par = 0;
    const uint32_t base = smem_u32(smem);
    const uint32_t opH = base + kOffOps, opL = opH + kStateTile;  // S, then dA
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      for (int ps = 0; ps < 2; ++ps)
        for (int c = 0; c < C; ++c, ++it) {
          const int st = slot3(it);
          mbar_wait(&br->split_full[st], par3(it));
          if (ps == 1 && c == 0) mbar_wait(&br->op_ready, j & 1);
          if (ps == 0 && c > 0 && c % kFlush == 0) mbar_wait(&br->acc_free, (nflush++) & 1);
          // a new G overwrites the accumulator columns: the last pass-2 item that
          // borrowed them must be drained
          if (ps == 0 && c == 0) mbar_wait(&br->out_free[2], ((par >> 2) & 1u) ^ 1u);
          tc_fence_after();
          const uint32_t X = base + kOffRing + st * kSlot, Y = X + kTile, Z = X + 2 * kTile;
          if (ps == 0) {
            if (elect_one()) {  // G += Q~^T dO (attention.cpp:405), Q~ = hi (Z) + lo (X)
              const int ks = (min(kRows, N - c * kRows) + 15) >> 4;
              issue_red(tmem + kAcc, Z, Y, ks, c % kFlush == 0);
              issue_red(tmem + kAcc, X, Y, ks, false);
            }
            __syncwarp();
            const int b = n1++ & 1;
            take_out(br, par, b);
            tc_fence_after();
            if (elect_one()) {
              // dQ~ (unscaled) = dO S^T (:410-411): A = dO (K-major), B row n = S row n
              issue_rowout<false>(tmem + out_col(b), Y, opH, opL);
              // G complete, and every MMA that reads this unit's S
              if (c == C - 1) mma_commit(&br->red_done);
              mma_commit(&br->mma_done[st]);
            }
            __syncwarp();
          } else {
            const int pr = (n2++ & 1) * 2;  // buffer pair (0, 1) or (2, 3)
            take_out(br, par, pr);
            tc_fence_after();
            if (elect_one()) issue_rowout3<true>(tmem + out_col(pr), Z, X, opH, opL);  // dV = K~ dA (:416)
            __syncwarp();
            take_out(br, par, pr + 1);
            tc_fence_after();
            if (elect_one()) {
              issue_rowout<false>(tmem + out_col(pr + 1), Y, opH, opL);  // dK~ = V dA^T (:415)
              mma_commit(&br->mma_done[st]);
              if (c == C - 1) mma_commit(&br->ops_free);  // every MMA reading this unit's dA
            }
            __syncwarp();
          }
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
            for (int hb = 0; hb < 2; ++hb) {
              if (ps == 0) {
                tma_store_4d(&tdq, X + 2 * kTile + hb * kHalf, 64 * hb, c * kRows, h, b);
              } else {
                tma_store_4d(&tdv, X + 2 * kTile + hb * kHalf, 64 * hb, c * kRows, h, b);
                tma_store_4d(&tdk, X + kTile + hb * kHalf, 64 * hb, c * kRows, h, b);
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
    int it = 0, j = 0, n1 = 0, n2 = 0;
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
        float* inv_st = invs + st * kRows;
        if (splitter) {  // ---------------- splitter ----------------
          if (ps == 0 && c == 0) {
            // this unit's S (saved by the forward) as bf16 hi / lo rows, once the
            // previous unit's last MMA reading dA from the same area is complete
            if (j > 0) mbar_wait(&br->ops_free, (j - 1) & 1);
            const int a = t >> 1, hh = t & 1;  // row a, columns 64 hh .. 64 hh + 63
            const float4* gs = reinterpret_cast<const float4*>(gS_all + (int64_t)u * (kD * kD) + a * kD + 64 * hh);
#pragma unroll 1
            for (int r = 0; r < 2; ++r) {
              float v[32];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float4 w = __ldg(gs + 8 * r + e);
                v[4 * e] = w.x;
                v[4 * e + 1] = w.y;
                v[4 * e + 2] = w.z;
                v[4 * e + 3] = w.w;
              }
              store_state_block(ops, a, 2 * hh + r, v);
            }
          }
          mbar_wait(&br->raw_full[st], par3(it));
          SplitRow s;
          split_load(X, t, s);
          const int r = c * kRows + s.row;
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
          split_store(Z, X, s);
          if (s.q == 0) inv_st[s.row] = iv;  // 1/norm for the epiloguer's Jacobian
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&br->split_full[st]);
        } else {  // ---------------- epiloguer ----------------
          if (ps == 0 && c == C - 1) {
            // G complete: dm = -ln(n) s <G, S> (:408); dA = s G (:412-413) over S in place
            mbar_wait(&br->red_done, j & 1);
            tc_fence_after();
            float dotf = 0.f;
#pragma unroll 1
            for (int q = 0; q < 4; ++q) {
              float gr[32], sv[32];
              acc_block(tmem, lane_base, q, C > kFlush, gr);
              load_state_block(ops, t, q, sv);
              dotf += dot32(gr, sv);
#pragma unroll
              for (int e = 0; e < 32; ++e) gr[e] *= uc.s;
              store_state_block(ops, t, q, gr);
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
          tc_fence_after();
          if (ps == 0 && c != C - 1 && c % kFlush == kFlush - 1) {  // long N: flush G
            flush_acc(tmem, lane_base, c == kFlush - 1);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&br->acc_free);
          }
          const int row = 16 * wq + (lane & 15), h = lane >> 4;
          const int r = c * kRows + row;
          const float iv = inv_st[row];
          // g = dQ~ (pass 1) or dK~ (pass 2, the second buffer of the item's pair); pr = g . x~
          const int bv = (n2 & 1) * 2;  // pass 2: dV in bv, dK~ in bv + 1
          const int bg = ps == 0 ? (n1 & 1) : bv + 1;
          const uint32_t Dg = tmem + out_col(bg) + lane_base;
          float pr = 0.f;
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            float g[32], x[32];
            out_block(Dg, hh, g);
            row_block(Z, X, row, hh, h, x);
            pr += dot32(g, x);
          }
          pr += __shfl_xor_sync(0xffffffffu, pr, 16);  // the row's other two blocks
          if (ps == 0) {
            // dQ_i = (g - (g.q~_i) q~_i) / nq_i, g = s dO S^T (:410-411, :421-428); staged in Z
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
              float g[32], x[32];
              out_block(Dg, hh, g);
              row_block(Z, X, row, hh, h, x);
#pragma unroll
              for (int e = 0; e < 32; ++e) g[e] = (uc.s * g[e] - uc.s * pr * x[e]) * iv;
              store_half(Z + hh * kHalf, row, h, g);
            }
            release_out(br, bg, lane);
            ++n1;
          } else {
            const bool f = r < N && tc::flag_at(fl, r);
            const bool nan_out = uc.tn == 0;
            // dK_i = v_i ? (g - (g.k~)k~) / nk : 0 (:430-437), staged in Y (V is done)
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
              float g[32], x[32];
              out_block(Dg, hh, g);
              row_block(Z, X, row, hh, h, x);
#pragma unroll
              for (int e = 0; e < 32; ++e) g[e] = nan_out ? qnan : (f ? (g[e] - pr * x[e]) * iv : 0.f);
              store_half(Y + hh * kHalf, row, h, g);
            }
            release_out(br, bg, lane);
            // dV_i = v_i ? (K~ dA)_i : 0 (:416, :439), staged in Z (K~ is done)
            const uint32_t Dv = tmem + out_col(bv) + lane_base;
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
              float g[32];
              out_block(Dv, hh, g);
#pragma unroll
              for (int e = 0; e < 32; ++e) g[e] = nan_out ? qnan : (f ? g[e] : 0.f);
              store_half(Z + hh * kHalf, row, h, g);
            }
            release_out(br, bv, lane);
            ++n2;
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
  if (p.dm_total) tc::last_cta_dm_total(p, units, smem + kOffRing);
}

}  // namespace tch

// ---- host side ----------------------------------------------------------------------

// 4-D bf16 map over (128, N, H, B), box (64, 64, 1, 1), 128-byte swizzle: two boxes per row
inline bool make_tch_map(CUtensorMap* map, const void* base, const OpParams& p) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {128, (cuuint64_t)p.N, (cuuint64_t)p.H, (cuuint64_t)p.B};
  cuuint64_t strides[3] = {(cuuint64_t)p.sn * 2, (cuuint64_t)p.sh * 2, (cuuint64_t)p.sb * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)tch::kRows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
inline bool tch_layout_ok(const OpParams& p, std::initializer_list<const void*> ptrs) {
  if (p.D != 128 || p.N < 1 || p.N > tch::kMaxN) return false;
  if ((p.sn * 2) % 16 || (p.sh * 2) % 16 || (p.sb * 2) % 16) return false;
  if (p.B * p.H > (1ll << 31) - 1) return false;
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<uintptr_t>(q) & 15)) return false;
  return encode_fn() != nullptr && getenv("COTTEN_NO_TCH") == nullptr;
}
template <typename T>
inline bool tch_fwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, __nv_bfloat16>::value) {
    return false;
  } else {
    return tch_layout_ok(p, {p.q, p.k, p.v, p.out});
  }
}
template <typename T>
inline bool tch_bwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, __nv_bfloat16>::value) {
    return false;
  } else {
    return p.saved_S != nullptr && tch_layout_ok(p, {p.q, p.k, p.v, p.dout, p.dq, p.dk, p.dv});
  }
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_tch_pdl(void (*kern)(KArgs...), int grid, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tch::kThreads);
  cfg.dynamicSmemBytes = tch::kSmemBytes;
  cfg.stream = st;
  static const bool pdl = getenv("COTTEN_NO_PDL") == nullptr;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
inline int launch_tch_fwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mo;
  if (!make_tch_map(&mq, p.q, p) || !make_tch_map(&mk, p.k, p) || !make_tch_map(&mv, p.v, p) ||
      !make_tch_map(&mo, p.out ? p.out : p.q, p))
    return -1;
  if (cudaFuncSetAttribute(tch::cos_fwd_tch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tch::kSmemBytes) != cudaSuccess)
    return -1;
  const int grid = std::min((int)(p.B * p.H), sm_count());
  OpParams q = p;
  q.l2_ahead = l2_ahead_items(true, (int)((p.N + tch::kRows - 1) / tch::kRows));
  if (launch_tch_pdl(tch::cos_fwd_tch_kernel, grid, st, mq, mk, mv, mo, q) != cudaSuccess) return -1;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}
inline int launch_tch_bwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mg, mdq, mdk, mdv;
  if (!make_tch_map(&mq, p.q, p) || !make_tch_map(&mk, p.k, p) || !make_tch_map(&mv, p.v, p) ||
      !make_tch_map(&mg, p.dout, p) || !make_tch_map(&mdq, p.dq, p) || !make_tch_map(&mdk, p.dk, p) ||
      !make_tch_map(&mdv, p.dv, p))
    return -1;
  if (cudaFuncSetAttribute(tch::cos_bwd_tch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tch::kSmemBytes) != cudaSuccess)
    return -1;
  const int grid = std::min((int)(p.B * p.H), sm_count());
  OpParams q = p;
  q.l2_ahead = l2_ahead_items();
  if (launch_tch_pdl(tch::cos_bwd_tch_kernel, grid, st, mq, mk, mv, mg, mdq, mdk, mdv, q) != cudaSuccess)
    return -1;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace cotten
