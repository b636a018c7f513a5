// Tensor-core (tcgen05 kind::f16) cosine-attention kernels for fp32 inputs,
// head_dim 128, any seq_len up to 16384 — BASELINE config #5's fp32 d_h = 128
// points, which the FP32-pipe kernels (kernels_rt.cuh, the A/B partner) serve
// at 0.11-0.13 of HBM.
//
// Arithmetic as kernels_tcf.cuh: every fp32 operand (q~ / k~, V, dO and the
// 128 x 128 state S / dA) enters the MMAs as three bf16 parts x = b0 + b1 + b2
// (exact), six products b0 b0' + b0 b1' + b1 b0' + b0 b2' + b2 b0' + b1 b1'
// accumulated in fp32 TMEM; the S / G running sum lives in TMEM as in
// kernels_tch.cuh, and so does the shared S / dA state area (three parts,
// 96 KB) and the borrowing of the accumulator columns by the backward's pass 2.
//
// Shared memory decides the shape: the state alone is 96 KB, and a row of
// three parts is 768 B per tensor, so items are 32 rows of two tensors —
// X, Y raw fp32 (four SW128 boxes of 32 columns each, 16 KB), parts 0 | 1
// written over them in place, part 2 of each in 8 KB beside them: 48 KB per
// slot, two slots.  Reductions are M = N = 128 over 16-row K steps; row
// outputs are M = 64 MMAs of which rows 0-31 are the item's rows (rows 32-63
// read whatever follows the 32-row part tile and are never looked at; the D
// rows 0-31 sit in TMEM lanes 0-15 and 32-47, so epiloguer warps 0-1 carry
// the row epilogues).  Per tile row the splitter's eight threads are spread
// over lanes rr + 4 pos (pos -> column block 0 3 1 2 4 7 5 6), so that each
// 8-lane LDS.128 of the raw boxes and STS.128 of the parts covers the 8 bank
// groups.
//   forward   pass 1 (K, V):  S += K~^T V                    (attention.cpp:345-353)
//             pass 2 (Q):     O = s Q~ S                     (:379-387)
//   backward  pass 1 (Q, dO): G += Q~^T dO,  dQ~ = s dO S^T  (:405, :410-411)
//             pass 2 (K, V):  dV = K~ dA,    dK~ = V dA^T    (:412-416)
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels_tch.cuh"

namespace cotten {
namespace tcg {

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
using tcb::mma_bf16;
using tcb::sdesc;
using tcf::load_parts8;
using tcf::store_parts8;
using tcf::tmem_ld_pair;

constexpr int kD = 128;
constexpr int kRows = 32;
constexpr uint32_t kBox = 4096;                  // 32 rows x 128 B: one fp32 box / one part half-tile
constexpr uint32_t kRaw = 4 * kBox;              // a raw fp32 tensor tile (parts 0 | 1 after the split)
constexpr uint32_t kPart = 2 * kBox;             // one bf16 part of a tensor tile
constexpr uint32_t kStateHalf = 16384;           // 128 state rows x 128 B
constexpr uint32_t kStatePart = 2 * kStateHalf;  // one bf16 part of the 128 x 128 state
constexpr int kRing = 2;
constexpr int kMaxN = 16384;
constexpr int kFlush = 16;  // S / G flushed into the running sum every 16 chunks (512 rows)
constexpr int kSplitWarps = 8, kEpiWarps = 4;
constexpr int kWarpEpi0 = kSplitWarps;
constexpr int kWarpProducer = 12, kWarpMma = 13, kWarpMask = 14, kWarpStore = 15;
constexpr int kThreads = 16 * 32;

// slot: X raw (parts 0 | 1) at +0, Y at +16K, X part 2 at +32K, Y part 2 at +40K
constexpr uint32_t kSlot = 2 * kRaw + 2 * kPart;
constexpr uint32_t kOffRing = 0;
constexpr uint32_t kOffOps = kOffRing + kRing * kSlot;    // state parts 0-2
constexpr uint32_t kOffFlags = kOffOps + 3 * kStatePart;  // 2 x 2 KB bitmasks
constexpr uint32_t kOffInv = kOffFlags + 2 * (kMaxN / 8);
constexpr uint32_t kOffMisc = kOffInv + kRing * kRows * 4;
constexpr uint32_t kOffBar = kOffMisc + 128;
constexpr uint32_t kSmemBytes = kOffBar + 32 * 8;
static_assert(kSmemBytes <= 227 * 1024, "shared-memory budget");
static_assert((kOffOps % 1024) == 0, "SW128 tiles are 1024-B aligned");

using tch::kAcc;
using tch::kOut0;
using tch::kOutCols;
using tch::kRun;
using tch::kTmemCols;
using tch::out_col;

// Optional per-item trace of the backward (-DCOTTEN_TCG_TRACE=1, variant builds
// only): clock64 stamps of the first tcb::kTraceItems items of every CTA into
// p.workspace [cta][item][8], the stamp meanings of kernels_tcb.cuh
// (scripts/dev/tcb_trace_report.py reads tcg_bwd.bin).
#ifndef COTTEN_TCG_TRACE
#define COTTEN_TCG_TRACE 0
#endif
#if COTTEN_TCG_TRACE
#define TCG_TRACE(k, cond)                                                                   \
  do {                                                                                       \
    if ((cond) && p.workspace && it < tcb::kTraceItems)                                      \
      static_cast<long long*>(p.workspace)[(blockIdx.x * tcb::kTraceItems + it) * 8 + (k)] = clock64(); \
  } while (0)
#else
#define TCG_TRACE(k, cond) \
  do {                     \
  } while (0)
#endif

__device__ __forceinline__ int slot2(int it) { return it & 1; }
__device__ __forceinline__ uint32_t par2(int it) { return (uint32_t)(it >> 1) & 1u; }

using tch::Bars;
using tch::setup;
using tch::teardown;
using tch::epi_sync;
using tch::arrive_staged;
using tch::release_out;
using tch::take_out;
using tch::acc_block;
using tch::flush_acc;

// ---- MMA issue (one thread) -------------------------------------------------------
__device__ __forceinline__ int part_i(int pr) { return pr == 2 ? 1 : pr == 4 ? 2 : pr == 5 ? 1 : 0; }
__device__ __forceinline__ int part_j(int pr) { return pr == 1 ? 1 : pr == 3 ? 2 : pr == 5 ? 1 : 0; }
// R (M = N = 128) += x^T y over `ksteps` 16-row groups; x, y = three MN-major part tiles each
__device__ __forceinline__ void issue_red(uint32_t d, const uint32_t (&x)[3], const uint32_t (&y)[3],
                                          int ksteps, bool first) {
  const uint32_t id = idesc_bf16(128, 128, true, true);
  for (int kk = 0; kk < ksteps; ++kk)
#pragma unroll
    for (int pr = 0; pr < 6; ++pr)
      mma_bf16(d, sdesc(x[part_i(pr)] + 2048u * kk, kBox, 1024u), sdesc(y[part_j(pr)] + 2048u * kk, kBox, 1024u),
               id, (first && kk == 0 && pr == 0) ? 0u : 1u);
}
template <bool kBMN>
__device__ __forceinline__ uint64_t state_desc(uint32_t b, int kk) {
  return kBMN ? sdesc(b + 2048u * kk, kStateHalf, 1024u)
              : sdesc(b + (uint32_t)(kk >> 2) * kStateHalf + 32u * (kk & 3), 16u, 1024u);
}
// D (M = 64: rows 0-31 the item's) = A (K-major part tiles) x B (state parts)
template <bool kBMN>
__device__ __forceinline__ void issue_rowout(uint32_t d, const uint32_t (&a)[3], const uint32_t (&b)[3]) {
  const uint32_t id = idesc_bf16(64, 128, false, kBMN);
#pragma unroll 1
  for (int kk = 0; kk < 8; ++kk)
#pragma unroll
    for (int pr = 0; pr < 6; ++pr)
      mma_bf16(d, sdesc(a[part_i(pr)] + (uint32_t)(kk >> 2) * kBox + 32u * (kk & 3), 16u, 1024u),
               state_desc<kBMN>(b[part_j(pr)], kk), id, (kk == 0 && pr == 0) ? 0u : 1u);
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

// ---- state parts (row a, 32-column block q: half-tile q / 2, granules 4 (q % 2) ..) ----
__device__ __forceinline__ void store_state_block(uint8_t* ops, int a, int q, const float (&x)[32]) {
  uint8_t* b = ops + (q >> 1) * kStateHalf;
#pragma unroll
  for (int g = 0; g < 4; ++g) store_parts8(b, b + kStatePart, b + 2 * kStatePart, a, 4 * (q & 1) + g, x + 8 * g);
}
__device__ __forceinline__ void load_state_block(const uint8_t* ops, int a, int q, float (&x)[32]) {
  const uint8_t* b = ops + (q >> 1) * kStateHalf;
#pragma unroll
  for (int g = 0; g < 4; ++g) load_parts8(b, b + kStatePart, b + 2 * kStatePart, a, 4 * (q & 1) + g, x + 8 * g);
}

// ---- splitter: eight threads per tile row (16 columns each) --------------------------
// lane = rr + 4 pos: row 4 warp + rr, column block qb = {0, 3, 1, 2, 4, 7, 5, 6}[pos]
// (columns 16 qb ..: fp32 box qb / 2, granules 4 (qb % 2) ..; part half-tile qb / 4,
// bf16 granules 2 (qb % 4), + 1)
struct SplitRow {
  int row, qb;
  float x[16];
  float ss;
};
__device__ __forceinline__ void split_load(const uint8_t* X, int t, SplitRow& s) {
  const int lane = t & 31, pos = lane >> 2;
  s.row = 4 * (t >> 5) + (lane & 3);
  s.qb = (pos & 4) | ((pos & 3) == 0 ? 0 : (pos & 3) == 1 ? 3 : (pos & 3) == 2 ? 1 : 2);
  const uint8_t* box = X + (s.qb >> 1) * kBox;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 v = *reinterpret_cast<const float4*>(box + goff(s.row, 4 * (s.qb & 1) + k));
    s.x[4 * k] = v.x;
    s.x[4 * k + 1] = v.y;
    s.x[4 * k + 2] = v.z;
    s.x[4 * k + 3] = v.w;
  }
  float a = 0.f, b = 0.f;
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    a = fmaf(s.x[e], s.x[e], a);
    b = fmaf(s.x[e + 1], s.x[e + 1], b);
  }
  float part = a + b;
  part += __shfl_xor_sync(0xffffffffu, part, 4);
  part += __shfl_xor_sync(0xffffffffu, part, 8);
  s.ss = part + __shfl_xor_sync(0xffffffffu, part, 16);
}
// parts 0 | 1 over the raw tile X, part 2 into P2.  Call after a __syncwarp that
// follows every split_load of the warp (a row's raw bytes are shared by its eight threads).
__device__ __forceinline__ void split_store(uint8_t* X, uint8_t* P2, const SplitRow& s) {
  uint8_t* h = X + (s.qb >> 2) * kBox;
  uint8_t* h2 = P2 + (s.qb >> 2) * kBox;
  store_parts8(h, h + kPart, h2, s.row, 2 * (s.qb & 3), s.x);
  store_parts8(h, h + kPart, h2, s.row, 2 * (s.qb & 3) + 1, s.x + 8);
}

// ---- row epilogue (warps 0-1 of the epiloguer: rows 16 wq + lane % 16, h = lane / 16) --
// column block q = 2 hh + h of the row: fp32 box q of a staging tile, parts half q / 2
__device__ __forceinline__ void row_block(const uint8_t* X, const uint8_t* P2, int row, int q, float (&x)[32]) {
  const uint8_t* h = X + (q >> 1) * kBox;
#pragma unroll
  for (int g = 0; g < 4; ++g) load_parts8(h, h + kPart, P2 + (q >> 1) * kBox, row, 4 * (q & 1) + g, x + 8 * g);
}
__device__ __forceinline__ void stage_block(uint8_t* T, int row, int q, const float (&x)[32]) {
#pragma unroll
  for (int k = 0; k < 8; ++k)
    *reinterpret_cast<float4*>(T + q * kBox + goff(row, k)) = make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
}

// ======================================================================================
// Forward
// ======================================================================================
// Pass 2 reads Q alone, so its items are 64 rows (raw fp32 as four 64-row
// boxes over X | Y = 32 KB, the three parts over X | Y and the part-2 area =
// 48 KB) and the row-output MMAs are full M = 64 ones; pass 1 keeps the
// 32-row (K, V) items.
constexpr int kRowsQ = 64;
constexpr uint32_t kBoxQ = 8192;   // 64 rows x 128 B
constexpr uint32_t kPartQ = 2 * kBoxQ;
// item i of this CTA's schedule: unit index j (0, 1, ...), pass, chunk
__device__ __forceinline__ bool fwd_item(int i, int P, int C1, int C2, int units, int& u, int& ps, int& c) {
  const int per = C1 + (P == 2 ? C2 : 0);
  const int jj = i / per, rem = i - jj * per;
  u = blockIdx.x + jj * gridDim.x;
  if (u >= units) return false;
  ps = rem >= C1;
  c = ps ? rem - C1 : rem;
  return true;
}
// Q splitter: four threads per 64-row tile row (32 columns each) at lanes
// rr + 8 q4 (row 8 warp + rr): an 8-lane LDS.128 phase is eight rows of one box
__device__ __forceinline__ void split_q(uint8_t* X, int t, float eps, int r, int N, float* norms) {
  const int lane = t & 31, q4 = lane >> 3, row = 8 * (t >> 5) + (lane & 7);
  float x[32];
  const uint8_t* box = X + q4 * kBoxQ;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float4 v = *reinterpret_cast<const float4*>(box + goff(row, k));
    x[4 * k] = v.x;
    x[4 * k + 1] = v.y;
    x[4 * k + 2] = v.z;
    x[4 * k + 3] = v.w;
  }
  float a = 0.f, b = 0.f;
#pragma unroll
  for (int e = 0; e < 32; e += 2) {
    a = fmaf(x[e], x[e], a);
    b = fmaf(x[e + 1], x[e + 1], b);
  }
  float ss = a + b;
  ss += __shfl_xor_sync(0xffffffffu, ss, 8);
  ss += __shfl_xor_sync(0xffffffffu, ss, 16);
  const float iv = rsqrtf(ss + eps);
  r += row;
  if (norms && r < N && q4 == 0) norms[r] = (ss + eps) * iv;  // q~ every row (:366-377)
#pragma unroll
  for (int e = 0; e < 32; ++e) x[e] *= iv;
  __syncwarp();  // the row's four threads have read its raw boxes
  uint8_t* h0 = X + (q4 >> 1) * kBoxQ;
#pragma unroll
  for (int g = 0; g < 4; ++g)
    store_parts8(h0, h0 + kPartQ, h0 + 2 * kPartQ, row, 4 * (q4 & 1) + g, x + 8 * g);
}
// O (64 x 128) = Q~ (64-row three-part tile, K-major) x S (three state parts, MN-major)
__device__ __forceinline__ void issue_rowout_q(uint32_t d, const uint32_t (&a)[3], const uint32_t (&b)[3]) {
  const uint32_t id = idesc_bf16(64, 128, false, true);
#pragma unroll 1
  for (int kk = 0; kk < 8; ++kk)
#pragma unroll
    for (int pr = 0; pr < 6; ++pr)
      mma_bf16(d, sdesc(a[part_i(pr)] + (uint32_t)(kk >> 2) * kBoxQ + 32u * (kk & 3), 16u, 1024u),
               state_desc<true>(b[part_j(pr)], kk), id, (kk == 0 && pr == 0) ? 0u : 1u);
}

__global__ void __launch_bounds__(kThreads, 1) cos_fwd_tcg_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap to,
    const OpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = (int)p.N, H = (int)p.H;
  const int units = (int)(p.B * p.H);
  const int C1 = (N + kRows - 1) / kRows, C2 = (N + kRowsQ - 1) / kRowsQ;
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
          for (int c = 0; c < (ps ? C2 : C1); ++c, ++it) {
            const int st = slot2(it);
            int fu, fps, fc;
            if (p.l2_ahead && fwd_item(it + p.l2_ahead, P, C1, C2, units, fu, fps, fc)) {
              const int fb = fu / H, fh = fu - fb * H;
              for (int hb = 0; hb < 4; ++hb) {
                if (fps == 0) {
                  tc::tma_prefetch_4d(&tk, 32 * hb, fc * kRows, fh, fb);
                  tc::tma_prefetch_4d(&tv, 32 * hb, fc * kRows, fh, fb);
                } else {
                  tc::tma_prefetch_4d(&tq, 32 * hb, fc * kRowsQ, fh, fb);
                }
              }
            }
            mbar_wait(&br->slot_free[st], par2(it) ^ 1u);
            uint8_t* X = smem + kOffRing + st * kSlot;
            if (ps == 0) {
              mbar_expect_tx(&br->raw_full[st], 2 * kRaw);
              for (int hb = 0; hb < 4; ++hb) {
                tma_load_4d(X + hb * kBox, &tk, 32 * hb, c * kRows, h, b, &br->raw_full[st]);
                tma_load_4d(X + kRaw + hb * kBox, &tv, 32 * hb, c * kRows, h, b, &br->raw_full[st]);
              }
            } else {  // Q: four 64-row boxes over X | Y
              mbar_expect_tx(&br->raw_full[st], 4 * kBoxQ);
              for (int hb = 0; hb < 4; ++hb)
                tma_load_4d(X + hb * kBoxQ, &tq, 32 * hb, c * kRowsQ, h, b, &br->raw_full[st]);
            }
          }
      }
    }
  } else if (warp == kWarpMma) {
    int it = 0, j = 0, nflush = 0, n1 = 0;
    uint32_t par = 0;
    const uint32_t base = smem_u32(smem);
    const uint32_t opS[3] = {base + kOffOps, base + kOffOps + kStatePart, base + kOffOps + 2 * kStatePart};
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      for (int ps = 0; ps < P; ++ps)
        for (int c = 0; c < (ps ? C2 : C1); ++c, ++it) {
          const int st = slot2(it);
          mbar_wait(&br->split_full[st], par2(it));
          if (ps == 0 && c == 0 && P == 1 && j > 0) mbar_wait(&br->op_ready, (j - 1) & 1);
          if (ps == 0 && c > 0 && c % kFlush == 0) mbar_wait(&br->acc_free, (nflush++) & 1);
          if (ps == 1 && c == 0) mbar_wait(&br->op_ready, j & 1);
          const int b = n1 & 1;
          if (ps == 1) take_out(br, par, b);
          tc_fence_after();
          const uint32_t X = base + kOffRing + st * kSlot;
          if (elect_one()) {
            if (ps == 0) {  // S += K~^T V (attention.cpp:345-353)
              const uint32_t xp[3] = {X, X + kPart, X + 2 * kRaw};
              const uint32_t yp[3] = {X + kRaw, X + kRaw + kPart, X + 2 * kRaw + kPart};
              const int ks = (min(kRows, N - c * kRows) + 15) >> 4;
              issue_red(tmem + kAcc, xp, yp, ks, c % kFlush == 0);
            } else {  // O = Q~ S (:379-387)
              const uint32_t qp[3] = {X, X + kPartQ, X + 2 * kPartQ};
              issue_rowout_q(tmem + out_col(b), qp, opS);
            }
            mma_commit(&br->mma_done[st]);
          }
          __syncwarp();
          if (ps == 1) ++n1;
        }
    }
  } else if (warp == kWarpMask) {
    tcg::mask_loop(p, smem, br, lane);
  } else if (warp == kWarpStore) {
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        for (int ps = 0; ps < P; ++ps)
          for (int c = 0; c < (ps ? C2 : C1); ++c, ++it) {
            const int st = slot2(it);
            mbar_wait(&br->staged[st], par2(it));
            if (ps == 1 && p.out) {  // O staged as four 64-row fp32 boxes over X | Y
              uint8_t* X = smem + kOffRing + st * kSlot;
              for (int hb = 0; hb < 4; ++hb) tma_store_4d(&to, X + hb * kBoxQ, 32 * hb, c * kRowsQ, h, b);
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
    int it = 0, j = 0, n1 = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int sl = j & 1;
      const uint32_t* fl = reinterpret_cast<const uint32_t*>(smem + kOffFlags + sl * (kMaxN / 8));
      float* norms = norms_all ? norms_all + (int64_t)u * 2 * N : nullptr;
      mbar_wait(&br->fl_full[sl], (j >> 1) & 1);
      const UnitConst uc = ucs[sl];
      const int items = C1 + (P == 2 ? C2 : 0);
      for (int k = 0; k < items; ++k, ++it) {
        const int ps = k >= C1, c = ps ? k - C1 : k;
        const int st = slot2(it);
        uint8_t* X = smem + kOffRing + st * kSlot;
        uint8_t* Y = X + kRaw;
        if (splitter) {  // ---------------- splitter ----------------
          mbar_wait(&br->raw_full[st], par2(it));
          if (ps == 0) {  // k~ masked (attention.cpp:334-343), V as it is
            SplitRow s;
            split_load(X, t, s);
            const int r = c * kRows + s.row;
            const float iv = rsqrtf(s.ss + eps);
            const bool f = r < N && tc::flag_at(fl, r);
            if (norms && r < N && s.qb == 0) norms[N + r] = f ? (s.ss + eps) * iv : 1.0f;
#pragma unroll
            for (int e = 0; e < 16; ++e) s.x[e] = f ? s.x[e] * iv : 0.f;  // NaN-safe zeros
            SplitRow v;
            split_load(Y, t, v);
            __syncwarp();
            split_store(X, X + 2 * kRaw, s);
            split_store(Y, X + 2 * kRaw + kPart, v);
          } else {
            split_q(X, t, eps, c * kRowsQ, N, norms);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&br->split_full[st]);
        } else {  // ---------------- epiloguer ----------------
          mbar_wait(&br->mma_done[st], par2(it));
          tc_fence_after();
          if (ps == 0) {
            arrive_staged(br, st, lane);  // a pass-1 item stages nothing: free the slot now
            if (c != C1 - 1 && c % kFlush == kFlush - 1) {  // long N: flush the accumulator
              flush_acc(tmem, lane_base, c == kFlush - 1);
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&br->acc_free);
            }
            if (c == C1 - 1) {  // S complete: saved S + the three part tiles
#pragma unroll 1
              for (int q = 0; q < 4; ++q) {
                float sv[32];
                acc_block(tmem, lane_base, q, C1 > kFlush, sv);
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
          } else {  // O rows = s (Q~ S), staged as four 64-row fp32 boxes over X | Y
            const int b = n1 & 1;
            const int row = 16 * wq + (lane & 15), h = lane >> 4;
            const uint32_t D = tmem + out_col(b) + lane_base;
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
              float o[32];
              tmem_ld_pair(D + 64u * hh, o);
              const int q = 2 * hh + h;
#pragma unroll
              for (int k2 = 0; k2 < 8; ++k2)
                *reinterpret_cast<float4*>(X + q * kBoxQ + goff(row, k2)) =
                    make_float4(o[4 * k2] * uc.s, o[4 * k2 + 1] * uc.s, o[4 * k2 + 2] * uc.s, o[4 * k2 + 3] * uc.s);
            }
            release_out(br, b, lane);
            ++n1;
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
__global__ void __launch_bounds__(kThreads, 1) cos_bwd_tcg_kernel(
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
      const int64_t sbytes = (int64_t)kD * kD * 4;
      const uint8_t* gS = static_cast<const uint8_t*>(p.saved_S);
      if (blockIdx.x < units) tc::bulk_prefetch_l2(gS + blockIdx.x * sbytes, (uint32_t)sbytes);
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        if (u + (int)gridDim.x < units) tc::bulk_prefetch_l2(gS + (u + gridDim.x) * sbytes, (uint32_t)sbytes);
        for (int ps = 0; ps < 2; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot2(it);
            tc::ItemPos f;
            if (p.l2_ahead && tc::item_pos(it + p.l2_ahead, 2, C, units, H, f))
              for (int hb = 0; hb < 4; ++hb) {
                tc::tma_prefetch_4d(f.ps == 0 ? &tq : &tk, 32 * hb, f.c * kRows, f.h, f.b);
                tc::tma_prefetch_4d(f.ps == 0 ? &tdo : &tv, 32 * hb, f.c * kRows, f.h, f.b);
              }
            mbar_wait(&br->slot_free[st], par2(it) ^ 1u);
            uint8_t* X = smem + kOffRing + st * kSlot;
            mbar_expect_tx(&br->raw_full[st], 2 * kRaw);
            for (int hb = 0; hb < 4; ++hb) {
              tma_load_4d(X + hb * kBox, ps == 0 ? &tq : &tk, 32 * hb, c * kRows, h, b, &br->raw_full[st]);
              tma_load_4d(X + kRaw + hb * kBox, ps == 0 ? &tdo : &tv, 32 * hb, c * kRows, h, b,
                          &br->raw_full[st]);
            }
          }
      }
    }
  } else if (warp == kWarpMma) {
    int it = 0, j = 0, nflush = 0, n1 = 0, n2 = 0;
    uint32_t par = 0;
    const uint32_t base = smem_u32(smem);
    const uint32_t opS[3] = {base + kOffOps, base + kOffOps + kStatePart, base + kOffOps + 2 * kStatePart};
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      for (int ps = 0; ps < 2; ++ps)
        for (int c = 0; c < C; ++c, ++it) {
          const int st = slot2(it);
          mbar_wait(&br->split_full[st], par2(it));
          TCG_TRACE(3, lane == 0);
          if (ps == 1 && c == 0) mbar_wait(&br->op_ready, j & 1);
          if (ps == 0 && c > 0 && c % kFlush == 0) mbar_wait(&br->acc_free, (nflush++) & 1);
          if (ps == 0 && c == 0) mbar_wait(&br->out_free[2], ((par >> 2) & 1u) ^ 1u);
          tc_fence_after();
          const uint32_t X = base + kOffRing + st * kSlot;
          const uint32_t xp[3] = {X, X + kPart, X + 2 * kRaw};
          const uint32_t yp[3] = {X + kRaw, X + kRaw + kPart, X + 2 * kRaw + kPart};
          if (ps == 0) {
            if (elect_one()) {  // G += Q~^T dO (attention.cpp:405)
              const int ks = (min(kRows, N - c * kRows) + 15) >> 4;
              issue_red(tmem + kAcc, xp, yp, ks, c % kFlush == 0);
            }
            __syncwarp();
            const int b = n1++ & 1;
            take_out(br, par, b);
            tc_fence_after();
            if (elect_one()) {
              issue_rowout<false>(tmem + out_col(b), yp, opS);  // dQ~ (unscaled) = dO S^T (:410-411)
              if (c == C - 1) mma_commit(&br->red_done);
              mma_commit(&br->mma_done[st]);
            }
            __syncwarp();
          } else {
            const int pr = (n2++ & 1) * 2;
            take_out(br, par, pr);
            tc_fence_after();
            if (elect_one()) issue_rowout<true>(tmem + out_col(pr), xp, opS);  // dV = K~ dA (:416)
            __syncwarp();
            take_out(br, par, pr + 1);
            tc_fence_after();
            if (elect_one()) {
              issue_rowout<false>(tmem + out_col(pr + 1), yp, opS);  // dK~ = V dA^T (:415)
              mma_commit(&br->mma_done[st]);
              if (c == C - 1) mma_commit(&br->ops_free);
            }
            __syncwarp();
          }
          TCG_TRACE(4, lane == 0);
        }
    }
  } else if (warp == kWarpMask) {
    tcg::mask_loop(p, smem, br, lane);
  } else if (warp == kWarpStore) {
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int b = u / H, h = u - b * H;
        for (int ps = 0; ps < 2; ++ps)
          for (int c = 0; c < C; ++c, ++it) {
            const int st = slot2(it);
            uint8_t* X = smem + kOffRing + st * kSlot;
            mbar_wait(&br->staged[st], par2(it));
            for (int hb = 0; hb < 4; ++hb) {
              if (ps == 0) {
                tma_store_4d(&tdq, X + hb * kBox, 32 * hb, c * kRows, h, b);
              } else {
                tma_store_4d(&tdk, X + hb * kBox, 32 * hb, c * kRows, h, b);
                tma_store_4d(&tdv, X + kRaw + hb * kBox, 32 * hb, c * kRows, h, b);
              }
            }
            bulk_wait_read0();
            mbar_arrive(&br->slot_free[st]);
            TCG_TRACE(7, true);
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
        const int st = slot2(it);
        uint8_t* X = smem + kOffRing + st * kSlot;
        uint8_t* Y = X + kRaw;
        uint8_t* X2 = X + 2 * kRaw;
        float* inv_st = invs + st * kRows;
        if (splitter) {  // ---------------- splitter ----------------
          if (ps == 0 && c == 0) {
            // this unit's S as three part tiles, once the last MMA reading the
            // previous unit's dA from the same area has completed
            if (j > 0) mbar_wait(&br->ops_free, (j - 1) & 1);
            const int a = t >> 1, hh = t & 1;
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
          TCG_TRACE(0, threadIdx.x == 0);
          mbar_wait(&br->raw_full[st], par2(it));
          TCG_TRACE(1, threadIdx.x == 0);
          SplitRow s, y;
          split_load(X, t, s);
          split_load(Y, t, y);
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
          if (s.qb == 0) inv_st[s.row] = iv;
          __syncwarp();
          split_store(X, X2, s);
          split_store(Y, X2 + kPart, y);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&br->split_full[st]);
          TCG_TRACE(2, threadIdx.x == 0);
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
          mbar_wait(&br->mma_done[st], par2(it));
          TCG_TRACE(5, t == 0);
          tc_fence_after();
          if (ps == 0 && c != C - 1 && c % kFlush == kFlush - 1) {  // long N: flush G
            flush_acc(tmem, lane_base, c == kFlush - 1);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&br->acc_free);
          }
          const int bv = (n2 & 1) * 2;  // pass 2: dV in bv, dK~ in bv + 1
          const int bg = ps == 0 ? (n1 & 1) : bv + 1;
          if (wq < 2) {
            const int row = 16 * wq + (lane & 15), h = lane >> 4;
            const int r = c * kRows + row;
            const float iv = inv_st[row];
            const uint32_t Dg = tmem + out_col(bg) + lane_base;
            // g = dQ~ or dK~, x~ = the part tiles rebuilt; pr = g . x~ over the row
            float pr = 0.f;
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
              float g[32], x[32];
              tmem_ld_pair(Dg + 64u * hh, g);
              row_block(X, X2, row, 2 * hh + h, x);
              pr += dot32(g, x);
            }
            pr += __shfl_xor_sync(0xffffffffu, pr, 16);
            if (ps == 0) {
              // dQ_i = (g - (g.q~_i) q~_i) / nq_i, g = s dO S^T (:410-411, :421-428); staged over X
              float g0[32], g1[32];
              {
                float x[32];
                tmem_ld_pair(Dg, g0);
                row_block(X, X2, row, h, x);
#pragma unroll
                for (int e = 0; e < 32; ++e) g0[e] = (uc.s * g0[e] - uc.s * pr * x[e]) * iv;
                tmem_ld_pair(Dg + 64u, g1);
                row_block(X, X2, row, 2 + h, x);
#pragma unroll
                for (int e = 0; e < 32; ++e) g1[e] = (uc.s * g1[e] - uc.s * pr * x[e]) * iv;
              }
              __syncwarp();  // the row's parts are read (by both of its threads) before X is overwritten
              stage_block(X, row, h, g0);
              stage_block(X, row, 2 + h, g1);
            } else {
              const bool f = r < N && tc::flag_at(fl, r);
              const bool nan_out = uc.tn == 0;
              // dK_i = v_i ? (g - (g.k~)k~) / nk : 0 (:430-437), staged over X
              float g0[32], g1[32];
              {
                float x[32];
                tmem_ld_pair(Dg, g0);
                row_block(X, X2, row, h, x);
#pragma unroll
                for (int e = 0; e < 32; ++e) g0[e] = nan_out ? qnan : (f ? (g0[e] - pr * x[e]) * iv : 0.f);
                tmem_ld_pair(Dg + 64u, g1);
                row_block(X, X2, row, 2 + h, x);
#pragma unroll
                for (int e = 0; e < 32; ++e) g1[e] = nan_out ? qnan : (f ? (g1[e] - pr * x[e]) * iv : 0.f);
              }
              __syncwarp();
              stage_block(X, row, h, g0);
              stage_block(X, row, 2 + h, g1);
              // dV_i = v_i ? (K~ dA)_i : 0 (:416, :439), staged over Y (V's parts are done)
              const uint32_t Dv = tmem + out_col(bv) + lane_base;
#pragma unroll 1
              for (int hh = 0; hh < 2; ++hh) {
                float g[32];
                tmem_ld_pair(Dv + 64u * hh, g);
#pragma unroll
                for (int e = 0; e < 32; ++e) g[e] = nan_out ? qnan : (f ? g[e] : 0.f);
                stage_block(Y, row, 2 * hh + h, g);
              }
            }
          }
          if (ps == 0) {
            release_out(br, bg, lane);
            ++n1;
          } else {
            release_out(br, bg, lane);
            release_out(br, bv, lane);
            ++n2;
          }
          arrive_staged(br, st, lane);
          TCG_TRACE(6, t == 0);
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

}  // namespace tcg

// ---- host side ----------------------------------------------------------------------

// 4-D fp32 map over (128, N, H, B), box (32, 32, 1, 1), 128-byte swizzle: four boxes per row
inline bool make_tcg_map(CUtensorMap* map, const void* base, const OpParams& p, int rows = tcg::kRows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {128, (cuuint64_t)p.N, (cuuint64_t)p.H, (cuuint64_t)p.B};
  cuuint64_t strides[3] = {(cuuint64_t)p.sn * 4, (cuuint64_t)p.sh * 4, (cuuint64_t)p.sb * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
inline bool tcg_layout_ok(const OpParams& p, std::initializer_list<const void*> ptrs) {
  if (p.D != 128 || p.N < 1 || p.N > tcg::kMaxN) return false;
  if ((p.sn * 4) % 16 || (p.sh * 4) % 16 || (p.sb * 4) % 16) return false;
  if (p.B * p.H > (1ll << 31) - 1) return false;
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<uintptr_t>(q) & 15)) return false;
  return encode_fn() != nullptr && getenv("COTTEN_NO_TCG") == nullptr;
}
template <typename T>
inline bool tcg_fwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, float>::value) {
    return false;
  } else {
    return tcg_layout_ok(p, {p.q, p.k, p.v, p.out});
  }
}
template <typename T>
inline bool tcg_bwd_supported(const OpParams& p) {
  if constexpr (!std::is_same<T, float>::value) {
    return false;
  } else {
    return p.saved_S != nullptr && tcg_layout_ok(p, {p.q, p.k, p.v, p.dout, p.dq, p.dk, p.dv});
  }
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_tcg_pdl(void (*kern)(KArgs...), int grid, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tcg::kThreads);
  cfg.dynamicSmemBytes = tcg::kSmemBytes;
  cfg.stream = st;
  static const bool pdl = getenv("COTTEN_NO_PDL") == nullptr;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
inline int launch_tcg_fwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mo;
  if (!make_tcg_map(&mq, p.q, p, tcg::kRowsQ) || !make_tcg_map(&mk, p.k, p) || !make_tcg_map(&mv, p.v, p) ||
      !make_tcg_map(&mo, p.out ? p.out : p.q, p, tcg::kRowsQ))
    return -1;
  if (cudaFuncSetAttribute(tcg::cos_fwd_tcg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tcg::kSmemBytes) != cudaSuccess)
    return -1;
  const int grid = std::min((int)(p.B * p.H), sm_count());
  OpParams q = p;
  q.l2_ahead = l2_ahead_items(true, (int)((p.N + 63) / 64));
  if (launch_tcg_pdl(tcg::cos_fwd_tcg_kernel, grid, st, mq, mk, mv, mo, q) != cudaSuccess) return -1;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}
inline int launch_tcg_bwd(const OpParams& p, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mg, mdq, mdk, mdv;
  if (!make_tcg_map(&mq, p.q, p) || !make_tcg_map(&mk, p.k, p) || !make_tcg_map(&mv, p.v, p) ||
      !make_tcg_map(&mg, p.dout, p) || !make_tcg_map(&mdq, p.dq, p) || !make_tcg_map(&mdk, p.dk, p) ||
      !make_tcg_map(&mdv, p.dv, p))
    return -1;
  if (cudaFuncSetAttribute(tcg::cos_bwd_tcg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tcg::kSmemBytes) != cudaSuccess)
    return -1;
  const int grid = std::min((int)(p.B * p.H), sm_count());
  OpParams q = p;
  q.l2_ahead = l2_ahead_items();
#if COTTEN_TCG_TRACE
  static void* tbuf = nullptr;
  if (!tbuf) cudaMalloc(&tbuf, (size_t)1024 * tcb::kTraceItems * 8 * sizeof(long long));
  cudaMemsetAsync(tbuf, 0, (size_t)grid * tcb::kTraceItems * 8 * sizeof(long long), st);
  q.workspace = tbuf;
#endif
  if (launch_tcg_pdl(tcg::cos_bwd_tcg_kernel, grid, st, mq, mk, mv, mg, mdq, mdk, mdv, q) != cudaSuccess)
    return -1;
#if COTTEN_TCG_TRACE
  if (const char* dir = getenv("COTTEN_TRACE_DIR")) {
    std::vector<long long> h((size_t)grid * tcb::kTraceItems * 8);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), tbuf, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    if (FILE* f = fopen((std::string(dir) + "/tcg_bwd.bin").c_str(), "wb")) {
      fwrite(h.data(), sizeof(long long), h.size(), f);
      fclose(f);
    }
  }
#endif
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace cotten
