// tcgen05 kind::f16 (bf16 operands, fp32 accumulate) probe: the descriptor
// conventions the bf16 tensor-core kernels (kernels_tcb.cuh) rely on.
//   tiles: 128 rows x 128 B (64 bf16), SWIZZLE_128B (16-byte granule j of row r
//   at j ^ (r & 7)); tile i at smem + i * 16 KB.
//   mode 0/1: MN-major A (tiles 0[,1] = M atoms) x MN-major B (tiles 4[,5]),
//             K = 32 rows (2 x K16): the S = K~^T V reduction; M = N = 64 (one
//             atom) or 128 (two atoms, LBO = 16 KB); SBO variants.
//   mode 2:   K-major A (tile 0: 128 rows x K=64) x K-major B (tile 4 rows =
//             N = 64) -> M = 128, N = 64: the row outputs with B = S^T rows.
//   mode 3:   K-major A x MN-major B (tile 4 rows = K = 64, N = 64).
//   mode 4:   mode 2 with N = 128, K = 128 (A = tiles 0,1 as two K panels,
//             B = tiles 4,5 rows 0..127 as K panels) — the d_h = 128 row output.
#include <cuda_bf16.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "../../paper_2602_06935_b200/csrc/kernels_tc.cuh"
using namespace cotten;
using namespace cotten::tc;

__device__ __forceinline__ uint64_t sd(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t type) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)type << 61);
}
__host__ __device__ inline uint32_t off16(int r, int c) {  // bf16 element (r, c) of a SW128 tile
  return (uint32_t)r * 128u + ((uint32_t)((c >> 3) ^ (r & 7)) << 4) + (uint32_t)(c & 7) * 2u;
}
__device__ __forceinline__ uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void probe(const __nv_bfloat16* src, float* out, int mode, int variant) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 6 * 8192; i += blockDim.x) {
    const int tile = i / 8192, r = (i % 8192) / 64, c = i % 64;
    *reinterpret_cast<__nv_bfloat16*>(smem + tile * 16384 + off16(r, c)) = src[i];
  }
  if (t == 0) { mbar_init(&bar, 1); d32::fence_barrier_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t b = smem_u32(smem), T = 16384;
  if (t == 0) {
    if (mode <= 1) {
      const int M = mode == 0 ? 64 : 128;
      uint32_t lbo = T, sbo = 1024;
      if (variant == 1) { lbo = 1024; sbo = T; }
      const uint32_t id = idesc_bf16(M, M, true, true);
      for (int kk = 0; kk < 2; ++kk)  // K16 step = 16 rows = 2 KB
        mma_f16(tmem, sd(b + 2048u * kk, lbo, sbo, 2), sd(b + 4 * T + 2048u * kk, lbo, sbo, 2), id, kk > 0);
    } else if (mode == 2 || mode == 3) {
      const bool bmn = mode == 3;
      const uint32_t id = idesc_bf16(128, 64, false, bmn);
      uint32_t lbo = T, sbo = 1024;
      if (variant == 1) { lbo = 1024; sbo = T; }
      for (int kk = 0; kk < 4; ++kk) {  // K = 64 = 4 x 16 (32 B along the row)
        const uint64_t bd = bmn ? sd(b + 4 * T + 2048u * kk, lbo, sbo, 2) : sd(b + 4 * T + 32u * kk, 16, 1024, 2);
        mma_f16(tmem, sd(b + 32u * kk, 16, 1024, 2), bd, id, kk > 0);
      }
    } else {  // mode 4: M=128, N=128, K=128: K panels 0/1 (A tiles 0,1; B tiles 4,5)
      const uint32_t id = idesc_bf16(128, 128, false, false);
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t pa = b + (kk >> 2) * T + 32u * (kk & 3);
        const uint32_t pb = b + 4 * T + (kk >> 2) * T + 32u * (kk & 3);
        mma_f16(tmem, sd(pa, 16, 1024, 2), sd(pb, 16, 1024, 2), id, kk > 0);
      }
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int h = 0; h < 4; ++h) {
    float r[32];
    tmem_ld32(tmem + ((32 * warp) << 16) + 32 * h, r);
    tmem_wait_ld();
    for (int c = 0; c < 32; ++c) out[t * 128 + 32 * h + c] = r[c];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

static float HF[6 * 8192];
static float tl(int i, int r, int c) { return HF[i * 8192 + r * 64 + c]; }

int main() {
  const int n = 6 * 8192;
  __nv_bfloat16* H = (__nv_bfloat16*)malloc(n * 2);
  float* hO = (float*)malloc(128 * 128 * 4);
  srand(1);
  for (int i = 0; i < n; ++i) {
    HF[i] = (rand() % 17 - 8) / 8.0f;
    H[i] = __float2bfloat16(HF[i]);
  }
  __nv_bfloat16* dS;
  float* dO;
  cudaMalloc(&dS, n * 2);
  cudaMalloc(&dO, 128 * 128 * 4);
  cudaMemcpy(dS, H, n * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16384);
  const int cases[][2] = {{0, 0}, {0, 1}, {1, 0}, {1, 1}, {2, 0}, {3, 0}, {3, 1}, {4, 0}};
  for (auto& cs : cases) {
    const int mode = cs[0], var = cs[1];
    cudaMemset(dO, 0, 128 * 128 * 4);
    probe<<<1, 128, 6 * 16384>>>(dS, dO, mode, var);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hO, dO, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    int M = 128, N = 64, K = 64;
    if (mode == 0) { M = 64; N = 64; K = 32; }
    if (mode == 1) { M = 128; N = 128; K = 32; }
    if (mode == 4) { N = 128; K = 128; }
    double maxerr = 0, ref00 = 0;
    for (int m = 0; m < M; ++m)
      for (int nn = 0; nn < N; ++nn) {
        double s = 0;
        for (int k = 0; k < K; ++k) {
          double a, bb;
          if (mode <= 1) { a = tl(m / 64, k, m % 64); bb = tl(4 + nn / 64, k, nn % 64); }
          else if (mode == 2) { a = tl(0, m, k); bb = tl(4, nn, k); }
          else if (mode == 3) { a = tl(0, m, k); bb = tl(4, k, nn); }
          else { a = tl(k / 64, m, k % 64); bb = tl(4 + k / 64, nn, k % 64); }
          s += a * bb;
        }
        if (m == 0 && nn == 0) ref00 = s;
        const int lane = (M == 64) ? (m % 16) + 32 * (m / 16) : m;
        maxerr = fmax(maxerr, fabs(s - hO[lane * 128 + nn]));
      }
    printf("mode %d var %d (%s): maxerr %g  D00 %g got %g\n", mode, var, cudaGetErrorString(e), maxerr,
           ref00, hO[0]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
