// tcgen05 kind::tf32 layout probe: K-major / MN-major operands, M=64 / M=128.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../../paper_2602_06935_b200/csrc/kernels_tc.cuh"
using namespace cotten;
using namespace cotten::tc;

// smem: 6 tiles of 128 rows x 32 fp32 (16 KB each), tile i filled from src[i*4096 ..] with
// element (r, c) at elem_off(r, c) in tile i.
__global__ void probe(const float* src, float* out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 6 * 4096; i += blockDim.x) {
    int tile = i / 4096, r = (i % 4096) / 32, c = i % 32;
    *reinterpret_cast<float*>(smem + tile * 16384 + elem_off(r, c)) = src[i];
  }
  if (t == 0) { mbar_init(&bar, 1); d32::fence_barrier_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t b = smem_u32(smem);
  const uint32_t T = 16384;
  if (t == 0) {
    if (mode == 0) {  // K-major A (tile0, 64 rows) x K-major B (tile4, 64 rows), M=64 N=64, K=32
      const uint32_t id = idesc_tf32(64, 64, false, false);
      for (int kk = 0; kk < 4; ++kk) mma_tf32(tmem, sdesc(b + 32 * kk, 16, 1024), sdesc(b + 4 * T + 32 * kk, 16, 1024), id, kk > 0);
    } else if (mode == 1) {  // MN-major A (tiles 0..3, LBO 16K), K-major... no: B MN-major? keep B K-major tile4 (32 rows), M=128 N=32, K=8 rows? K of B-Kmajor is columns: use K=32 via 4 steps
      // A[m][k]: MN-major: k = row of tile, m = 32*tile + col.  K steps over 8 rows (1024 B).
      // B[k][n]: K-major: row n of tile4, column k. K=8 per step -> columns 8kk..8kk+7 = 32 B offset.
      const uint32_t id = idesc_tf32(128, 32, true, false);
      for (int kk = 0; kk < 4; ++kk) mma_tf32(tmem, sdesc(b + 1024 * kk, T, 1024), sdesc(b + 4 * T + 32 * kk, 16, 1024), id, kk > 0);
    } else if (mode == 2) {  // K-major A tile0 (128 rows), MN-major B tiles 4,5 (LBO 16K) N=64: B[k][n] = tile(4+n/32)[k][n%32], k = row
      const uint32_t id = idesc_tf32(128, 64, false, true);
      for (int kk = 0; kk < 4; ++kk) mma_tf32(tmem, sdesc(b + 32 * kk, 16, 1024), sdesc(b + 4 * T + 1024 * kk, T, 1024), id, kk > 0);
    } else {  // MN-major A (tiles 0,1), MN-major B (tiles 4,5), M=64 N=64, K = 32 rows
      const uint32_t id = idesc_tf32(64, 64, true, true);
      for (int kk = 0; kk < 4; ++kk) mma_tf32(tmem, sdesc(b + 1024 * kk, T, 1024), sdesc(b + 4 * T + 1024 * kk, T, 1024), id, kk > 0);
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  float r[32], r2[32];
  tmem_ld32(tmem + ((32 * warp) << 16), r);
  tmem_ld32(tmem + ((32 * warp) << 16) + 32, r2);
  tmem_wait_ld();
  for (int c = 0; c < 32; ++c) { out[t * 64 + c] = r[c]; out[t * 64 + 32 + c] = r2[c]; }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

static float* H;
static float tile(int i, int r, int c) { return H[i * 4096 + r * 32 + c]; }

int main() {
  const int n = 6 * 4096;
  H = (float*)malloc(n * 4);
  float* hO = (float*)malloc(128 * 64 * 4);
  srand(1);
  for (int i = 0; i < n; ++i) H[i] = (rand() % 17 - 8) / 8.0f;
  float *dS, *dO;
  cudaMalloc(&dS, n * 4); cudaMalloc(&dO, 128 * 64 * 4);
  cudaMemcpy(dS, H, n * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16384);
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(dO, 0, 128 * 64 * 4);
    probe<<<1, 128, 6 * 16384>>>(dS, dO, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hO, dO, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    int M = (mode == 0 || mode == 3) ? 64 : 128, N = (mode == 1) ? 32 : 64;
    // expected D[m][nn]
    static double D[128][64];
    for (int m = 0; m < M; ++m) for (int nn = 0; nn < N; ++nn) {
      double s = 0;
      for (int k = 0; k < 32; ++k) {
        double a, bb;
        if (mode == 0 || mode == 2) a = tile(0, m, k); else a = tile(m / 32, k, m % 32);
        if (mode == 0 || mode == 1) bb = tile(4, nn, k); else bb = tile(4 + nn / 32, k, nn % 32);
        s += a * bb;
      }
      D[m][nn] = s;
    }
    printf("mode %d (%s) M=%d N=%d\n", mode, cudaGetErrorString(e), M, N);
    // for each m: which lane matches row m (over all N columns)?
    int shown = 0;
    for (int m = 0; m < M; ++m) {
      int best = -1; double be = 1e30;
      for (int l = 0; l < 128; ++l) { double er = 0; for (int c = 0; c < N; ++c) er = fmax(er, fabs(D[m][c] - hO[l * 64 + c])); if (er < be) { be = er; best = l; } }
      if (m < 4 || m % 16 == 0 || m % 16 == 15 || be > 1e-6) { if (shown++ < 40) printf("   m=%3d -> lane %3d err %g\n", m, best, be); }
    }
  }
  return 0;
}
