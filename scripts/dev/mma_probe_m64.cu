// tcgen05 kind::tf32 probe: M = 64 MMAs at TMEM lane offset 16 (the
// "half-subpartition" data-path layout: row m at lane off + (m % 16) + 32 (m / 16)).
//   mode 0/1: SS reduction (MN-major A, B in the 32-byte-granule swizzle), M=64 N=64 K=32, D at lane off 0 / 16
//   mode 2/3: TS row output, A from TMEM (lane = row), B K-major, M=64 N=32 K=32, A and D at lane off 0 / 16
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../../paper_2602_06935_b200/csrc/kernels_tc.cuh"
using namespace cotten;
using namespace cotten::tc;

__device__ __forceinline__ uint64_t sdesc_t(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t type) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)type << 61);
}
__device__ __forceinline__ uint32_t off32(int r, int c) {
  return (uint32_t)r * 128u + ((uint32_t)(((c >> 3) ^ (r & 3))) << 5) + (uint32_t)(c & 7) * 4u;
}

__global__ void probe(const float* src, float* out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  const bool ts = mode >= 2;
  const uint32_t off = (mode & 1) ? 16u : 0u;
  for (int i = t; i < 6 * 4096; i += blockDim.x) {
    int tile = i / 4096, r = (i % 4096) / 32, c = i % 32;
    uint32_t o = ts ? elem_off(r, c) : off32(r, c);
    *reinterpret_cast<float*>(smem + tile * 16384 + o) = src[i];
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
  {  // zero the D columns, and (ts) lane L of cols 128..159 = tile0 row L
    float z[32], v[32];
    for (int c = 0; c < 32; ++c) { z[c] = 0.f; v[c] = src[t * 32 + c]; }
    tmem_st32(tmem + ((32 * warp) << 16), z);
    tmem_st32(tmem + ((32 * warp) << 16) + 32, z);
    tmem_st32(tmem + ((32 * warp) << 16) + 128, v);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const uint32_t b = smem_u32(smem);
  const uint32_t T = 16384;
  if (t == 0) {
    if (!ts) {
      const uint32_t id = idesc_tf32(64, 64, true, true);
      for (int kk = 0; kk < 4; ++kk)
        mma_tf32(tmem + (off << 16), sdesc_t(b + 1024 * kk, T, 512, 1), sdesc_t(b + 4 * T + 1024 * kk, T, 512, 1), id, kk > 0);
    } else {
      const uint32_t id = idesc_tf32(64, 32, false, false);
      for (int kk = 0; kk < 4; ++kk)
        mma_tf32_ts(tmem + (off << 16), tmem + (off << 16) + 128 + 8 * kk, sdesc(b + 4 * T + 32 * kk, 16, 1024), id,
                    (uint32_t)(kk > 0));
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
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
  int fails = 0;
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(dO, 0, 128 * 64 * 4);
    probe<<<1, 128, 6 * 16384>>>(dS, dO, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hO, dO, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    const bool ts = mode >= 2;
    const int off = (mode & 1) ? 16 : 0;
    const int M = 64, N = ts ? 32 : 64;
    double maxerr = 0, other = 0;
    bool used[128] = {};
    for (int m = 0; m < M; ++m) {
      const int lane = off + (m % 16) + 32 * (m / 16);
      used[lane] = true;
      for (int nn = 0; nn < N; ++nn) {
        double s = 0;
        for (int k = 0; k < 32; ++k) {
          double a = ts ? tile(0, lane, k) : tile(m / 32, k, m % 32);
          double bb = ts ? tile(4, nn, k) : tile(4 + nn / 32, k, nn % 32);
          s += a * bb;
        }
        maxerr = fmax(maxerr, fabs(s - hO[lane * 64 + nn]));
      }
    }
    for (int l = 0; l < 128; ++l)
      if (!used[l]) for (int c = 0; c < 64; ++c) other = fmax(other, fabs(hO[l * 64 + c]));
    printf("mode %d (%s, lane off %d): maxerr %g, max |other lanes| %g\n", mode, ts ? "TS M64 N32" : "SS M64 N64",
           off, maxerr, other);
    if (e != cudaSuccess) { printf("  %s\n", cudaGetErrorString(e)); return 1; }
    fails += maxerr > 1e-3 || other != 0;
  }
  printf(fails ? "FAIL\n" : "ALL OK\n");
  return 0;
}
