// tcgen05 issue-rate probe: cycles per MMA for the shapes the kernels use.
#include <cstdio>
#include "../../paper_2602_06935_b200/csrc/kernels_tc.cuh"
using namespace cotten;
using namespace cotten::tc;

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred P1;\nelect.sync _|P1, 0xffffffff;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(pred));
  return pred != 0;
}
template <int mode>
__global__ void rate(long long* out, int n) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i & 255);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); d32::fence_barrier_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot, b = smem_u32(smem);
  if (warp == 0) {
    const bool leader = elect_one();
    long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < n; ++i) {
      if (!leader) continue;
      const uint32_t kk = i & 3;
      switch (mode) {  // compile-time
        case 0: mma_tf32(tmem, sdesc(b + 32 * kk, 16, 1024), sdesc(b + 32768 + 32 * kk, 16, 1024), idesc_tf32(128, 32, false, false), 1); break;
        case 1: mma_tf32_ts(tmem, tmem + 256 + 8 * kk, sdesc(b + 32768 + 32 * kk, 16, 1024), idesc_tf32(128, 32, false, false), 1); break;
        case 2: mma_tf32(tmem, sdesc(b + 1024 * kk, 16384, 512, 1), sdesc(b + 32768 + 1024 * kk, 16384, 512, 1), idesc_tf32(64, 64, true, true), 1); break;
        case 3: mma_tf32(tmem, sdesc(b + 32 * kk, 16, 1024), sdesc(b + 32768 + 32 * kk, 16, 1024), idesc_tf32(128, 64, false, false), 1); break;
        case 4: mma_tf32(tmem, sdesc(b + 32 * kk, 16, 1024), sdesc(b + 32768 + 32 * kk, 16, 1024), idesc_tf32(128, 128, false, false), 1); break;
        case 5: mma_tf32(tmem, sdesc(b + 32 * kk, 16, 1024), sdesc(b + 32768 + 32 * kk, 16, 1024), idesc_tf32(128, 256, false, false), 1); break;
        case 6: mma_f16(tmem, sdesc(b + 32 * kk, 16, 1024), sdesc(b + 32768 + 32 * kk, 16, 1024), (1u << 4) | (1u << 7) | (1u << 10) | (4u << 17) | (8u << 24), 1); break;  // bf16 M128 N32 K16
        case 7: mma_tf32(tmem, sdesc(b + 1024 * kk, 16, 1024), sdesc(b + 32768 + 32 * kk, 16, 1024), idesc_tf32(64, 32, false, false), 1); break;
        case 8: mma_tf32_ts(tmem, tmem + 256 + 8 * kk, sdesc(b + 32768 + 32 * kk, 16, 1024), idesc_tf32(128, 64, false, false), 1); break;
        case 9: mma_tf32(tmem, sdesc(b + 1024 * kk, 16384, 512, 1), sdesc(b + 32768 + 1024 * kk, 16384, 512, 1), idesc_tf32(128, 64, true, true), 1); break;
        case 10: mma_tf32(tmem + 32 * (i & 7), sdesc(b + 32 * kk, 16, 1024), sdesc(b + 32768 + 32 * kk, 16, 1024), idesc_tf32(128, 32, false, false), 1); break;
        case 11: mma_tf32_ts(tmem + 32 * (i & 7), tmem + 256 + 8 * kk, sdesc(b + 32768 + 32 * kk, 16, 1024), idesc_tf32(128, 32, false, false), 1); break;
        case 12: mma_tf32(tmem, sdesc(b + 32 * kk, 16, 1024), sdesc(b + 32768 + 32 * kk, 16, 1024), idesc_tf32(128, 32, false, false), 0); break;
        case 13: mma_tf32(tmem + 64 * (i & 3), sdesc(b + 1024 * kk, 16384, 512, 1), sdesc(b + 32768 + 1024 * kk, 16384, 512, 1), idesc_tf32(64, 64, true, true), 1); break;
        case 14: mma_f16(tmem + 256 * (i & 1), sdesc(b + 32 * kk, 16, 1024), sdesc(b + 32768 + 32 * kk, 16, 1024), (1u << 4) | (1u << 7) | (1u << 10) | (32u << 17) | (8u << 24), 1); break;  // bf16 M128 N256 K16, 2 accs
      }
    }
    __syncwarp();
    long long t1 = clock64();
    if (leader) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (leader) { out[mode * 2] = t1 - t0; out[mode * 2 + 1] = t2 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d; cudaMalloc(&d, 64 * 8);

  const char* names[] = {"SS tf32 M128 N32 K-major", "TS tf32 M128 N32", "SS tf32 M64 N64 MN-major(32B)", "SS tf32 M128 N64",
                         "SS tf32 M128 N128", "SS tf32 M128 N256", "SS bf16 M128 N32 K16", "SS tf32 M64 N32", "TS tf32 M128 N64", "SS tf32 M128 N64 MN-major", "SS M128N32 8 accs", "TS M128N32 8 accs", "SS M128N32 acc=0", "SS M64N64 MN 4 accs", "bf16 M128N256 2 accs"};
  const int n = 2000;
  void (*ks[15])(long long*, int) = {rate<0>, rate<1>, rate<2>, rate<3>, rate<4>, rate<5>, rate<6>, rate<7>, rate<8>, rate<9>, rate<10>, rate<11>, rate<12>, rate<13>, rate<14>};
  for (int mode = 0; mode < 15; ++mode) {
    cudaFuncSetAttribute(ks[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    ks[mode]<<<1, 128, 65536>>>(d, n);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[64]; cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
    printf("%-32s issue %6.1f  total %6.1f cyc/MMA  (%s)\n", names[mode], (double)h[mode * 2] / n, (double)h[mode * 2 + 1] / n, cudaGetErrorString(e));
  }
  return 0;
}
