// tcgen05.ld .16x32bx2 probe: does lane l >= 16 of a warp read lane (l - 16) of the
// warp's subpartition at columns + immHalfSplitoff?  (M = 64 accumulators use lanes
// 0-15 of each subpartition; this would let 32 threads share the 16 rows.)
#include <cstdio>
#include <cstdint>
__global__ void probe(float* out) {
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t lb = (uint32_t)(32 * warp) << 16;
  for (int c = 0; c < 64; ++c) {  // lane L = t, column c = 1000 L + c
    const float v = 1000.f * t + c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lb + c), "r"(__float_as_uint(v)) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], 32;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(tmem + lb));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int c = 0; c < 32; ++c) out[t * 32 + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  (void)lane;
}
int main() {
  float* d;
  cudaMalloc(&d, 128 * 32 * 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  static float h[128 * 32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(e));
  int bad = 0;
  for (int t = 0; t < 128; ++t) {
    const int w = t / 32, l = t % 32;
    const int lane = 32 * w + (l & 15), col0 = (l >= 16) ? 32 : 0;
    for (int c = 0; c < 32; ++c)
      if (h[t * 32 + c] != 1000.f * lane + col0 + c) ++bad;
  }
  printf("thread 17: %g %g ... ; thread 1: %g; mismatches vs (lane 32w + l%%16, col + 32 (l >= 16)): %d\n",
         h[17 * 32], h[17 * 32 + 1], h[1 * 32], bad);
  return 0;
}
