// Does tcgen05.mma kind::tf32 truncate, round, or keep the low mantissa bits of fp32 operands?
#include <cstdio>
#include "../../paper_2602_06935_b200/csrc/kernels_tc.cuh"
using namespace cotten;
using namespace cotten::tc;
__global__ void probe(const float* a_vals, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  // A: 128 rows x 32 (K-major SW128), row m: element k=0 is a_vals[m % 8], rest 0.  B: 32 rows (n), element k=0 = 1.
  for (int i = t; i < 128 * 32; i += blockDim.x) {
    const int r = i / 32, c = i % 32;
    *reinterpret_cast<float*>(smem + elem_off(r, c)) = (c == 0) ? a_vals[r % 8] : 0.f;
  }
  for (int i = t; i < 32 * 32; i += blockDim.x) {
    const int r = i / 32, c = i % 32;
    *reinterpret_cast<float*>(smem + 16384 + elem_off(r, c)) = (c == 0) ? 1.f : 0.f;
  }
  if (t == 0) { mbar_init(&bar, 1); d32::fence_barrier_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async(); tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot, b = smem_u32(smem);
  if (warp == 0 && elect_one()) {
    mma_tf32(tmem, sdesc(b, 16, 1024), sdesc(b + 16384, 16, 1024), idesc_tf32(128, 32, false, false), 0);
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  float r[32];
  tmem_ld32(tmem + ((32 * warp) << 16), r);
  tmem_wait_ld();
  if (t < 8) out[t] = r[0];
  tc_fence_before(); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}
int main() {
  float h[8] = {1.0f + 0x1p-11f + 0x1p-12f, 1.0f + 0x1p-11f, 1.0f + 0x1p-12f, 1.0f + 0x1p-10f + 0x1p-11f,
                -(1.0f + 0x1p-11f + 0x1p-12f), 1.0f + 0x1.fffp-11f, 3.0f + 0x1p-10f, 1.0f};
  float *d, *o; cudaMalloc(&d, 32); cudaMalloc(&o, 32);
  cudaMemcpy(d, h, 32, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  probe<<<1, 128, 32768>>>(d, o);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  float r[8]; cudaMemcpy(r, o, 32, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 8; ++i) {
    unsigned in, outb; memcpy(&in, &h[i], 4); memcpy(&outb, &r[i], 4);
    unsigned tr = in & 0xFFFFE000u, rn = (in + 0x1000u) & 0xFFFFE000u;
    printf("in %a -> %a   (trunc %s, rn %s, exact %s)\n", h[i], r[i], outb == tr ? "Y" : "n", outb == rn ? "Y" : "n", outb == in ? "Y" : "n");
  }
  return 0;
}
