// tcgen05 kind::f16 probe for the d_h = 128 bf16 kernels (kernels_tch.cuh):
//   mode 0: reduction R = X^T Y, M = N = 128 (two 64-feature SW128 atoms per
//           operand, LBO = 8 KB), K = 64 rows, both MN-major
//   mode 1: row output O = X S, M = 64 rows, N = 128, K = 128; A K-major (two
//           half-tiles), B MN-major (state half-tiles, LBO = 16 KB)
//   mode 2: row output O = X S^T, B K-major (N = 128 state rows)
// Values are multiples of 1/16 in [-1/2, 1/2], so every sum is exact in fp32.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mma_probe_d128 mma_probe_d128.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2602_06935_b200/csrc/kernels_tcb.cuh"
using namespace cotten;
using cotten::tc::elect_one; using cotten::tc::fence_proxy_async; using cotten::tc::tc_fence_before; using cotten::tc::tc_fence_after; using cotten::tc::mma_commit; using cotten::tc::tmem_ld32; using cotten::tc::tmem_wait_ld;
using cotten::tcb::goff;
using cotten::tcb::idesc_bf16;
using cotten::tcb::mma_bf16;
using cotten::tcb::sdesc;

constexpr uint32_t kHalf = 8192, kStateHalf = 16384;

__global__ void probe(const float* x, const float* y, const float* s, float* out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  uint8_t* X = smem;
  uint8_t* Y = smem + 2 * kHalf;
  uint8_t* S = smem + 4 * kHalf;
  for (int i = t; i < 64 * 128; i += blockDim.x) {
    const int r = i / 128, c = i % 128;
    const uint32_t o = (c >> 6) * kHalf + goff(r, (c & 63) >> 3) + (c & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(X + o) = __float2bfloat16_rn(x[i]);
    *reinterpret_cast<__nv_bfloat16*>(Y + o) = __float2bfloat16_rn(y[i]);
  }
  for (int i = t; i < 128 * 128; i += blockDim.x) {
    const int r = i / 128, c = i % 128;
    const uint32_t o = (c >> 6) * kStateHalf + goff(r, (c & 63) >> 3) + (c & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(S + o) = __float2bfloat16_rn(s[i]);
  }
  if (t == 0) {
    d32::mbar_init(&bar, 1);
    d32::fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(d32::smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t bx = d32::smem_u32(X), by = d32::smem_u32(Y), bs = d32::smem_u32(S);
  if (warp == 0) {
    if (elect_one()) {
      if (mode == 0) {
        const uint32_t id = idesc_bf16(128, 128, true, true);
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16(tmem, sdesc(bx + 2048u * kk, kHalf, 1024u), sdesc(by + 2048u * kk, kHalf, 1024u), id,
                   kk > 0 ? 1u : 0u);
      } else {
        const bool bmn = mode == 1;
        const uint32_t id = idesc_bf16(64, 128, false, bmn);
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = sdesc(bx + (kk >> 2) * kHalf + 32u * (kk & 3), 16u, 1024u);
          const uint64_t bd = bmn ? sdesc(bs + 2048u * kk, kStateHalf, 1024u)
                                  : sdesc(bs + (kk >> 2) * kStateHalf + 32u * (kk & 3), 16u, 1024u);
          mma_bf16(tmem, ad, bd, id, kk > 0 ? 1u : 0u);
        }
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  d32::mbar_wait(&bar, 0);
  tc_fence_after();
  for (int q = 0; q < 4; ++q) {
    float r[32];
    tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + 32u * q, r);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) out[t * 128 + 32 * q + e] = r[e];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  std::vector<float> x(64 * 128), y(64 * 128), s(128 * 128);
  srand(1);
  auto rv = [] { return (float)((rand() % 17) - 8) / 16.f; };
  for (auto& v : x) v = rv();
  for (auto& v : y) v = rv();
  for (auto& v : s) v = rv();
  float *dx, *dy, *ds, *dout;
  cudaMalloc(&dx, x.size() * 4);
  cudaMalloc(&dy, y.size() * 4);
  cudaMalloc(&ds, s.size() * 4);
  cudaMalloc(&dout, 128 * 128 * 4);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, y.data(), y.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, s.data(), s.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 4 * kHalf + 2 * kStateHalf + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int bad_total = 0;
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(dout, 0, 128 * 128 * 4);
    probe<<<1, 128, smem>>>(dx, dy, ds, dout, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> o(128 * 128);
    cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    if (mode == 0) {
      for (int a = 0; a < 128; ++a)
        for (int b = 0; b < 128; ++b) {
          double ref = 0;
          for (int r = 0; r < 64; ++r) ref += (double)x[r * 128 + a] * y[r * 128 + b];
          if (o[a * 128 + b] != (float)ref && bad++ < 5)
            printf("  mode 0 R[%d][%d] = %g want %g\n", a, b, o[a * 128 + b], ref);
        }
    } else {
      for (int m = 0; m < 64; ++m)
        for (int n = 0; n < 128; ++n) {
          double ref = 0;
          for (int k = 0; k < 128; ++k)
            ref += (double)x[m * 128 + k] * (mode == 1 ? s[k * 128 + n] : s[n * 128 + k]);
          const int lane = (m % 16) + 32 * (m / 16);
          if (o[lane * 128 + n] != (float)ref && bad++ < 5)
            printf("  mode %d O[%d][%d] = %g want %g\n", mode, m, n, o[lane * 128 + n], ref);
        }
    }
    printf("mode %d: %d mismatches\n", mode, bad);
    bad_total += bad;
  }
  printf(bad_total ? "FAIL\n" : "PASS\n");
  return bad_total ? 1 : 0;
}
