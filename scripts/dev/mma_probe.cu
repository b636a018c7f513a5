// Standalone tcgen05 kind::tf32 probe: checks descriptor conventions used by kernels_tc.cuh.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../../paper_2602_06935_b200/csrc/kernels_tc.cuh"
using namespace cotten;
using namespace cotten::tc;

// mode 0: D[128x32] = A[128x32 rows, K-major SW128] * B[32 rows (n) x 32 (k), K-major SW128]
// mode 1: D[64x64]  = A MN-major (atoms at 0 and LBO) * B MN-major, K = 8*ks rows
__global__ void probe(const float* A, const float* Bm, float* out, int mode, int ks) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // fill: A tile at 0 (128 rows x 32, swizzled), A2 at 16K; B at 32K, B2 at 48K
  for (int i = t; i < 4 * 128 * 32; i += blockDim.x) {
    int tile = i / 4096, r = (i % 4096) / 32, c = i % 32;
    float val = (tile < 2 ? A : Bm)[(tile & 1) * 4096 + r * 32 + c];
    *reinterpret_cast<float*>(smem + tile * 16384 + elem_off(r, c)) = val;
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
  const uint32_t base = smem_u32(smem);
  if (t == 0) {
    if (mode == 0) {
      const uint32_t id = idesc_tf32(128, 32, false, false);
      for (int kk = 0; kk < 4; ++kk)
        mma_tf32(tmem, sdesc(base + 32 * kk, 16, 1024), sdesc(base + 32768 + 32 * kk, 16, 1024), id, kk > 0);
    } else {
      issue_reduction(tmem, base, base + 32768, 16384, ks, true);
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

int main() {
  const int n = 2 * 4096;
  float *hA = (float*)malloc(n * 4), *hB = (float*)malloc(n * 4), *hO = (float*)malloc(128 * 64 * 4);
  srand(1);
  for (int i = 0; i < n; ++i) { hA[i] = (rand() % 17 - 8) / 8.0f; hB[i] = (rand() % 13 - 6) / 4.0f; }
  float *dA, *dB, *dO;
  cudaMalloc(&dA, n * 4); cudaMalloc(&dB, n * 4); cudaMalloc(&dO, 128 * 64 * 4);
  cudaMemcpy(dA, hA, n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, n * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dO, 0, 128 * 64 * 4);
    const int ks = 16;
    probe<<<1, 128, 65536>>>(dA, dB, dO, mode, ks);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    cudaMemcpy(hO, dO, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    if (mode == 0) {  // D[m][nn] = sum_k A[m][k] * B[nn][k]
      for (int m = 0; m < 128; ++m) for (int nn = 0; nn < 32; ++nn) {
        double s = 0; for (int k = 0; k < 32; ++k) s += (double)hA[m * 32 + k] * hB[nn * 32 + k];
        maxerr = fmax(maxerr, fabs(s - hO[m * 64 + nn])); maxref = fmax(maxref, fabs(s));
      }
      printf("  K-major 128x32x32: maxerr %g maxref %g  D[0][0..3] %g %g %g %g\n", maxerr, maxref, hO[0], hO[1], hO[2], hO[3]);
    } else {  // x = [A0 | A1] (MN atoms), y = [B0 | B1]; D[m][c] = sum_r x[r][m] y[r][c], lanes: m -> (m%16)+32(m/16)
      for (int m = 0; m < 64; ++m) for (int c = 0; c < 64; ++c) {
        double s = 0;
        for (int r = 0; r < 8 * ks; ++r) s += (double)hA[(m / 32) * 4096 + r * 32 + m % 32] * hB[(c / 32) * 4096 + r * 32 + c % 32];
        int lanei = (m % 16) + 32 * (m / 16);
        maxerr = fmax(maxerr, fabs(s - hO[lanei * 64 + c])); maxref = fmax(maxref, fabs(s));
      }
      printf("  MN-major 64x64x%d: maxerr %g maxref %g  lane0 %g %g lane16 %g\n", 8 * ks, maxerr, maxref, hO[0], hO[1], hO[16 * 64]);
      // alternative layout guess: lane = m
      double e2 = 0;
      for (int m = 0; m < 64; ++m) for (int c = 0; c < 64; ++c) {
        double s = 0;
        for (int r = 0; r < 8 * ks; ++r) s += (double)hA[(m / 32) * 4096 + r * 32 + m % 32] * hB[(c / 32) * 4096 + r * 32 + c % 32];
        e2 = fmax(e2, fabs(s - hO[m * 64 + c]));
      }
      printf("  (if lane=m: maxerr %g)\n", e2);
      // search: for each expected row m, best-matching lane / column permutation
      for (int m = 0; m < 64; m += 5) {
        double ref[64];
        for (int c = 0; c < 64; ++c) { double s = 0; for (int r = 0; r < 8 * ks; ++r) s += (double)hA[(m / 32) * 4096 + r * 32 + m % 32] * hB[(c / 32) * 4096 + r * 32 + c % 32]; ref[c] = s; }
        int best = -1; double be = 1e30;
        for (int l = 0; l < 128; ++l) { double e = 0; for (int c = 0; c < 64; ++c) e = fmax(e, fabs(ref[c] - hO[l * 64 + c])); if (e < be) { be = e; best = l; } }
        int fl = -1, fc = -1;
        for (int l = 0; l < 128 && fl < 0; ++l) for (int c = 0; c < 64; ++c) if (fabs(hO[l * 64 + c] - ref[0]) < 1e-9 && ref[0] != 0) { fl = l; fc = c; break; }
        printf("  row m=%d best lane %d err %g ; ref[0]=%g found at lane %d col %d\n", m, best, be, ref[0], fl, fc);
      }
      for (int l = 0; l < 128; l += 8) printf("  lane %3d: %8.3f %8.3f %8.3f %8.3f\n", l, hO[l*64], hO[l*64+1], hO[l*64+32], hO[l*64+33]);
    }
  }
  return 0;
}
