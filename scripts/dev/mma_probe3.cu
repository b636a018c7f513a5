// tcgen05 kind::tf32 probe 3: MN-major operands in SWIZZLE_128B_BASE32B (layout type 1),
// descriptor variants; A-from-TMEM (ts) mode.
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
// 32B-granule swizzle within 128 B rows: granule g of row r at (g ^ (r & 3))
__device__ __forceinline__ uint32_t off32(int r, int c) {
  return (uint32_t)r * 128u + ((uint32_t)(((c >> 3) ^ (r & 3))) << 5) + (uint32_t)(c & 7) * 4u;
}

__global__ void probe(const float* src, float* out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 6 * 4096; i += blockDim.x) {
    int tile = i / 4096, r = (i % 4096) / 32, c = i % 32;
    uint32_t o = (mode >= 10) ? elem_off(r, c) : off32(r, c);
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
  if (mode == 10) {  // ts: each thread writes row t of tile0 (32 values) into TMEM lane t, cols 128..159
    float v[32];
    for (int c = 0; c < 32; ++c) v[c] = src[t * 32 + c];
    uint32_t* u = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + 128 + ((32 * warp) << 16)),
        "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]), "r"(u[8]),
        "r"(u[9]), "r"(u[10]), "r"(u[11]), "r"(u[12]), "r"(u[13]), "r"(u[14]), "r"(u[15]), "r"(u[16]),
        "r"(u[17]), "r"(u[18]), "r"(u[19]), "r"(u[20]), "r"(u[21]), "r"(u[22]), "r"(u[23]), "r"(u[24]),
        "r"(u[25]), "r"(u[26]), "r"(u[27]), "r"(u[28]), "r"(u[29]), "r"(u[30]), "r"(u[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const uint32_t b = smem_u32(smem);
  const uint32_t T = 16384;
  if (t == 0) {
    if (mode < 10) {
      // MN-major A (tiles 0,1 as the two M atoms), MN-major B (tiles 4,5), M=64 N=64, K = 32 rows (4 x 8)
      uint32_t lbo = T, sbo = 512, kstep = 1024;
      if (mode == 1) { lbo = 512; sbo = T; }
      if (mode == 2) { lbo = T; sbo = 1024; }
      if (mode == 3) { lbo = 1024; sbo = T; }
      const uint32_t id = idesc_tf32(64, 64, true, true);
      for (int kk = 0; kk < 4; ++kk)
        mma_tf32(tmem, sdesc_t(b + kstep * kk, lbo, sbo, 1), sdesc_t(b + 4 * T + kstep * kk, lbo, sbo, 1), id, kk > 0);
    } else {  // ts: A from TMEM cols 128.., B K-major tile4 (32 rows), M=128 N=32
      const uint32_t id = idesc_tf32(128, 32, false, false);
      for (int kk = 0; kk < 4; ++kk)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                     "r"(tmem + 128 + 8 * kk), "l"(sdesc(b + 4 * T + 32 * kk, 16, 1024)), "r"(id), "r"((uint32_t)(kk > 0)));
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
  int modes[] = {0, 1, 2, 3, 10};
  for (int mode : modes) {
    cudaMemset(dO, 0, 128 * 64 * 4);
    probe<<<1, 128, 6 * 16384>>>(dS, dO, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hO, dO, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    const bool ts = mode >= 10;
    int M = ts ? 128 : 64, N = ts ? 32 : 64;
    static double D[128][64];
    for (int m = 0; m < M; ++m) for (int nn = 0; nn < N; ++nn) {
      double s = 0;
      for (int k = 0; k < 32; ++k) {
        double a = ts ? tile(0, m, k) : tile(m / 32, k, m % 32);
        double bb = ts ? tile(4, nn, k) : tile(4 + nn / 32, k, nn % 32);
        s += a * bb;
      }
      D[m][nn] = s;
    }
    double maxerr = 0;
    for (int m = 0; m < M; ++m) {
      int lane = ts ? m : (m % 16) + 32 * (m / 16);
      for (int c = 0; c < N; ++c) maxerr = fmax(maxerr, fabs(D[m][c] - hO[lane * 64 + c]));
    }
    printf("mode %2d (%s): maxerr %g   D[0][0]=%g got %g\n", mode, cudaGetErrorString(e), maxerr, D[0][0], hO[0]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
