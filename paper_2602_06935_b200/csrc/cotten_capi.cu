// C-ABI of the cosine-attention operator (include/cotten.h): validation,
// kernel dispatch, per-stream workspaces and the host-buffer entry points.
// Error conventions mirror the reference C API (capi.cpp:21-44).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <type_traits>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cotten.h"
#include "common.cuh"
#include "kernels_d32.cuh"
#include "kernels_generic.cuh"
#include "kernels_rt.cuh"
#include "kernels_tc.cuh"
#include "kernels_tcb.cuh"
#include "kernels_tcf.cuh"
#include "kernels_tch.cuh"
#include "kernels_tcg.cuh"

namespace cotten {
namespace {

thread_local std::string g_last_error;
thread_local int g_launches = 0;
// Launch-duration profile (cotten_profile_begin/end): each device call of this
// thread takes the next [start, end] slot of the caller's buffer.
struct Profile {
  unsigned long long* buf = nullptr;
  int slots = 0, next = 0;
  unsigned long long* take() { return (buf && next < slots) ? buf + 2 * next++ : nullptr; }
};
thread_local Profile g_prof;

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void usage(const std::string& what) { throw Error{COTTEN_ERR_USAGE, what}; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define COTTEN_CUDA(call)                                                                  \
  do {                                                                                     \
    cudaError_t err_ = (call);                                                             \
    if (err_ != cudaSuccess)                                                               \
      throw Error{COTTEN_ERR_INTERNAL, std::string(#call) + ": " + cudaGetErrorString(err_)}; \
  } while (0)

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return COTTEN_OK;
  } catch (const Error& e) {
    return fail(e.code, e.msg);
  } catch (const std::exception& e) {
    return fail(COTTEN_ERR_INTERNAL, e.what());
  } catch (...) {
    return fail(COTTEN_ERR_INTERNAL, "unknown error");
  }
}


size_t elem_size(int dtype) {
  switch (dtype) {
    case COTTEN_F32: return 4;
    case COTTEN_BF16: return 2;
    case COTTEN_F64: return 8;
  }
  usage("cotten: unknown dtype");
}
size_t acc_size(int dtype) { return dtype == COTTEN_F64 ? 8 : 4; }

// Resolved, validated view of a cotten_desc (check_qkv, attention.cpp:37-46).
struct Layout {
  int64_t B, H, N, D, sb, sh, sn, msb;
  int dtype, flags;
  double eps;
  int64_t units() const { return B * H; }
  // Elements spanned by one tensor, for staging copies of the host API.
  int64_t span() const { return (B - 1) * sb + (H - 1) * sh + (N - 1) * sn + D; }
  // The host entry points copy whole spans, so they need a gap-free layout.
  void require_dense(const char* what) const {
    if (span() != B * H * N * D)
      usage(std::string(what) + ": host entry points need a dense (gap-free) layout");
  }
};

Layout resolve(const cotten_desc* d, const char* what) {
  if (d == nullptr) usage(std::string(what) + ": null descriptor");
  Layout L{};
  L.B = d->batch;
  L.H = d->heads;
  L.N = d->seq_len;
  L.D = d->head_dim;
  L.dtype = d->dtype;
  L.flags = d->flags;
  L.eps = d->eps;
  if (L.B < 1 || L.H < 1 || L.N < 1 || L.D < 1)
    usage(std::string(what) + ": empty matrix (batch, heads, seq_len, head_dim must be >= 1)");
  elem_size(L.dtype);
  if (!(L.eps >= 0.0) || !std::isfinite(L.eps)) usage(std::string(what) + ": eps must be >= 0");
  if (d->stride_b == 0 && d->stride_h == 0 && d->stride_n == 0) {
    L.sn = L.D;
    L.sh = L.N * L.D;
    L.sb = L.H * L.N * L.D;
  } else {
    L.sb = d->stride_b;
    L.sh = d->stride_h;
    L.sn = d->stride_n;
    if (L.sn < L.D || L.sh < 1 || L.sb < 1)
      usage(std::string(what) + ": strides must be positive and stride_n >= head_dim");
  }
  L.msb = d->mask_stride_b == 0 ? L.N : d->mask_stride_b;
  if (L.msb < L.N) usage(std::string(what) + ": mask length (mask_stride_b < seq_len)");
  return L;
}

constexpr size_t kSmemBudget = 227 * 1024;

void check_generic_fits(const Layout& L) {
  const size_t need = L.dtype == COTTEN_F64 ? gen_fwd_smem<double>(L.D) : gen_fwd_smem<float>(L.D);
  if (need > kSmemBudget)
    usage("cotten: head_dim " + std::to_string(L.D) + " exceeds the shared-memory budget");
}

OpParams make_params(const Layout& L) {
  OpParams p{};
  p.B = L.B;
  p.H = L.H;
  p.N = L.N;
  p.D = L.D;
  p.sb = L.sb;
  p.sh = L.sh;
  p.sn = L.sn;
  p.msb = L.msb;
  p.eps = L.eps;
  return p;
}

// ---- per-device state ---------------------------------------------------

std::mutex g_dev_mu;
std::vector<int*> g_status;  // one sticky status word per device

int* device_status_word() {
  int dev = 0;
  COTTEN_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if ((int)g_status.size() <= dev) g_status.resize(dev + 1, nullptr);
  if (g_status[dev] == nullptr) {
    COTTEN_CUDA(cudaMalloc(&g_status[dev], sizeof(int)));
    COTTEN_CUDA(cudaMemset(g_status[dev], 0, sizeof(int)));
  }
  return g_status[dev];
}

// Grow-only device scratch (per-unit dm, a recomputed S, the generic
// backward's G workspace, the tcgen05 backward's CTA-completion counter).
// One set per (device, stream): launches on one stream are ordered, so they
// may share it, and launches on different streams never do (two concurrent
// cotten_bwd(..., dm_total) calls on two streams each get their own counter).
// Allocation happens only when a call needs more than any earlier call on
// that stream; during CUDA-graph capture it is refused (warm the stream up
// with one eager call first, as graph capture requires anyway).
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
};
struct StreamScratch {
  Scratch slot[4];
};
enum ScratchSlot { kScrDm, kScrS, kScrG, kScrCounter };
struct ScratchKey {
  int dev;
  cudaStream_t st;
  std::thread::id tid;  // only for the per-thread default stream
  bool operator<(const ScratchKey& o) const {
    if (dev != o.dev) return dev < o.dev;
    if (st != o.st) return st < o.st;
    return tid < o.tid;
  }
};
std::mutex g_scratch_mu;
std::map<ScratchKey, StreamScratch> g_scratch;  // entries live for the process

void* scratch_get(cudaStream_t st, ScratchSlot which, size_t need, bool zeroed = false) {
  int dev = 0;
  COTTEN_CUDA(cudaGetDevice(&dev));
  const ScratchKey key{dev, st,
                       st == cudaStreamPerThread ? std::this_thread::get_id() : std::thread::id()};
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  Scratch& s = g_scratch[key].slot[which];
  if (need > s.bytes) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
      throw Error{COTTEN_ERR_INTERNAL,
                  "cotten: workspace growth during graph capture (run one eager call on this "
                  "stream with the same shape before capturing)"};
    if (s.ptr) COTTEN_CUDA(cudaStreamSynchronize(st));  // earlier launches may still use it
    if (s.ptr) cudaFree(s.ptr);
    s.ptr = nullptr;
    s.bytes = 0;
    COTTEN_CUDA(cudaMalloc(&s.ptr, need));
    if (zeroed) COTTEN_CUDA(cudaMemset(s.ptr, 0, need));  // kernels keep it zero between launches
    s.bytes = need;
  }
  return s.ptr;
}

// ---- launches -------------------------------------------------------------

template <typename T>
void launch_fwd_t(const Layout& L, OpParams p, cudaStream_t st) {
  using A = typename AccOf<T>::type;
  const bool tensor = !(L.flags & (COTTEN_FLAG_FORCE_GENERIC | COTTEN_FLAG_FP32_PIPE));
  if (tensor && tcg_fwd_supported<T>(p)) {
    const int n = launch_tcg_fwd(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: fp32 d_h=128 tensor-core forward launch failed"};
    g_launches += n;
  } else if (tensor && tcf_fwd_supported<T>(p)) {
    const int n = launch_tcf_fwd(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: fp32 d_h=64 tensor-core forward launch failed"};
    g_launches += n;
  } else if (tensor && tch_fwd_supported<T>(p)) {
    const int n = launch_tch_fwd(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: bf16 d_h=128 tensor-core forward launch failed"};
    g_launches += n;
  } else if (tensor && tcb_fwd_supported<T>(p)) {
    const int n = launch_tcb_fwd(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: bf16 tensor-core forward launch failed"};
    g_launches += n;
  } else if (tensor && tc_fwd_supported<T>(p)) {
    const int n = launch_tc_fwd(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: tensor-core forward launch failed"};
    g_launches += n;
  } else if (!(L.flags & COTTEN_FLAG_FORCE_GENERIC) && fast_fwd_supported<T>(p)) {
    const int n = launch_fast_fwd<T>(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: fast forward launch failed (tensor map)"};
    g_launches += n;
  } else if (!(L.flags & COTTEN_FLAG_FORCE_GENERIC) && rt_supported<T>(p, false)) {
    if constexpr (!std::is_same<T, double>::value) launch_rt_fwd<T>(p, st);
    g_launches += 1;
  } else {
    check_generic_fits(L);
    const size_t smem = gen_fwd_smem<A>(L.D);
    COTTEN_CUDA(cudaFuncSetAttribute(cos_fwd_generic<T, A>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cos_fwd_generic<T, A><<<(unsigned)L.units(), kGenThreads, smem, st>>>(p);
    g_launches += 1;
  }
  COTTEN_CUDA(cudaGetLastError());
}

template <typename T>
void launch_bwd_t(const Layout& L, OpParams p, cudaStream_t st) {
  using A = typename AccOf<T>::type;
  const bool tensor = !(L.flags & (COTTEN_FLAG_FORCE_GENERIC | COTTEN_FLAG_FP32_PIPE));
  if (tensor && tcg_bwd_supported<T>(p)) {
    const int n = launch_tcg_bwd(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: fp32 d_h=128 tensor-core backward launch failed"};
    g_launches += n;
  } else if (tensor && tcf_bwd_supported<T>(p)) {
    const int n = launch_tcf_bwd(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: fp32 d_h=64 tensor-core backward launch failed"};
    g_launches += n;
  } else if (tensor && tch_bwd_supported<T>(p)) {
    const int n = launch_tch_bwd(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: bf16 d_h=128 tensor-core backward launch failed"};
    g_launches += n;
  } else if (tensor && tcb_bwd_supported<T>(p)) {
    const int n = launch_tcb_bwd(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: bf16 tensor-core backward launch failed"};
    g_launches += n;
  } else if (tensor && tc_bwd_supported<T>(p)) {
    const int n = launch_tc_bwd(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: tensor-core backward launch failed"};
    g_launches += n;
  } else if (!(L.flags & COTTEN_FLAG_FORCE_GENERIC) && fast_bwd_supported<T>(p)) {
    const int n = launch_fast_bwd<T>(p, st);
    COTTEN_CUDA(cudaGetLastError());
    if (n < 0) throw Error{COTTEN_ERR_INTERNAL, "cotten: fast backward launch failed (tensor map)"};
    g_launches += n;
  } else if (!(L.flags & COTTEN_FLAG_FORCE_GENERIC) && rt_supported<T>(p, true)) {
    if constexpr (!std::is_same<T, double>::value) launch_rt_bwd<T>(p, st);
    g_launches += 1;
  } else {
    const bool gg = gen_bwd_smem<A>(L.D) > kSmemBudget;
    if (gen_bwd_smem<A>(L.D, gg) > kSmemBudget)
      usage("cotten: head_dim " + std::to_string(L.D) + " exceeds the shared-memory budget");
    const size_t smem = gen_bwd_smem<A>(L.D, gg);
    auto kern = gg ? cos_bwd_generic<T, A, true> : cos_bwd_generic<T, A, false>;
    if (gg) p.workspace = scratch_get(st, kScrG, L.units() * L.D * L.D * sizeof(A));
    COTTEN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)L.units(), kGenThreads, smem, st>>>(p);
    g_launches += 1;
  }
  COTTEN_CUDA(cudaGetLastError());
}

void launch_fwd(const Layout& L, const OpParams& p, cudaStream_t st) {
  switch (L.dtype) {
    case COTTEN_F32: return launch_fwd_t<float>(L, p, st);
    case COTTEN_BF16: return launch_fwd_t<__nv_bfloat16>(L, p, st);
    case COTTEN_F64: return launch_fwd_t<double>(L, p, st);
  }
}
void launch_bwd(const Layout& L, const OpParams& p, cudaStream_t st) {
  switch (L.dtype) {
    case COTTEN_F32: return launch_bwd_t<float>(L, p, st);
    case COTTEN_BF16: return launch_bwd_t<__nv_bfloat16>(L, p, st);
    case COTTEN_F64: return launch_bwd_t<double>(L, p, st);
  }
}

void device_fwd(const Layout& L, const void* q, const void* k, const void* v,
                const uint8_t* valid, double m, void* out, void* saved_S, void* saved_norms,
                cudaStream_t st, const double* m_dev = nullptr) {
  if (!q || !k || !v) usage("cosine_attention_fused: null input");
  if (!out && !saved_S && !saved_norms) usage("cosine_attention_fused: no output requested");
  if (!m_dev && !std::isfinite(m)) usage("cosine_attention_fused: m must be finite");
  OpParams p = make_params(L);
  p.q = q;
  p.k = k;
  p.v = v;
  p.valid = valid;
  p.m = m;
  p.m_dev = m_dev;
  p.out = out;
  p.saved_S = saved_S;
  p.saved_norms = saved_norms;
  p.status = device_status_word();
  p.tstamp = g_prof.take();
  launch_fwd(L, p, st);
}

void device_bwd(const Layout& L, const void* q, const void* k, const void* v,
                const uint8_t* valid, double m, const void* d_out, const void* saved_S, void* dq,
                void* dk, void* dv, double* dm_unit, double* dm_total, cudaStream_t st,
                const double* m_dev = nullptr) {
  if (!q || !k || !v || !d_out) usage("cosine_attention_backward: null input");
  if (!dq || !dk || !dv) usage("cosine_attention_backward: null gradient output");
  if (!m_dev && !std::isfinite(m)) usage("cosine_attention_backward: m must be finite");
  OpParams p = make_params(L);
  p.q = q;
  p.k = k;
  p.v = v;
  p.valid = valid;
  p.m = m;
  p.m_dev = m_dev;
  p.status = device_status_word();
  p.tstamp = g_prof.take();  // every kernel of this call stamps the same slot
  if (saved_S == nullptr) {  // recompute the state with an S-only forward
    void* s = scratch_get(st, kScrS, L.units() * L.D * L.D * acc_size(L.dtype));
    OpParams f = p;
    f.saved_S = s;
    launch_fwd(L, f, st);
    saved_S = s;
  }
  p.saved_S = const_cast<void*>(saved_S);
  p.dout = d_out;
  p.dq = dq;
  p.dk = dk;
  p.dv = dv;
  p.dm_unit = dm_unit;
  if (dm_total && !dm_unit)
    p.dm_unit = static_cast<double*>(scratch_get(st, kScrDm, L.units() * sizeof(double)));
  const bool tensor = !(L.flags & (COTTEN_FLAG_FORCE_GENERIC | COTTEN_FLAG_FP32_PIPE));
  const bool tc_path = tensor && ((L.dtype == COTTEN_F32 && (tc_bwd_supported<float>(p) ||
                                                              tcf_bwd_supported<float>(p) ||
                                                              tcg_bwd_supported<float>(p))) ||
                                  (L.dtype == COTTEN_BF16 && (tcb_bwd_supported<__nv_bfloat16>(p) ||
                                                               tch_bwd_supported<__nv_bfloat16>(p))));
  if (dm_total && tc_path) {  // the tcgen05 kernel's last CTA writes the total (no extra launch)
    p.dm_total = dm_total;
    p.grid_done = static_cast<unsigned*>(scratch_get(st, kScrCounter, sizeof(unsigned), true));
  }
  launch_bwd(L, p, st);
  if (dm_total && !tc_path) {
    dm_reduce_kernel<<<1, 256, 0, st>>>(p.dm_unit, L.units(), dm_total);
    g_launches += 1;
    COTTEN_CUDA(cudaGetLastError());
  }
}

}  // namespace

// Shared with the encoder translation unit (encoder.cu): one thread-local
// last-error string and one status word per device for the whole library.
void set_last_error(const std::string& msg) { g_last_error = msg; }
int* status_word_for_current_device() { return device_status_word(); }

namespace {

// ---- host entry points ----------------------------------------------------

// Mask check on the host, exactly check_qkv's (attention.cpp:42-45).
void host_check_mask(const Layout& L, const uint8_t* valid, const char* what) {
  if (valid == nullptr) return;
  for (int64_t b = 0; b < L.B; ++b) {
    const uint8_t* row = valid + b * L.msb;
    int64_t c = 0;
    for (int64_t i = 0; i < L.N; ++i) c += row[i] != 0;
    if (c == 0) usage(std::string(what) + ": no real rows (sequence " + std::to_string(b) + ")");
  }
}

// Per-thread staging state for the host entry points.
// Staging streams of the host entry points: the batch is cut into slices of
// whole sequences and slice i's uploads, kernels and downloads are queued on
// pipe[i % kPipe], so uploads of one slice, kernels of the next and downloads
// of the previous overlap (the two PCIe directions run on separate copy
// engines; end to end the host calls are PCIe-bound).
constexpr int kPipe = 3;
constexpr size_t kSliceBytes = size_t(2) << 20;  // min bytes per tensor per slice
constexpr int kMaxSlices = 8;
// COTTEN_HOST_SLICE_KB / COTTEN_HOST_MAX_SLICES override the two (tuning)
size_t slice_bytes() {
  static const size_t v = [] {
    const char* e = std::getenv("COTTEN_HOST_SLICE_KB");
    return e ? std::max<size_t>(64, std::strtoull(e, nullptr, 10)) << 10 : kSliceBytes;
  }();
  return v;
}
int max_slices() {
  static const int v = [] {
    const char* e = std::getenv("COTTEN_HOST_MAX_SLICES");
    return e ? std::max(1, std::atoi(e)) : kMaxSlices;
  }();
  return v;
}

// One staging context per (host thread, device): a thread that alternates
// between GPUs keeps each device's buffers and streams (nothing is dropped
// or leaked on a switch).
struct HostCtx {
  cudaStream_t stream = nullptr;
  cudaStream_t pipe[kPipe] = {};
  int dev = -1;
  void* bufs[12] = {};
  size_t sizes[12] = {};
  ~HostCtx() {
    // Process teardown may have destroyed the context already; ignore errors.
    if (dev < 0 || cudaSetDevice(dev) != cudaSuccess) return;
    for (void* b : bufs)
      if (b) cudaFree(b);
    if (stream) cudaStreamDestroy(stream);
    for (cudaStream_t p : pipe)
      if (p) cudaStreamDestroy(p);
  }
  void ensure(int cur) {
    dev = cur;
    if (stream == nullptr) COTTEN_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    for (cudaStream_t& p : pipe)
      if (p == nullptr) COTTEN_CUDA(cudaStreamCreateWithFlags(&p, cudaStreamNonBlocking));
  }
  void* buf(int slot, size_t need) {
    if (need > sizes[slot]) {
      if (bufs[slot]) cudaFree(bufs[slot]);
      bufs[slot] = nullptr;
      sizes[slot] = 0;
      COTTEN_CUDA(cudaMalloc(&bufs[slot], need));
      sizes[slot] = need;
    }
    return bufs[slot];
  }
};
// Staging contexts outlive the threads that used them: a thread's contexts go back
// to a process-wide pool when it exits and the next new thread takes one from
// there.  The reference calls the op from short-lived parallel_chunks workers
// (encoder.cpp:295,345); with a context per thread every such call paid 4 x
// cudaStreamCreate, the staging cudaMallocs and, at thread exit, a device-
// synchronising cudaFree (measured from the bench's e2e with threads created per
// window: single windows fell from 70 k to 6-20 k seq/s, profiles/r02an_e2e_threads).
// The pool is never destroyed (process teardown may already have torn the CUDA
// context down).
struct HostPool {
  std::mutex mu;
  std::map<int, std::vector<HostCtx*>> free;
};
HostPool* g_hpool = new HostPool;
struct ThreadHosts {
  std::map<int, HostCtx*> ctx;
  ~ThreadHosts() {
    std::lock_guard<std::mutex> lk(g_hpool->mu);
    for (auto& kv : ctx) g_hpool->free[kv.first].push_back(kv.second);
  }
};
thread_local ThreadHosts g_hosts;
thread_local HostCtx* g_host = nullptr;
// At most COTTEN_HOST_MAX_CONCURRENT (default 8) host-entry calls stage and run
// at once per process; further callers queue.  The host path is PCIe-bound; with
// persistent callers 4-8 concurrent calls keep both copy directions busy (ML-1M
// e2e: 8 threads 83 k seq/s with the limit at 8, 79 k at 4; 16 threads 71 k with
// the limit at 8 — profiles/r02an_e2e_threads), while the reference calls the op
// from cfg.threads parallel_chunks workers.
class HostGate {
 public:
  void acquire() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return busy_ < limit(); });
    ++busy_;
  }
  void release() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      --busy_;
    }
    cv_.notify_one();
  }

 private:
  static int limit() {
    static const int v = [] {
      const char* e = std::getenv("COTTEN_HOST_MAX_CONCURRENT");
      return e ? std::max(1, std::atoi(e)) : 8;
    }();
    return v;
  }
  std::mutex mu_;
  std::condition_variable cv_;
  int busy_ = 0;
};
HostGate g_gate;
struct HostSlot {
  HostSlot() { g_gate.acquire(); }
  ~HostSlot() { g_gate.release(); }
  HostSlot(const HostSlot&) = delete;
  HostSlot& operator=(const HostSlot&) = delete;
};
// Select (creating on first use) the calling thread's context on the current device.
void host_begin() {
  int cur = 0;
  COTTEN_CUDA(cudaGetDevice(&cur));
  HostCtx*& h = g_hosts.ctx[cur];
  if (h == nullptr) {
    {
      std::lock_guard<std::mutex> lk(g_hpool->mu);
      std::vector<HostCtx*>& f = g_hpool->free[cur];
      if (!f.empty()) {
        h = f.back();
        f.pop_back();
      }
    }
    if (h == nullptr) h = new HostCtx;
  }
  g_host = h;
  g_host->ensure(cur);
}

enum Slot { kQ, kK, kV, kO, kDO, kDQ, kDK, kDV, kMask, kS, kNorms, kDm };

void* h2d(int slot, const void* src, size_t bytes) {
  void* dst = g_host->buf(slot, bytes);
  COTTEN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, g_host->stream));
  return dst;
}
void d2h(void* dst, const void* src, size_t bytes) {
  if (dst) COTTEN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g_host->stream));
}

// Slices of whole sequences for the pipelined host path.  A slice of
// sequences is one contiguous byte range only when the batch is the outermost
// dimension (sb * B == span); any other dense layout ([N][B][H][D],
// [H][B][N][D], ...) is staged as one slice covering the whole span.  f64 and
// the generic kernels' shapes stay on one slice too (their launches are
// short and per-slice scratch would only multiply workspace).
struct Slices {
  int64_t per = 0;  // sequences per slice
  int n = 1;
  bool batch_major = true;
  size_t bytes(const Layout& L, int64_t nb, size_t es) const {
    return batch_major ? (size_t)(nb * L.sb) * es : (size_t)L.span() * es;
  }
};
Slices plan_slices(const Layout& L, size_t tensor_bytes) {
  Slices sl;
  sl.batch_major = L.sb * L.B == L.span();
  int n = (int)std::min<size_t>(max_slices(), std::max<size_t>(1, tensor_bytes / slice_bytes()));
  const bool fast_shape = L.D == 32 || L.D == 64 || L.D == 128;
  if (L.dtype == COTTEN_F64 || !fast_shape || (L.flags & COTTEN_FLAG_FORCE_GENERIC) ||
      !sl.batch_major)
    n = 1;
  n = (int)std::min<int64_t>(n, L.B);
  sl.per = (L.B + n - 1) / n;
  sl.n = (int)((L.B + sl.per - 1) / sl.per);
  return sl;
}
void pipe_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (src && bytes) COTTEN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
}
void pipe_d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (dst && bytes) COTTEN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
}
void pipe_sync() {
  for (cudaStream_t p : g_host->pipe) COTTEN_CUDA(cudaStreamSynchronize(p));
}
template <typename P>
P* at(P* base, int64_t bytes) {
  return base ? reinterpret_cast<P*>(reinterpret_cast<uint8_t*>(const_cast<void*>(
                    static_cast<const void*>(base))) + bytes)
              : nullptr;
}

}  // namespace
}  // namespace cotten

using namespace cotten;

extern "C" {

const char* cotten_version(void) { return "cotten-b200 0.1 (sm_100a)"; }
const char* cotten_last_error(void) { return g_last_error.c_str(); }
int cotten_last_launch_count(void) { return g_launches; }

int cotten_fwd(const cotten_desc* desc, const void* q, const void* k, const void* v,
               const uint8_t* valid, double m, void* out, void* saved_S, void* saved_norms,
               void* stream) {
  g_launches = 0;
  return guarded([&] {
    Layout L = resolve(desc, "cosine_attention_fused");
    device_fwd(L, q, k, v, valid, m, out, saved_S, saved_norms, (cudaStream_t)stream);
  });
}

int cotten_bwd(const cotten_desc* desc, const void* q, const void* k, const void* v,
               const uint8_t* valid, double m, const void* d_out, const void* saved_S, void* dq,
               void* dk, void* dv, double* dm_unit, double* dm_total, void* stream) {
  g_launches = 0;
  return guarded([&] {
    Layout L = resolve(desc, "cosine_attention_backward");
    device_bwd(L, q, k, v, valid, m, d_out, saved_S, dq, dk, dv, dm_unit, dm_total,
               (cudaStream_t)stream);
  });
}

int cotten_fwd_mdev(const cotten_desc* desc, const void* q, const void* k, const void* v,
                    const uint8_t* valid, const double* m_dev, void* out, void* saved_S,
                    void* saved_norms, void* stream) {
  g_launches = 0;
  return guarded([&] {
    Layout L = resolve(desc, "cosine_attention_fused");
    if (m_dev == nullptr) usage("cosine_attention_fused: null m_dev");
    device_fwd(L, q, k, v, valid, 0.0, out, saved_S, saved_norms, (cudaStream_t)stream, m_dev);
  });
}

int cotten_bwd_mdev(const cotten_desc* desc, const void* q, const void* k, const void* v,
                    const uint8_t* valid, const double* m_dev, const void* d_out,
                    const void* saved_S, void* dq, void* dk, void* dv, double* dm_unit,
                    double* dm_total, void* stream) {
  g_launches = 0;
  return guarded([&] {
    Layout L = resolve(desc, "cosine_attention_backward");
    if (m_dev == nullptr) usage("cosine_attention_backward: null m_dev");
    device_bwd(L, q, k, v, valid, 0.0, d_out, saved_S, dq, dk, dv, dm_unit, dm_total,
               (cudaStream_t)stream, m_dev);
  });
}

int cotten_profile_begin(void* stamps, int slots) {
  return guarded([&] {
    if (stamps == nullptr || slots < 1) usage("cotten_profile_begin: null buffer or no slots");
    g_prof.buf = static_cast<unsigned long long*>(stamps);
    g_prof.slots = slots;
    g_prof.next = 0;
  });
}

int cotten_profile_end(void) {
  const int used = g_prof.next;
  g_prof = Profile{};
  return used;
}

int cotten_device_status(int device, int32_t* bits, int reset) {
  return guarded([&] {
    if (!bits) usage("cotten_device_status: null output");
    int prev = 0;
    COTTEN_CUDA(cudaGetDevice(&prev));
    COTTEN_CUDA(cudaSetDevice(device));
    int* w = device_status_word();
    COTTEN_CUDA(cudaDeviceSynchronize());
    int h = 0;
    COTTEN_CUDA(cudaMemcpy(&h, w, sizeof(int), cudaMemcpyDeviceToHost));
    if (reset) COTTEN_CUDA(cudaMemset(w, 0, sizeof(int)));
    *bits = h;
    COTTEN_CUDA(cudaSetDevice(prev));
  });
}

int cotten_fwd_host(const cotten_desc* desc, const void* q, const void* k, const void* v,
                    const uint8_t* valid, double m, void* out, void* saved_S,
                    void* saved_norms) {
  g_launches = 0;
  return guarded([&] {
    Layout L = resolve(desc, "cosine_attention_fused");
    if (!q || !k || !v) usage("cosine_attention_fused: null input");
    host_check_mask(L, valid, "cosine_attention_fused");
    L.require_dense("cosine_attention_fused");
    const HostSlot slot_;  // concurrency gate, held to the end of the call
    host_begin();
    const size_t tb = L.span() * elem_size(L.dtype);
    const size_t sbytes = L.units() * L.D * L.D * acc_size(L.dtype);
    const size_t nbytes = L.units() * 2 * L.N * acc_size(L.dtype);
    const size_t es = elem_size(L.dtype), as = acc_size(L.dtype);
    void* dq = g_host->buf(kQ, tb);
    void* dk = g_host->buf(kK, tb);
    void* dv = g_host->buf(kV, tb);
    uint8_t* dmask = valid ? static_cast<uint8_t*>(g_host->buf(kMask, (L.B - 1) * L.msb + L.N)) : nullptr;
    void* dout = out ? g_host->buf(kO, tb) : nullptr;
    void* dS = saved_S ? g_host->buf(kS, sbytes) : nullptr;
    void* dN = saved_norms ? g_host->buf(kNorms, nbytes) : nullptr;
    const Slices sl = plan_slices(L, tb);
    for (int i = 0; i < sl.n; ++i) {  // pipelined slices of whole sequences
      cudaStream_t st = g_host->pipe[i % kPipe];
      const int64_t b0 = i * sl.per, nb = std::min(sl.per, L.B - b0);
      Layout Lc = L;
      Lc.B = nb;
      const size_t off = b0 * L.sb * es, len = sl.bytes(L, nb, es);
      const size_t soff = b0 * L.H * L.D * L.D * as, slen = nb * L.H * L.D * L.D * as;
      const size_t noff = b0 * L.H * 2 * L.N * as, nlen = nb * L.H * 2 * L.N * as;
      pipe_h2d(at(dq, off), at(q, off), len, st);
      pipe_h2d(at(dk, off), at(k, off), len, st);
      pipe_h2d(at(dv, off), at(v, off), len, st);
      if (dmask) pipe_h2d(dmask + b0 * L.msb, valid + b0 * L.msb, (nb - 1) * L.msb + L.N, st);
      device_fwd(Lc, at(dq, off), at(dk, off), at(dv, off), dmask ? dmask + b0 * L.msb : nullptr, m,
                 at(dout, off), at(dS, soff), at(dN, noff), st);
      pipe_d2h(at(out, off), at(dout, off), out ? len : 0, st);
      pipe_d2h(at(saved_S, soff), at(dS, soff), saved_S ? slen : 0, st);
      pipe_d2h(at(saved_norms, noff), at(dN, noff), saved_norms ? nlen : 0, st);
    }
    pipe_sync();
  });
}

int cotten_bwd_host(const cotten_desc* desc, const void* q, const void* k, const void* v,
                    const uint8_t* valid, double m, const void* d_out, const void* saved_S,
                    void* dq, void* dk, void* dv, double* dm_unit, double* dm_total) {
  g_launches = 0;
  return guarded([&] {
    Layout L = resolve(desc, "cosine_attention_backward");
    if (!q || !k || !v || !d_out) usage("cosine_attention_backward: null input");
    if (!dq || !dk || !dv) usage("cosine_attention_backward: null gradient output");
    host_check_mask(L, valid, "cosine_attention_backward");
    L.require_dense("cosine_attention_backward");
    const HostSlot slot_;  // concurrency gate, held to the end of the call
    host_begin();
    const size_t tb = L.span() * elem_size(L.dtype);
    const size_t sbytes = L.units() * L.D * L.D * acc_size(L.dtype);
    const size_t es = elem_size(L.dtype), as = acc_size(L.dtype);
    void* gq = g_host->buf(kQ, tb);
    void* gk = g_host->buf(kK, tb);
    void* gv = g_host->buf(kV, tb);
    void* gdo = g_host->buf(kDO, tb);
    uint8_t* dmask = valid ? static_cast<uint8_t*>(g_host->buf(kMask, (L.B - 1) * L.msb + L.N)) : nullptr;
    void* gS = g_host->buf(kS, sbytes);  // uploaded, or recomputed per slice when not given
    void* gdq = g_host->buf(kDQ, tb);
    void* gdk = g_host->buf(kDK, tb);
    void* gdv = g_host->buf(kDV, tb);
    double* gdm = static_cast<double*>(g_host->buf(kDm, (L.units() + 1) * sizeof(double)));
    const Slices sl = plan_slices(L, tb);
    for (int i = 0; i < sl.n; ++i) {  // pipelined slices of whole sequences
      cudaStream_t st = g_host->pipe[i % kPipe];
      const int64_t b0 = i * sl.per, nb = std::min(sl.per, L.B - b0);
      Layout Lc = L;
      Lc.B = nb;
      const size_t off = b0 * L.sb * es, len = sl.bytes(L, nb, es);
      const size_t soff = b0 * L.H * L.D * L.D * as, slen = nb * L.H * L.D * L.D * as;
      const uint8_t* mk = dmask ? dmask + b0 * L.msb : nullptr;
      pipe_h2d(at(gq, off), at(q, off), len, st);
      pipe_h2d(at(gk, off), at(k, off), len, st);
      pipe_h2d(at(gv, off), at(v, off), len, st);
      pipe_h2d(at(gdo, off), at(d_out, off), len, st);
      if (dmask) pipe_h2d(dmask + b0 * L.msb, valid + b0 * L.msb, (nb - 1) * L.msb + L.N, st);
      if (saved_S)
        pipe_h2d(at(gS, soff), at(saved_S, soff), slen, st);
      else  // the state from an S-only forward of this slice
        device_fwd(Lc, at(gq, off), at(gk, off), at(gv, off), mk, m, nullptr, at(gS, soff), nullptr, st);
      // dm per unit only: the batch total is one fixed-order sum after the slices
      device_bwd(Lc, at(gq, off), at(gk, off), at(gv, off), mk, m, at(gdo, off), at(gS, soff),
                 at(gdq, off), at(gdk, off), at(gdv, off), gdm + b0 * L.H, nullptr, st);
      pipe_d2h(at(dq, off), at(gdq, off), len, st);
      pipe_d2h(at(dk, off), at(gdk, off), len, st);
      pipe_d2h(at(dv, off), at(gdv, off), len, st);
      pipe_d2h(dm_unit ? dm_unit + b0 * L.H : nullptr, gdm + b0 * L.H, nb * L.H * sizeof(double), st);
    }
    pipe_sync();
    if (dm_total) {  // the same partition and tree as the single-launch total (bit-identical)
      dm_reduce_kernel<<<1, 256, 0, g_host->stream>>>(gdm, L.units(), gdm + L.units());
      g_launches += 1;
      COTTEN_CUDA(cudaGetLastError());
      d2h(dm_total, gdm + L.units(), sizeof(double));
    }
    COTTEN_CUDA(cudaStreamSynchronize(g_host->stream));
  });
}

}  // extern "C"

// ---- device-resident host cache -----------------------------------------------
struct cotten_host_cache {
  Layout L;
  double m = 0.0;
  int dev = 0;
  void* q = nullptr;
  void* k = nullptr;
  void* v = nullptr;
  uint8_t* mask = nullptr;
  void* S = nullptr;
  size_t tb = 0, mbytes = 0, sbytes = 0;
};

namespace {
// Per-device pool of the caches' device buffers (first fit by size).
std::mutex g_pool_mu;
std::map<int, std::multimap<size_t, void*>> g_pool;
void* pool_get(int dev, size_t bytes) {
  if (bytes == 0) return nullptr;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto& fl = g_pool[dev];
    auto it = fl.lower_bound(bytes);
    if (it != fl.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      fl.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  COTTEN_CUDA(cudaMalloc(&p, bytes));
  return p;
}
void pool_put(int dev, void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool[dev].emplace(bytes, p);
}
// Capacity actually held by a pooled block is >= the request; keep the request
// size rounded so the block returns to a bucket that serves the same shape.
size_t pool_round(size_t b) { return (b + 4095) & ~size_t(4095); }
}  // namespace

extern "C" {

int cotten_fwd_host_cached(const cotten_desc* desc, const void* q, const void* k, const void* v,
                           const uint8_t* valid, double m, void* out, void* saved_norms,
                           cotten_host_cache** cache) {
  g_launches = 0;
  return guarded([&] {
    if (!cache) usage("cosine_attention_fused: null cache output");
    *cache = nullptr;
    Layout L = resolve(desc, "cosine_attention_fused");
    if (!q || !k || !v) usage("cosine_attention_fused: null input");
    host_check_mask(L, valid, "cosine_attention_fused");
    L.require_dense("cosine_attention_fused");
    const HostSlot slot_;  // concurrency gate, held to the end of the call
    host_begin();
    std::unique_ptr<cotten_host_cache> c(new cotten_host_cache);
    c->L = L;
    c->m = m;
    COTTEN_CUDA(cudaGetDevice(&c->dev));
    const size_t es = elem_size(L.dtype), as = acc_size(L.dtype);
    c->tb = pool_round(L.span() * es);
    c->mbytes = valid ? pool_round((L.B - 1) * L.msb + L.N) : 0;
    c->sbytes = pool_round(L.units() * L.D * L.D * as);
    auto release = [&] {
      pool_put(c->dev, c->q, c->tb);
      pool_put(c->dev, c->k, c->tb);
      pool_put(c->dev, c->v, c->tb);
      pool_put(c->dev, c->mask, c->mbytes);
      pool_put(c->dev, c->S, c->sbytes);
    };
    try {
      c->q = pool_get(c->dev, c->tb);
      c->k = pool_get(c->dev, c->tb);
      c->v = pool_get(c->dev, c->tb);
      c->mask = static_cast<uint8_t*>(pool_get(c->dev, c->mbytes));
      c->S = pool_get(c->dev, c->sbytes);
      const size_t tb = L.span() * es;
      const size_t nbytes = L.units() * 2 * L.N * as;
      void* dout = out ? g_host->buf(kO, tb) : nullptr;
      void* dN = saved_norms ? g_host->buf(kNorms, nbytes) : nullptr;
      const Slices sl = plan_slices(L, tb);
      for (int i = 0; i < sl.n; ++i) {  // pipelined slices, as cotten_fwd_host
        cudaStream_t st = g_host->pipe[i % kPipe];
        const int64_t b0 = i * sl.per, nb = std::min(sl.per, L.B - b0);
        Layout Lc = L;
        Lc.B = nb;
        const size_t off = b0 * L.sb * es, len = sl.bytes(L, nb, es);
        const size_t soff = b0 * L.H * L.D * L.D * as;
        const size_t noff = b0 * L.H * 2 * L.N * as, nlen = nb * L.H * 2 * L.N * as;
        pipe_h2d(at(c->q, off), at(q, off), len, st);
        pipe_h2d(at(c->k, off), at(k, off), len, st);
        pipe_h2d(at(c->v, off), at(v, off), len, st);
        if (c->mask) pipe_h2d(c->mask + b0 * L.msb, valid + b0 * L.msb, (nb - 1) * L.msb + L.N, st);
        device_fwd(Lc, at(c->q, off), at(c->k, off), at(c->v, off),
                   c->mask ? c->mask + b0 * L.msb : nullptr, m, at(dout, off), at(c->S, soff),
                   at(dN, noff), st);
        pipe_d2h(at(out, off), at(dout, off), out ? len : 0, st);
        pipe_d2h(at(saved_norms, noff), at(dN, noff), saved_norms ? nlen : 0, st);
      }
      pipe_sync();
    } catch (...) {
      release();
      throw;
    }
    *cache = c.release();
  });
}

int cotten_bwd_host_cached(const cotten_host_cache* c, const void* d_out, void* dq, void* dk,
                           void* dv, double* dm_unit, double* dm_total) {
  g_launches = 0;
  return guarded([&] {
    if (!c) usage("cosine_attention_backward: missing cache");  // UsageError, attention.cpp:398-400
    if (!d_out) usage("cosine_attention_backward: null input");
    if (!dq || !dk || !dv) usage("cosine_attention_backward: null gradient output");
    int cur = 0;
    COTTEN_CUDA(cudaGetDevice(&cur));
    if (cur != c->dev) usage("cosine_attention_backward: cache belongs to another device");
    const Layout& L = c->L;
    const HostSlot slot_;  // concurrency gate, held to the end of the call
    host_begin();
    const size_t es = elem_size(L.dtype), as = acc_size(L.dtype);
    const size_t tb = L.span() * es;
    void* gdo = g_host->buf(kDO, tb);
    void* gdq = g_host->buf(kDQ, tb);
    void* gdk = g_host->buf(kDK, tb);
    void* gdv = g_host->buf(kDV, tb);
    double* gdm = static_cast<double*>(g_host->buf(kDm, (L.units() + 1) * sizeof(double)));
    const Slices sl = plan_slices(L, tb);
    for (int i = 0; i < sl.n; ++i) {
      cudaStream_t st = g_host->pipe[i % kPipe];
      const int64_t b0 = i * sl.per, nb = std::min(sl.per, L.B - b0);
      Layout Lc = L;
      Lc.B = nb;
      const size_t off = b0 * L.sb * es, len = sl.bytes(L, nb, es);
      const size_t soff = b0 * L.H * L.D * L.D * as;
      pipe_h2d(at(gdo, off), at(d_out, off), len, st);
      device_bwd(Lc, at(c->q, off), at(c->k, off), at(c->v, off),
                 c->mask ? c->mask + b0 * L.msb : nullptr, c->m, at(gdo, off), at(c->S, soff),
                 at(gdq, off), at(gdk, off), at(gdv, off), gdm + b0 * L.H, nullptr, st);
      pipe_d2h(at(dq, off), at(gdq, off), len, st);
      pipe_d2h(at(dk, off), at(gdk, off), len, st);
      pipe_d2h(at(dv, off), at(gdv, off), len, st);
      pipe_d2h(dm_unit ? dm_unit + b0 * L.H : nullptr, gdm + b0 * L.H, nb * L.H * sizeof(double), st);
    }
    pipe_sync();
    if (dm_total) {  // the same partition and tree as the single-launch total (bit-identical)
      dm_reduce_kernel<<<1, 256, 0, g_host->stream>>>(gdm, L.units(), gdm + L.units());
      g_launches += 1;
      COTTEN_CUDA(cudaGetLastError());
      d2h(dm_total, gdm + L.units(), sizeof(double));
    }
    COTTEN_CUDA(cudaStreamSynchronize(g_host->stream));
  });
}

int cotten_host_cache_free(cotten_host_cache* c) {
  return guarded([&] {
    if (!c) return;
    pool_put(c->dev, c->q, c->tb);
    pool_put(c->dev, c->k, c->tb);
    pool_put(c->dev, c->v, c->tb);
    pool_put(c->dev, c->mask, c->mbytes);
    pool_put(c->dev, c->S, c->sbytes);
    delete c;
  });
}

int cotten_fwd_bwd_host(const cotten_desc* desc, const void* q, const void* k, const void* v,
                        const uint8_t* valid, double m, const void* d_out, void* out, void* dq,
                        void* dk, void* dv, double* dm_total) {
  g_launches = 0;
  return guarded([&] {
    Layout L = resolve(desc, "cosine_attention_fused");
    if (!q || !k || !v || !d_out) usage("cosine_attention_fused: null input");
    if (!out || !dq || !dk || !dv) usage("cosine_attention_fused: null output");
    host_check_mask(L, valid, "cosine_attention_fused");
    L.require_dense("cosine_attention_fused");
    const HostSlot slot_;  // concurrency gate, held to the end of the call
    host_begin();
    const size_t tb = L.span() * elem_size(L.dtype);
    const size_t sbytes = L.units() * L.D * L.D * acc_size(L.dtype);
    void* gq = h2d(kQ, q, tb);
    void* gk = h2d(kK, k, tb);
    void* gv = h2d(kV, v, tb);
    void* gdo = h2d(kDO, d_out, tb);
    const uint8_t* dmask =
        valid ? static_cast<const uint8_t*>(h2d(kMask, valid, (L.B - 1) * L.msb + L.N)) : nullptr;
    void* go = g_host->buf(kO, tb);
    void* gS = g_host->buf(kS, sbytes);
    void* gdq = g_host->buf(kDQ, tb);
    void* gdk = g_host->buf(kDK, tb);
    void* gdv = g_host->buf(kDV, tb);
    double* gdm = static_cast<double*>(g_host->buf(kDm, (L.units() + 1) * sizeof(double)));
    device_fwd(L, gq, gk, gv, dmask, m, go, gS, nullptr, g_host->stream);
    device_bwd(L, gq, gk, gv, dmask, m, gdo, gS, gdq, gdk, gdv, gdm, gdm + L.units(),
               g_host->stream);
    d2h(out, go, tb);
    d2h(dq, gdq, tb);
    d2h(dk, gdk, tb);
    d2h(dv, gdv, tb);
    d2h(dm_total, gdm + L.units(), sizeof(double));
    COTTEN_CUDA(cudaStreamSynchronize(g_host->stream));
  });
}

}  // extern "C"
