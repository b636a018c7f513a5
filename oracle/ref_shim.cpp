// TEST INFRASTRUCTURE ONLY — extern "C" entry points over the UNMODIFIED
// reference operator, compiled together with the reference's own sources
// (/root/reference/proj/src/{attention,matrix,alloc_tracker}.cpp) into
// oracle/_ref/libcosrec_ref.so by oracle/Makefile.  Nothing here is product
// code: tests use it to pin the C restatement (cosine_oracle.c) and to make
// golden vectors; bench.py times it as the CPU reference arm.
//
// Calls exactly what the reference's callers call:
//   cosine_attention_fused(q, k, v, m, cfg, &cache, &mask)  attention.hpp:84-86
//   cosine_attention_backward(cache, d_out)                 attention.hpp:87
//   cosine_attention_naive(q, k, v, m, eps)                 attention.hpp:76-77
// Error mapping follows the reference C API (capi.cpp:28-44, cosrec.h:18-22).
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "cosrec/attention.hpp"
#include "cosrec/errors.hpp"

using cosrec::AttentionCache;
using cosrec::AttentionConfig;
using cosrec::AttentionGrads;
using cosrec::Matrix;
using cosrec::RowMask;

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const cosrec::UsageError& e) {
    g_last_error = e.what();
    return 2;
  } catch (const cosrec::NumericError& e) {
    g_last_error = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 1;
  }
}

Matrix from_f64(const double* p, std::size_t n, std::size_t d) {
  Matrix m(n, d);
  std::memcpy(m.data(), p, n * d * sizeof(double));
  return m;
}

void to_f64(const Matrix& m, double* p) {
  if (p) std::memcpy(p, m.data(), m.size() * sizeof(double));
}

AttentionConfig cfg_for(double eps, std::size_t tile) {
  AttentionConfig cfg;
  cfg.mechanism = cosrec::Mechanism::Cosine;
  cfg.eps = eps;
  cfg.tile_size = tile;
  return cfg;
}

// Persistent worker pool (one per process) so the timed CPU arm is not
// thread-spawn bound at small batches (SURVEY §6 caveat).
class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return static_cast<int>(workers_.size()); }
  // Runs fn(unit) for unit in [0, units) across the workers, dynamic schedule.
  void run(int64_t units, const std::function<void(int64_t)>& fn) {
    std::unique_lock<std::mutex> lk(mu_);
    fn_ = &fn;
    units_ = units;
    next_.store(0);
    pending_ = size();
    ++gen_;
    cv_.notify_all();
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(int) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int64_t)>* fn;
      int64_t units;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        fn = fn_;
        units = units_;
      }
      for (;;) {
        const int64_t u = next_.fetch_add(1);
        if (u >= units) break;
        (*fn)(u);
      }
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int64_t)>* fn_ = nullptr;
  int64_t units_ = 0;
  std::atomic<int64_t> next_{0};
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

std::unique_ptr<Pool> g_pool;
std::mutex g_pool_mu;

Pool& pool(int threads) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (threads < 1) threads = static_cast<int>(std::thread::hardware_concurrency());
  if (threads < 1) threads = 1;
  if (!g_pool || g_pool->size() != threads) {
    g_pool.reset();
    g_pool = std::make_unique<Pool>(threads);
  }
  return *g_pool;
}

}  // namespace

extern "C" {

const char* cosref_last_error(void) { return g_last_error.c_str(); }

int cosref_hardware_threads(void) { return static_cast<int>(std::thread::hardware_concurrency()); }

// One (sequence, head): the reference forward with cache (and mask if given).
// Any of the cache outputs may be NULL.
int cosref_fwd(const double* q, const double* k, const double* v, const uint8_t* valid,
               int64_t n, int64_t d, double m, double eps, int64_t tile, double* out,
               double* norm_q, double* norm_k, double* qn, double* kn, double* S,
               int64_t* true_n) {
  return guarded([&] {
    Matrix mq = from_f64(q, n, d), mk = from_f64(k, n, d), mv = from_f64(v, n, d);
    AttentionCache cache;
    RowMask mask;
    if (valid) mask = RowMask::from_valid(std::vector<uint8_t>(valid, valid + n));
    Matrix o = cosrec::cosine_attention_fused(mq, mk, mv, m, cfg_for(eps, tile), &cache,
                                              valid ? &mask : nullptr);
    to_f64(o, out);
    to_f64(cache.norm_q, norm_q);
    to_f64(cache.norm_k, norm_k);
    to_f64(cache.qn, qn);
    to_f64(cache.kn, kn);
    to_f64(cache.kv, S);
    if (true_n) *true_n = static_cast<int64_t>(cache.true_n);
  });
}

// One (sequence, head): forward with cache, then the reference backward.
int cosref_fwd_bwd(const double* q, const double* k, const double* v, const uint8_t* valid,
                   int64_t n, int64_t d, double m, double eps, int64_t tile, const double* d_out,
                   double* out, double* dq, double* dk, double* dv, double* dm) {
  return guarded([&] {
    Matrix mq = from_f64(q, n, d), mk = from_f64(k, n, d), mv = from_f64(v, n, d);
    AttentionCache cache;
    RowMask mask;
    if (valid) mask = RowMask::from_valid(std::vector<uint8_t>(valid, valid + n));
    Matrix o = cosrec::cosine_attention_fused(mq, mk, mv, m, cfg_for(eps, tile), &cache,
                                              valid ? &mask : nullptr);
    AttentionGrads g = cosrec::cosine_attention_backward(cache, from_f64(d_out, n, d));
    to_f64(o, out);
    to_f64(g.dq, dq);
    to_f64(g.dk, dk);
    to_f64(g.dv, dv);
    if (dm) *dm = g.dm;
  });
}

// The reference's n x n oracle route (no mask).
int cosref_naive(const double* q, const double* k, const double* v, int64_t n, int64_t d,
                 double m, double eps, double* out) {
  return guarded([&] {
    Matrix o = cosrec::cosine_attention_naive(from_f64(q, n, d), from_f64(k, n, d),
                                              from_f64(v, n, d), m, eps);
    to_f64(o, out);
  });
}

// Backward with an empty (never-filled) cache: the reference's UsageError.
int cosref_bwd_without_cache(int64_t n, int64_t d) {
  return guarded([&] {
    AttentionCache cache;
    cosrec::cosine_attention_backward(cache, Matrix(n, d));
  });
}

// Whole batch over the float32 [B][H][N][D]-strided device layout, on a
// persistent pool of `threads` workers (<=0: all hardware threads).  Each unit
// is widened to float64 and run through the reference forward (with cache and
// mask) and, when d_out != NULL, the reference backward — the per-(seq, head)
// call pattern of multi_head_attention(_backward) (attention.cpp:513,554).
// Results are narrowed back to float32 (outputs may be NULL to skip).
int cosref_batched_f32(const float* q, const float* k, const float* v, const float* d_out,
                       const uint8_t* valid, int64_t B, int64_t H, int64_t N, int64_t D,
                       int64_t sb, int64_t sh, int64_t sn, int64_t mask_sb, double m, double eps,
                       int64_t tile, float* out, float* dq, float* dk, float* dv,
                       double* dm_unit, int threads) {
  std::atomic<int> rc{0};
  std::mutex err_mu;
  std::string err;
  auto body = [&](int64_t u) {
    const int64_t b = u / H, h = u % H;
    const int64_t base = b * sb + h * sh;
    int code = guarded([&] {
      Matrix mq(N, D), mk(N, D), mv(N, D);
      for (int64_t i = 0; i < N; ++i)
        for (int64_t j = 0; j < D; ++j) {
          mq(i, j) = q[base + i * sn + j];
          mk(i, j) = k[base + i * sn + j];
          mv(i, j) = v[base + i * sn + j];
        }
      AttentionCache cache;
      RowMask mask;
      if (valid)
        mask = RowMask::from_valid(
            std::vector<uint8_t>(valid + b * mask_sb, valid + b * mask_sb + N));
      Matrix o = cosrec::cosine_attention_fused(mq, mk, mv, m, cfg_for(eps, tile), &cache,
                                                valid ? &mask : nullptr);
      if (out)
        for (int64_t i = 0; i < N; ++i)
          for (int64_t j = 0; j < D; ++j) out[base + i * sn + j] = static_cast<float>(o(i, j));
      if (d_out) {
        Matrix g(N, D);
        for (int64_t i = 0; i < N; ++i)
          for (int64_t j = 0; j < D; ++j) g(i, j) = d_out[base + i * sn + j];
        AttentionGrads gr = cosrec::cosine_attention_backward(cache, g);
        for (int64_t i = 0; i < N; ++i)
          for (int64_t j = 0; j < D; ++j) {
            const int64_t o2 = base + i * sn + j;
            if (dq) dq[o2] = static_cast<float>(gr.dq(i, j));
            if (dk) dk[o2] = static_cast<float>(gr.dk(i, j));
            if (dv) dv[o2] = static_cast<float>(gr.dv(i, j));
          }
        if (dm_unit) dm_unit[u] = gr.dm;
      }
    });
    if (code != 0) {
      std::lock_guard<std::mutex> lk(err_mu);
      if (rc.load() == 0) {
        rc.store(code);
        err = g_last_error;
      }
    }
  };
  pool(threads).run(B * H, body);
  if (rc.load() != 0) g_last_error = err;
  return rc.load();
}

}  // extern "C"
