// Drop-in replacement of the reference's cosine-attention operator.
//
// Defines, with the reference's exact C++ signatures and types,
//   cosrec::cosine_attention_fused     (/root/reference/proj/include/cosrec/attention.hpp:84-86)
//   cosrec::cosine_attention_backward  (attention.hpp:87)
// on top of the C-ABI in include/cotten.h (the sm_100a kernels).  Compiled
// against the reference's own headers; the reference library supplies Matrix,
// AllocTracker and the error types at load time.  Linked (or LD_PRELOADed)
// ahead of the reference library, these definitions take over every call the
// reference makes through its dispatcher — attention_forward/backward
// (attention.cpp:443-468) -> multi_head_attention(_backward) (:487-565) ->
// block_forward/backward -> model_forward/backward (encoder.cpp) — with the
// reference source unchanged.
//
// Semantics mirrored from attention.cpp:
//   check_qkv (:37-46): ShapeError on empty / mismatched Q, K, V or a mask of
//   the wrong length; UsageError when the mask has no real row; tile_size == 0
//   is a UsageError (:301); the backward without a cosine cache is a
//   UsageError (:398-400).  The cache is filled like :308-322, :390-393.
// Arithmetic: the fp32 tcgen05 / FP32-pipe kernels by default (normwise
// <= 2e-4 through the reference's 2-layer encoder, tests/test_dropin.py);
// COTTEN_ADAPTER_DTYPE=f64 selects the float64 kernels, for which the
// reference's own 1e-10 tolerances hold.
// AttentionByteProbe (attention.cpp:470-485, :511-515): the host staging
// buffers of one call are TrackedAllocator vectors, so the reference's probe
// scope around each head reports them as the call's transient bytes (> 0,
// test_training.cpp:269-272); on the device nothing transient is allocated
// (per-thread persistent staging, cotten_capi.cu HostCtx).
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cotten.h"
#include "cosrec/attention.hpp"
#include "cosrec/errors.hpp"

namespace cosrec {
namespace {

std::atomic<long> g_calls{0};

int adapter_dtype() {
  const char* e = std::getenv("COTTEN_ADAPTER_DTYPE");
  return (e != nullptr && std::strcmp(e, "f64") == 0) ? COTTEN_F64 : COTTEN_F32;
}

template <typename T>
using Staging = std::vector<T, TrackedAllocator<T>>;  // seen by AllocTracker scopes

void rethrow(int rc) {
  if (rc == COTTEN_OK) return;
  const std::string msg = cotten_last_error();
  if (rc == COTTEN_ERR_USAGE) throw UsageError(msg);
  if (rc == COTTEN_ERR_NUMERIC) throw NumericError(msg);
  throw std::runtime_error(msg);
}

void check_qkv(const Matrix& q, const Matrix& k, const Matrix& v, const RowMask* mask,
               const char* what) {
  require_nonempty(q, what);
  require_same_shape(q, k, what);
  require_same_shape(q, v, what);
  if (mask != nullptr) {
    if (mask->valid.size() != q.rows()) throw ShapeError(std::string(what) + ": mask length");
    if (mask->true_count == 0) throw UsageError(std::string(what) + ": no real rows");
  }
}

cotten_desc unit_desc(std::size_t n, std::size_t d, int dtype, double eps) {
  cotten_desc desc{};
  desc.batch = 1;
  desc.heads = 1;
  desc.seq_len = static_cast<int64_t>(n);
  desc.head_dim = static_cast<int64_t>(d);
  desc.dtype = dtype;
  desc.eps = eps;
  return desc;
}

Staging<float> narrow(const Matrix& m) {
  Staging<float> f(m.size());
  for (std::size_t i = 0; i < m.size(); ++i) f[i] = static_cast<float>(m.data()[i]);
  return f;
}

}  // namespace

Matrix cosine_attention_fused(const Matrix& q, const Matrix& k, const Matrix& v, double m,
                              const AttentionConfig& cfg, AttentionCache* cache,
                              const RowMask* mask) {
  check_qkv(q, k, v, mask, "cosine_attention_fused");
  if (cfg.tile_size == 0) throw UsageError("cosine_attention_fused: tile_size must be >= 1");
  g_calls.fetch_add(1, std::memory_order_relaxed);
  const std::size_t n = q.rows(), d = q.cols();
  const int dtype = adapter_dtype();
  const cotten_desc desc = unit_desc(n, d, dtype, cfg.eps);
  const uint8_t* valid = mask != nullptr ? mask->valid.data() : nullptr;
  Matrix out = make_result(n, d);
  Staging<double> S, norms;
  if (dtype == COTTEN_F64) {
    if (cache != nullptr) {
      S.resize(d * d);
      norms.resize(2 * n);
    }
    rethrow(cotten_fwd_host(&desc, q.data(), k.data(), v.data(), valid, m, out.data(),
                            cache ? S.data() : nullptr, cache ? norms.data() : nullptr));
  } else {
    const Staging<float> fq = narrow(q), fk = narrow(k), fv = narrow(v);
    Staging<float> fo(n * d), fS(cache ? d * d : 0), fn(cache ? 2 * n : 0);
    rethrow(cotten_fwd_host(&desc, fq.data(), fk.data(), fv.data(), valid, m, fo.data(),
                            cache ? fS.data() : nullptr, cache ? fn.data() : nullptr));
    for (std::size_t i = 0; i < n * d; ++i) out.data()[i] = fo[i];
    S.assign(fS.begin(), fS.end());
    norms.assign(fn.begin(), fn.end());
  }
  if (cache != nullptr) {  // attention.cpp:308-322, :390-393
    AllocTracker::Pause pause;
    cache->mechanism = Mechanism::Cosine;
    cache->q = q;
    cache->k = k;
    cache->v = v;
    cache->qn = Matrix(n, d);
    cache->kn = Matrix(n, d);
    cache->norm_q = Matrix(n, 1);
    cache->norm_k = Matrix(n, 1);
    cache->kv = Matrix(d, d);
    for (std::size_t i = 0; i < n; ++i) {
      const bool real = mask == nullptr || mask->valid[i] != 0;
      cache->norm_q(i, 0) = norms[i];
      cache->norm_k(i, 0) = norms[n + i];  // 1.0 on padded rows (:336)
      for (std::size_t j = 0; j < d; ++j) {
        cache->qn(i, j) = q(i, j) / norms[i];
        cache->kn(i, j) = real ? k(i, j) / norms[n + i] : 0.0;
      }
    }
    std::memcpy(cache->kv.data(), S.data(), d * d * sizeof(double));
    cache->m = m;
    cache->eps = cfg.eps;
    cache->valid = mask != nullptr ? mask->valid : std::vector<std::uint8_t>{};
    cache->true_n = mask != nullptr ? mask->true_count : n;
  }
  return out;
}

AttentionGrads cosine_attention_backward(const AttentionCache& cache, const Matrix& d_out) {
  if (cache.mechanism != Mechanism::Cosine || cache.qn.empty())
    throw UsageError("cosine_attention_backward: cache missing");
  require_same_shape(cache.qn, d_out, "cosine_attention_backward");
  g_calls.fetch_add(1, std::memory_order_relaxed);
  const std::size_t n = d_out.rows(), d = d_out.cols();
  const int dtype = adapter_dtype();
  const cotten_desc desc = unit_desc(n, d, dtype, cache.eps);
  const uint8_t* valid = cache.valid.empty() ? nullptr : cache.valid.data();
  AttentionGrads g;
  g.dq = Matrix(n, d);
  g.dk = Matrix(n, d);
  g.dv = Matrix(n, d);
  double dm = 0.0;
  if (dtype == COTTEN_F64) {
    rethrow(cotten_bwd_host(&desc, cache.q.data(), cache.k.data(), cache.v.data(), valid, cache.m,
                            d_out.data(), cache.kv.data(), g.dq.data(), g.dk.data(), g.dv.data(),
                            nullptr, &dm));
  } else {
    const Staging<float> fq = narrow(cache.q), fk = narrow(cache.k), fv = narrow(cache.v);
    const Staging<float> fg = narrow(d_out), fS = narrow(cache.kv);
    Staging<float> dq(n * d), dk(n * d), dv(n * d);
    rethrow(cotten_bwd_host(&desc, fq.data(), fk.data(), fv.data(), valid, cache.m, fg.data(),
                            fS.data(), dq.data(), dk.data(), dv.data(), nullptr, &dm));
    for (std::size_t i = 0; i < n * d; ++i) {
      g.dq.data()[i] = dq[i];
      g.dk.data()[i] = dk[i];
      g.dv.data()[i] = dv[i];
    }
  }
  g.dm = dm;
  return g;
}

}  // namespace cosrec

// Number of operator calls served by the B200 path (proves the interposition).
extern "C" long cotten_adapter_calls(void) { return cosrec::g_calls.load(); }
