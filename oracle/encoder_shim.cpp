// TEST INFRASTRUCTURE ONLY — extern "C" entry points over the UNMODIFIED
// reference encoder / loss / optimizer / batch assembly, compiled from the
// reference's own sources (/root/reference/proj/src/{encoder,attention,matrix,
// alloc_tracker,training,data}.cpp) into oracle/_ref/libcosrec_encoder.so by
// oracle/Makefile.  The device encoder (paper_2602_06935_b200/csrc/encoder.cu)
// is checked against these calls in tests/test_encoder_gpu.py; nothing here is
// product code.
//
// Flat parameter arrays follow for_each_matrix (encoder.hpp:52-72), the same
// order as the device buffers (include/cotten_encoder.h); m separately.
//
//   ref_enc_init        init_encoder (encoder.cpp:26-60)
//   ref_enc_step        model_forward (:276-325) + nll_loss (training.cpp:58-87)
//                       + model_backward (encoder.cpp:327-377); exports the
//                       dropout masks the reference drew (for the device run)
//   ref_enc_clip_adam   clip_gradients + adam_step (training.cpp:89-143)
//   ref_fit_mask_eval   fit_sequence (data.cpp:193-199) + mask_sequence eval
//                       (training.cpp:15-56)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "cosrec/data.hpp"
#include "cosrec/encoder.hpp"
#include "cosrec/errors.hpp"
#include "cosrec/training.hpp"

using namespace cosrec;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const UsageError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

ModelConfig make_cfg(int64_t vocab, int64_t dim, int64_t layers, int64_t heads, int64_t max_seq,
                     double dropout, double ln_eps, double attn_eps) {
  ModelConfig c;
  c.vocab = (std::size_t)vocab;
  c.dim = (std::size_t)dim;
  c.layers = (std::size_t)layers;
  c.max_seq = (std::size_t)max_seq;
  c.dropout = dropout;
  c.ln_eps = ln_eps;
  c.attn.mechanism = Mechanism::Cosine;
  c.attn.heads = (std::size_t)heads;
  c.attn.eps = attn_eps;
  c.threads = 1;
  return c;
}

void to_flat(EncoderParams& p, double* flat, double* m) {
  std::size_t o = 0;
  for_each_matrix(p, [&](Matrix& x) {
    std::memcpy(flat + o, x.data(), x.size() * sizeof(double));
    o += x.size();
  });
  std::size_t l = 0;
  for_each_scalar(p, [&](double& s) { m[l++] = s; });
}
void from_flat(EncoderParams& p, const double* flat, const double* m) {
  std::size_t o = 0;
  for_each_matrix(p, [&](Matrix& x) {
    std::memcpy(x.data(), flat + o, x.size() * sizeof(double));
    o += x.size();
  });
  std::size_t l = 0;
  for_each_scalar(p, [&](double& s) { s = m[l++]; });
}

}  // namespace

extern "C" {

const char* ref_enc_last_error(void) { return g_err.c_str(); }

int64_t ref_enc_param_count(int64_t vocab, int64_t dim, int64_t layers, int64_t heads,
                            int64_t max_seq) {
  const ModelConfig c = make_cfg(vocab, dim, layers, heads, max_seq, 0.0, 1e-5, 1e-6);
  EncoderParams p = init_encoder(c, 0);
  int64_t n = 0;
  for_each_matrix(p, [&](Matrix& x) { n += (int64_t)x.size(); });
  return n;
}

int ref_enc_init(int64_t vocab, int64_t dim, int64_t layers, int64_t heads, int64_t max_seq,
                 uint64_t seed, double* flat, double* m) {
  return guarded([&] {
    const ModelConfig c = make_cfg(vocab, dim, layers, heads, max_seq, 0.0, 1e-5, 1e-6);
    EncoderParams p = init_encoder(c, seed);
    to_flat(p, flat, m);
  });
}

// ids [B][n]; per sequence the query slots positions[pos_off[b] .. pos_off[b+1]);
// targets per slot.  Outputs: logits [K][vocab+2], loss, grads (flat + m).
// train != 0 with dropout > 0 draws masks from dropout_seed exactly as
// model_forward does and copies them to masks_out [(1+2L)][B*n][d] when given.
int ref_enc_step(int64_t vocab, int64_t dim, int64_t layers, int64_t heads, int64_t max_seq,
                 double dropout, double ln_eps, double attn_eps, const double* flat,
                 const double* m, int64_t B, int64_t n, const int32_t* ids,
                 const int64_t* pos_off, const int64_t* positions, const int32_t* targets,
                 int train, uint64_t dropout_seed, double* logits_out, double* loss_out,
                 double* grads_out, double* gm_out, double* masks_out) {
  return guarded([&] {
    const ModelConfig c =
        make_cfg(vocab, dim, layers, heads, max_seq, dropout, ln_eps, attn_eps);
    EncoderParams p = init_encoder(c, 0);
    from_flat(p, flat, m);
    SequenceBatch sb;
    std::vector<int32_t> tg;
    for (int64_t b = 0; b < B; ++b) {
      sb.ids.emplace_back(ids + b * n, ids + (b + 1) * n);
      std::vector<std::size_t> pos;
      for (int64_t k = pos_off[b]; k < pos_off[b + 1]; ++k) {
        pos.push_back((std::size_t)positions[k]);
        tg.push_back(targets[k]);
      }
      sb.positions.push_back(std::move(pos));
    }
    ForwardOut f = model_forward(sb, p, c, train != 0, dropout_seed);
    if (logits_out) std::memcpy(logits_out, f.logits.data(), f.logits.size() * sizeof(double));
    LossOut lo = nll_loss(f.logits, tg);
    if (loss_out) *loss_out = lo.loss;
    EncoderParams g = model_backward(f.cache, p, c, lo.d_logits);
    if (grads_out) to_flat(g, grads_out, gm_out);
    if (masks_out && train && dropout > 0.0) {
      const std::size_t rd = (std::size_t)(B * n * dim);
      auto put = [&](std::size_t slot, int64_t b, const Matrix& mk) {
        std::memcpy(masks_out + slot * rd + (std::size_t)(b * n * dim), mk.data(),
                    mk.size() * sizeof(double));
      };
      for (int64_t b = 0; b < B; ++b) {
        const SeqCache& sc = f.cache.seqs[b];
        put(0, b, sc.emb_drop_mask);
        for (int64_t l = 0; l < layers; ++l) {
          put(1 + 2 * l, b, sc.blocks[l].drop1_mask);
          put(2 + 2 * l, b, sc.blocks[l].drop2_mask);
        }
      }
    }
  });
}

// clip_gradients then adam_step on flat arrays (state arrays updated in place)
int ref_enc_clip_adam(int64_t vocab, int64_t dim, int64_t layers, int64_t heads, int64_t max_seq,
                      double* flat, double* m, double* gflat, double* gm, double* m1flat,
                      double* m1m, double* m2flat, double* m2m, long step_before, double max_norm,
                      double lr, double wd, double* norm_out) {
  return guarded([&] {
    const ModelConfig c = make_cfg(vocab, dim, layers, heads, max_seq, 0.0, 1e-5, 1e-6);
    EncoderParams p = init_encoder(c, 0), g = p;
    from_flat(p, flat, m);
    from_flat(g, gflat, gm);
    AdamState st = make_adam_state(p);
    from_flat(st.m1, m1flat, m1m);
    from_flat(st.m2, m2flat, m2m);
    st.step = step_before;
    const double norm = clip_gradients(g, max_norm);
    if (norm_out) *norm_out = norm;
    adam_step(p, g, st, lr, wd);
    to_flat(p, flat, m);
    to_flat(g, gflat, gm);
    to_flat(st.m1, m1flat, m1m);
    to_flat(st.m2, m2flat, m2m);
  });
}

// Ragged histories -> fit_sequence(n) -> mask_sequence in eval mode: ids
// [B][n] with the last real slot replaced by the mask token, that slot and
// its target per sequence.
int ref_fit_mask_eval(const int32_t* items, const int64_t* offs, int64_t B, int64_t n,
                      int64_t vocab, int32_t* ids_out, int64_t* slot_out, int32_t* target_out) {
  return guarded([&] {
    std::mt19937_64 rng(0);
    for (int64_t b = 0; b < B; ++b) {
      std::vector<int32_t> seq(items + offs[b], items + offs[b + 1]);
      std::vector<int32_t> row = fit_sequence(seq, (std::size_t)n);
      MaskedSeq ms = mask_sequence(row, 0.15, rng, false, (std::size_t)vocab, false);
      std::memcpy(ids_out + b * n, ms.seq.data(), n * sizeof(int32_t));
      slot_out[b] = (int64_t)ms.positions[0];
      target_out[b] = ms.targets[0];
    }
  });
}

// The timed CPU arm of bench.py's encoder line: `reps` training steps of the
// reference on one batch — model_forward (cfg.threads workers, encoder.cpp:295)
// + nll_loss + model_backward (:345) + clip_gradients + adam_step, exactly the
// body of train()'s batch loop (training.cpp:176-189).  Per-rep wall seconds
// into secs_out.
int ref_enc_bench(int64_t vocab, int64_t dim, int64_t layers, int64_t heads, int64_t max_seq,
                  double dropout, int64_t threads, int64_t B, int64_t n, const int32_t* ids,
                  const int64_t* pos_off, const int64_t* positions, const int32_t* targets,
                  int reps, double* secs_out) {
  return guarded([&] {
    ModelConfig c = make_cfg(vocab, dim, layers, heads, max_seq, dropout, 1e-5, 1e-6);
    c.threads = (std::size_t)threads;
    EncoderParams p = init_encoder(c, 0);
    AdamState st = make_adam_state(p);
    SequenceBatch sb;
    std::vector<int32_t> tg;
    for (int64_t b = 0; b < B; ++b) {
      sb.ids.emplace_back(ids + b * n, ids + (b + 1) * n);
      std::vector<std::size_t> pos;
      for (int64_t k = pos_off[b]; k < pos_off[b + 1]; ++k) {
        pos.push_back((std::size_t)positions[k]);
        tg.push_back(targets[k]);
      }
      sb.positions.push_back(std::move(pos));
    }
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      ForwardOut f = model_forward(sb, p, c, true, (uint64_t)r);
      LossOut lo = nll_loss(f.logits, tg);
      EncoderParams g = model_backward(f.cache, p, c, lo.d_logits);
      clip_gradients(g, 1.0);
      adam_step(p, g, st, 1e-3, 1e-3);
      const auto t1 = std::chrono::steady_clock::now();
      secs_out[r] = std::chrono::duration<double>(t1 - t0).count();
    }
  });
}

}  // extern "C"
