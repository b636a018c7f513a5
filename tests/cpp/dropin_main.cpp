// Drop-in check: the reference's OWN encoder (encoder.cpp / attention.cpp,
// compiled unmodified from /root/reference) runs a 2-layer Cotten4Rec
// forward + backward.  Built twice by tests/cpp/Makefile:
//   dropin_ref  — reference library only (CPU float64 operator);
//   dropin_gpu  — the same program with libcotten_cosrec.so linked ahead of
//                 the reference, so every cosine_attention_fused / _backward
//                 call the reference makes (attention.cpp:453,465 via
//                 multi_head_attention, encoder.cpp:311,360) lands on the B200
//                 kernels.
// Each writes logits, every parameter gradient and dm per layer as raw
// float64 to argv[1]; tests/test_dropin_gpu.py compares the two files.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "cosrec/attention.hpp"
#include "cosrec/encoder.hpp"
#include "cosrec/errors.hpp"

extern "C" long cotten_adapter_calls(void) __attribute__((weak));

using namespace cosrec;

// Bench mode (argv: out.bin threads bench B reps): the reference encoder at
// the ML-1M shape (|V| = 3706, N = 200, d = 64, H = 2, 2 layers, dropout
// 0.1), model_forward + model_backward per rep; prints the median seconds.
// Run as dropin_ref and dropin_gpu it times the reference with and without
// the B200 operator under it.
int bench(const char* out, int threads, int B, int reps) {
  ModelConfig cfg;
  cfg.vocab = 3706;
  cfg.dim = 64;
  cfg.layers = 2;
  cfg.max_seq = 200;
  cfg.dropout = 0.1;
  cfg.attn.mechanism = Mechanism::Cosine;
  cfg.attn.heads = 2;
  cfg.attn.eps = 1e-6;
  cfg.threads = threads;
  EncoderParams params = init_encoder(cfg, 7);
  std::mt19937_64 rng(5);
  SequenceBatch batch;
  for (int s = 0; s < B; ++s) {
    const int len = 20 + static_cast<int>(rng() % 181);
    std::vector<std::int32_t> ids(cfg.max_seq, kPadId);
    std::vector<std::size_t> pos;
    for (int t = 0; t < len; ++t) {
      const std::size_t slot = cfg.max_seq - len + t;
      ids[slot] = 1 + static_cast<std::int32_t>(rng() % cfg.vocab);
      if (rng() % 100 < 15) pos.push_back(slot);
    }
    if (pos.empty()) pos.push_back(cfg.max_seq - 1);
    batch.ids.push_back(ids);
    batch.positions.push_back(pos);
  }
  std::vector<double> secs;
  for (int r = 0; r <= reps; ++r) {  // rep 0 warms up (device context, workspaces)
    const auto t0 = std::chrono::steady_clock::now();
    ForwardOut fo = model_forward(batch, params, cfg, /*train=*/true, 11 + r);
    Matrix d_logits = fo.logits;
    for (std::size_t i = 0; i < d_logits.size(); ++i) d_logits.data()[i] *= 0.01;
    EncoderParams grads = model_backward(fo.cache, params, cfg, d_logits);
    const auto t1 = std::chrono::steady_clock::now();
    if (r > 0) secs.push_back(std::chrono::duration<double>(t1 - t0).count());
    if (r == 0) {  // logits + every gradient of the warm-up rep, for the parity check
      std::vector<double> dump(fo.logits.data(), fo.logits.data() + fo.logits.size());
      for_each_matrix(grads, [&](Matrix& m) { dump.insert(dump.end(), m.data(), m.data() + m.size()); });
      for_each_scalar(grads, [&](double& x) { dump.push_back(x); });
      if (std::FILE* f = std::fopen(out, "wb")) {
        std::fwrite(dump.data(), sizeof(double), dump.size(), f);
        std::fclose(f);
      }
    }
  }
  std::sort(secs.begin(), secs.end());
  const long calls = cotten_adapter_calls ? cotten_adapter_calls() : -1;
  std::printf("bench B=%d threads=%d reps=%d median_s=%.6f seq_per_s=%.3f adapter_calls=%ld\n", B,
              threads, reps, secs[secs.size() / 2], B / secs[secs.size() / 2], calls);
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s out.bin [threads] [bench B reps]\n", argv[0]);
    return 2;
  }
  if (argc > 3 && std::strcmp(argv[3], "bench") == 0)
    return bench(argv[1], std::atoi(argv[2]), argc > 4 ? std::atoi(argv[4]) : 64,
                 argc > 5 ? std::atoi(argv[5]) : 3);
  ModelConfig cfg;
  cfg.vocab = 40;
  cfg.dim = 64;
  cfg.layers = 2;
  cfg.max_seq = 24;
  cfg.dropout = 0.0;
  cfg.attn.mechanism = Mechanism::Cosine;
  cfg.attn.heads = 2;
  cfg.attn.eps = 1e-6;
  cfg.threads = argc > 2 ? std::atoi(argv[2]) : 4;  // concurrent operator calls (encoder.cpp:295)
  EncoderParams params = init_encoder(cfg, 7);
  for (auto& layer : params.layers) layer.attn.m = 0.85;

  SequenceBatch batch;
  const int lens[6] = {24, 17, 5, 1, 12, 20};
  for (int s = 0; s < 6; ++s) {
    std::vector<std::int32_t> ids(cfg.max_seq, kPadId);  // left padding (data.cpp:193-199)
    for (int t = 0; t < lens[s]; ++t)
      ids[cfg.max_seq - lens[s] + t] = 1 + (7 * s + 3 * t) % static_cast<int>(cfg.vocab);
    batch.ids.push_back(ids);
    batch.positions.push_back({cfg.max_seq - 1, static_cast<std::size_t>(cfg.max_seq - 2)});
  }
  // AttentionByteProbe (attention.cpp:470-485, :511-515): the per-head peak of
  // tracked transient bytes; through the adapter these are its host staging
  // buffers (test_training.cpp:269-272 requires > 0).
  AttentionByteProbe::reset();
  AttentionByteProbe::enable();
  ForwardOut fo = model_forward(batch, params, cfg, /*train=*/true, 11);
  AttentionByteProbe::disable();
  const long probe_peak = static_cast<long>(AttentionByteProbe::peak());
  Matrix d_logits = fo.logits;
  for (std::size_t i = 0; i < d_logits.size(); ++i) d_logits.data()[i] *= 0.01;
  EncoderParams grads = model_backward(fo.cache, params, cfg, d_logits);

  std::vector<double> dump(fo.logits.data(), fo.logits.data() + fo.logits.size());
  for_each_matrix(grads, [&](Matrix& m) { dump.insert(dump.end(), m.data(), m.data() + m.size()); });
  for_each_scalar(grads, [&](double& x) { dump.push_back(x); });
  std::FILE* f = std::fopen(argv[1], "wb");
  if (!f) return 3;
  std::fwrite(dump.data(), sizeof(double), dump.size(), f);
  std::fclose(f);

  // The operator-level error contract still holds through the drop-in.
  int errors = 0;
  try {
    AttentionCache empty;
    cosine_attention_backward(empty, Matrix(2, 2));
    errors++;
  } catch (const UsageError&) {
  }
  try {
    AttentionConfig c;
    RowMask none = RowMask::from_valid({0, 0});
    cosine_attention_fused(Matrix(2, 2), Matrix(2, 2), Matrix(2, 2), 1.0, c, nullptr, &none);
    errors++;
  } catch (const UsageError&) {
  }
  try {
    AttentionConfig c;
    cosine_attention_fused(Matrix(2, 2), Matrix(3, 2), Matrix(2, 2), 1.0, c);
    errors++;
  } catch (const ShapeError&) {
  }
  const long calls = cotten_adapter_calls ? cotten_adapter_calls() : -1;
  std::printf("values=%zu adapter_calls=%ld error_contract_failures=%d probe_peak=%ld\n",
              dump.size(), calls, errors, probe_peak);
  return errors == 0 ? 0 : 1;
}
