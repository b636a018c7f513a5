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
#include <cmath>
#include <cstdio>
#include <vector>

#include "cosrec/attention.hpp"
#include "cosrec/encoder.hpp"
#include "cosrec/errors.hpp"

extern "C" long cotten_adapter_calls(void) __attribute__((weak));

using namespace cosrec;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s out.bin [threads]\n", argv[0]);
    return 2;
  }
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
  ForwardOut fo = model_forward(batch, params, cfg, /*train=*/true, 11);
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
  std::printf("values=%zu adapter_calls=%ld error_contract_failures=%d\n", dump.size(), calls,
              errors);
  return errors == 0 ? 0 : 1;
}
