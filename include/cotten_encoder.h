/*
 * cotten_encoder.h — C-ABI of the B200 Cotten4Rec encoder step around the
 * cosine-attention operator, device-resident.
 *
 * Each entry point replaces one reference function for a whole batch at once
 * (the reference runs them per sequence on parallel_chunks workers):
 *
 *   cotten_enc_assemble      make_batches/fit_sequence (data.cpp:193-222),
 *                            mask_sequence (training.cpp:15-56) and
 *                            mask_for_ids (encoder.cpp:268-272)
 *   cotten_enc_forward       model_forward (encoder.cpp:276-325): embed (:80-95),
 *                            block_forward (:183-219) x layers — multi-head
 *                            attention (attention.cpp:487-526: fused QKV
 *                            projection -> cotten_fwd on the projection output
 *                            in place -> W_o), dropout, residual, layer_norm
 *                            (:97-128), FFN-GELU — the query-slot gather
 *                            (:313-318) and prediction_scores (:259-264)
 *   cotten_enc_loss          nll_loss (training.cpp:58-87)
 *   cotten_enc_backward      model_backward (encoder.cpp:327-377):
 *                            block_backward (:221-257), layer_norm_backward
 *                            (:130-154), multi_head_attention_backward
 *                            (attention.cpp:528-565) with cotten_bwd
 *   cotten_enc_clip_adam     clip_gradients (training.cpp:89-102) + adam_step
 *                            (:111-143) on the flat gradient buffer
 *
 * Parameters, gradients and Adam moments are flat float arrays in the
 * reference's for_each_matrix order (encoder.hpp:52-72: item_embeddings,
 * position_embeddings, per layer w_q[h].., w_k[h].., w_v[h].., w_o, ffn_w1,
 * ffn_b1, ffn_w2, ffn_b2, ln1_gain, ln1_bias, ln2_gain, ln2_bias; head_w,
 * head_b) — each matrix row-major like Matrix (matrix.hpp:10-13) — followed
 * by the per-layer exponents m (for_each_scalar, encoder.hpp:74-77), kept in
 * float64 because the operator reads them as its double m.  One contiguous
 * gradient buffer is what a data-parallel step all-reduces (one NCCL call).
 *
 * Conventions as include/cotten.h: 0 = OK, COTTEN_ERR_USAGE (2) for the
 * reference's UsageError/ShapeError/DataError conditions checked on the host,
 * COTTEN_ERR_INTERNAL (1) for CUDA/cuBLAS failures; cotten_last_error().
 * Device pointers unless stated; every call is asynchronous on `stream`.
 * Arithmetic is fp32 (the reference's is fp64); GEMMs are cuBLAS SGEMM
 * (plain FP32, no TF32), the operator is the tcgen05 kernel pair.
 */
#ifndef COTTEN_ENCODER_H
#define COTTEN_ENCODER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cotten_enc_config {
  int64_t vocab;    /* |V|: real items 1..vocab; 0 = pad, vocab+1 = mask token */
  int64_t dim;      /* d (ModelConfig::dim, encoder.hpp:21) */
  int64_t layers;   /* L */
  int64_t heads;    /* H (AttentionConfig::heads); d % H == 0 */
  int64_t max_seq;  /* position-embedding rows; every batch has N <= max_seq */
  double dropout;   /* p (inverted dropout, encoder.cpp:159-165) */
  double ln_eps;    /* layer-norm eps (encoder.hpp:25) */
  double attn_eps;  /* AttentionConfig::eps */
} cotten_enc_config;

typedef struct cotten_encoder cotten_encoder; /* opaque */

/* Allocates parameters, gradients, Adam moments and the activation cache for
 * batches of up to max_batch sequences x max_seq rows and max_queries query
 * slots.  Parameters start at zero (upload real ones with cotten_enc_params). */
int cotten_enc_create(const cotten_enc_config* cfg, int64_t max_batch, int64_t max_queries,
                      cotten_encoder** out);
int cotten_enc_destroy(cotten_encoder* enc);

/* Flat layout: n_tensors = 4 + L*(3H + 9) (see cotten_enc_layout);
 * offsets[i] is the float offset of tensor i, offsets[n] = the float count;
 * the L doubles of m follow at cotten_enc_m_params / cotten_enc_m_grads. */
int64_t cotten_enc_tensor_count(const cotten_encoder* enc);
int cotten_enc_layout(const cotten_encoder* enc, int64_t* offsets /* [n+1] */,
                      int64_t* rows /* [n] */, int64_t* cols /* [n] */);
float* cotten_enc_params(cotten_encoder* enc);
float* cotten_enc_grads(cotten_encoder* enc);
double* cotten_enc_m_params(cotten_encoder* enc);
double* cotten_enc_m_grads(cotten_encoder* enc);

/* Batch assembly (f4).  Ragged histories in CSR form (items[offsets[b] ..
 * offsets[b+1]), device int32 / int64) become left-padded rows of n ids
 * (fit_sequence: the last min(len, n) items, data.cpp:193-199), then the
 * training mask (training.cpp:15-56): train != 0 draws each real slot with
 * probability p_mask (redrawn until a sequence has one), with BERT corruption
 * (80 % mask token, 10 % random item, 10 % kept) when bert != 0; train == 0
 * masks the last real slot.  Outputs: ids [B][n] (corrupted), valid [B][n]
 * (id != 0, mask_for_ids), the query slots (sequence-major, ascending) as
 * rows [K] = b*n + slot and targets [K], and the count K in *k_total (device
 * int32).  The draws come from a counter-based hash of (seed, b, slot,
 * round) — the reference's sequential mt19937_64 stream cannot be split
 * across threads — so only the eval mask is bit-identical to the reference.
 * max_queries bounds K (an error bit in cotten_device_status when exceeded). */
int cotten_enc_assemble(cotten_encoder* enc, const int32_t* items, const int64_t* offsets,
                        int64_t B, int64_t n, int train, double p_mask, int bert, uint64_t seed,
                        int32_t* ids, uint8_t* valid, int32_t* query_rows, int32_t* targets,
                        int32_t* k_total, void* stream);

/* Forward over ids [B][n] (n <= max_seq) with the query rows [K]
 * (b*n + slot).  train != 0 applies dropout: masks from `dropout_masks`
 * when non-NULL (floats in {0, 1/(1-p)}, (1 + 2L) consecutive [B*n][d]
 * blocks: embedding, then per layer the attention and the FFN branch — the
 * order the reference draws them, encoder.cpp:299-303, :190-194, :209-213),
 * else drawn on the device from `dropout_seed`.  logits [K][vocab+2] are
 * written to `logits` (or to internal storage when NULL). */
int cotten_enc_forward(cotten_encoder* enc, const int32_t* ids, int64_t B, int64_t n,
                       const int32_t* query_rows, int64_t K, int train, uint64_t dropout_seed,
                       const float* dropout_masks, float* logits, void* stream);

/* nll_loss over the last forward's logits: loss (one double, mean over the K
 * rows) and d_logits written in place of the logits (training.cpp:58-87). */
int cotten_enc_loss(cotten_encoder* enc, const int32_t* targets, double* loss, void* stream);

/* Backward of the last forward, from d_logits (the loss's, or the caller's
 * when d_logits != NULL): gradients into cotten_enc_grads / _m_grads
 * (overwritten, not accumulated). */
int cotten_enc_backward(cotten_encoder* enc, const float* d_logits, void* stream);

/* clip_gradients(max_norm) then adam_step(lr, weight_decay) with the
 * reference's betas/eps (training.hpp:40-46), on device; the pre-clip global
 * norm is written to *norm_out (device double) when non-NULL. */
int cotten_enc_clip_adam(cotten_encoder* enc, double max_norm, double lr, double weight_decay,
                         double* norm_out, void* stream);

/* Logits buffer of the last forward (device, [K][vocab+2]). */
float* cotten_enc_logits(cotten_encoder* enc);

#ifdef __cplusplus
}
#endif
#endif /* COTTEN_ENCODER_H */
