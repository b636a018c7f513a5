/* TEST INFRASTRUCTURE ONLY — see cosine_oracle.c.  Float64 CPU restatement of
 * the reference cosine-attention operator (attention.cpp:285-441). */
#ifndef COSINE_ORACLE_H
#define COSINE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

size_t cos_oracle_true_count(const uint8_t* valid, size_t n);
int cos_oracle_fwd(const double* q, const double* k, const double* v, const uint8_t* valid,
                   size_t n, size_t d, double m, double eps, double* out, double* norm_q,
                   double* norm_k, double* qn, double* kn, double* S);
int cos_oracle_bwd(const double* qn, const double* kn, const double* norm_q,
                   const double* norm_k, const double* S, const double* v,
                   const uint8_t* valid, size_t true_n, size_t n, size_t d, double m,
                   const double* d_out, double* dq, double* dk, double* dv, double* dm);
int cos_oracle_fwd_bwd(const double* q, const double* k, const double* v, const uint8_t* valid,
                       size_t n, size_t d, double m, double eps, const double* d_out,
                       double* out, double* dq, double* dk, double* dv, double* dm);
int cos_oracle_naive(const double* q, const double* k, const double* v, size_t n, size_t d,
                     double m, double eps, double* out);
int cos_oracle_batched_f32(const float* q, const float* k, const float* v, const float* d_out,
                           const uint8_t* valid, int64_t B, int64_t H, int64_t N, int64_t D,
                           int64_t sb, int64_t sh, int64_t sn, int64_t mask_sb, double m,
                           double eps, double* out, double* dq, double* dk, double* dv,
                           double* dm_unit);

#ifdef __cplusplus
}
#endif
#endif
