/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the cosine-attention hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this code, and only as the checker or the
 * timed CPU baseline.  The product path (paper_2602_06935_b200/, libcotten.so)
 * never links or calls it; it fails loudly when its CUDA library is missing.
 *
 * A plain-C, float64 restatement of the reference operator
 *   cosine_attention_fused    /root/reference/proj/src/attention.cpp:297-395
 *   cosine_attention_backward /root/reference/proj/src/attention.cpp:397-441
 *   cosine_attention_naive    /root/reference/proj/src/attention.cpp:285-295
 * for ONE (sequence, head) unit, row-major n x d, with the reference's
 * summation order (rows ascending, the same loop nests as the blocked GEMMs in
 * /root/reference/proj/src/matrix.cpp:33-109, which add in ascending k) so that,
 * compiled with -ffp-contract=off, it reproduces the reference bit for bit.
 *
 * Parity is pinned two ways (tests/test_oracle.py):
 *   1. against the reference itself, compiled from its own sources into
 *      oracle/_ref/libcosrec_ref.so by oracle/Makefile (bit-exact on random
 *      masked inputs), and
 *   2. against the golden vectors in tests/golden/ (generated from that
 *      library by tests/golden/make_golden.py) and the reference's own
 *      known-answer tests (test_attention.cpp:93-170,212-251,
 *      test_attention_grad.cpp:62-123).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "cosine_oracle.h"

/* attention.cpp:83-87 — returns sqrt(sum x^2 + eps); callers divide by it. */
static double row_norm(const double* row, size_t d, double eps) {
  double ss = 0.0;
  for (size_t j = 0; j < d; ++j) ss += row[j] * row[j];
  return sqrt(ss + eps);
}

/* attention.cpp:26-33 (RowMask::from_valid) */
size_t cos_oracle_true_count(const uint8_t* valid, size_t n) {
  if (valid == NULL) return n;
  size_t c = 0;
  for (size_t i = 0; i < n; ++i)
    if (valid[i]) c += 1;
  return c;
}

/* attention.cpp:297-395.  Returns 0, or 2 for the reference's UsageError
 * (true_count == 0, attention.cpp:44).  norm_q / norm_k / qn / kn / S may be
 * NULL (the reference's cache == nullptr). */
int cos_oracle_fwd(const double* q, const double* k, const double* v, const uint8_t* valid,
                   size_t n, size_t d, double m, double eps, double* out, double* norm_q,
                   double* norm_k, double* qn, double* kn, double* S) {
  if (n == 0 || d == 0) return 2;
  const size_t true_n = cos_oracle_true_count(valid, n);
  if (true_n == 0) return 2;
  const double scale = exp(-m * log((double)true_n)); /* :303-304 */
  double* acc = (double*)calloc(d * d, sizeof(double));
  double* trow = (double*)malloc(d * sizeof(double));
  memset(out, 0, n * d * sizeof(double));

  /* Pass 1 (:328-361): K rows normalised on the fly; padded rows are zero. */
  for (size_t i = 0; i < n; ++i) {
    if (valid != NULL && !valid[i]) { /* :334-338 — padded K never read */
      for (size_t j = 0; j < d; ++j) trow[j] = 0.0;
      if (norm_k) norm_k[i] = 1.0;
    } else {
      const double* krow = k + i * d;
      const double norm = row_norm(krow, d, eps);
      const double inv = 1.0 / norm;
      for (size_t j = 0; j < d; ++j) trow[j] = krow[j] * inv;
      if (norm_k) norm_k[i] = norm;
    }
    const double* vrow = v + i * d; /* :345-353 */
    for (size_t a = 0; a < d; ++a) {
      const double ta = trow[a];
      double* arow = acc + a * d;
      for (size_t b = 0; b < d; ++b) arow[b] += ta * vrow[b];
    }
    if (kn)
      for (size_t j = 0; j < d; ++j) kn[i * d + j] = trow[j];
  }

  /* Pass 2 (:363-388): every Q row (padded included) normalised, O = s Q~ S. */
  for (size_t i = 0; i < n; ++i) {
    const double* qrow = q + i * d;
    const double norm = row_norm(qrow, d, eps);
    const double inv = 1.0 / norm;
    for (size_t j = 0; j < d; ++j) trow[j] = qrow[j] * inv;
    if (norm_q) norm_q[i] = norm;
    if (qn)
      for (size_t j = 0; j < d; ++j) qn[i * d + j] = trow[j];
    double* orow = out + i * d;
    for (size_t a = 0; a < d; ++a) {
      const double w = scale * trow[a];
      const double* arow = acc + a * d;
      for (size_t b = 0; b < d; ++b) orow[b] += w * arow[b];
    }
  }
  if (S) memcpy(S, acc, d * d * sizeof(double));
  free(acc);
  free(trow);
  return 0;
}

/* attention.cpp:397-441.  Inputs are the cache fields the reference keeps
 * (qn, kn, norm_q, norm_k, kv = S, v, valid, true_n, m) plus d_out. */
int cos_oracle_bwd(const double* qn, const double* kn, const double* norm_q,
                   const double* norm_k, const double* S, const double* v,
                   const uint8_t* valid, size_t true_n, size_t n, size_t d, double m,
                   const double* d_out, double* dq, double* dk, double* dv, double* dm) {
  if (n == 0 || d == 0 || true_n == 0) return 2;
  const double log_n = log((double)true_n); /* :402-403 */
  const double scale = exp(-m * log_n);
  double* qt_dout = (double*)calloc(d * d, sizeof(double));
  double* d_qn = (double*)calloc(n * d, sizeof(double));
  double* d_kn = (double*)calloc(n * d, sizeof(double));

  /* :405 gemm_tn(qn, d_out) — matrix.cpp:88-109, ascending row order */
  for (size_t kk = 0; kk < n; ++kk)
    for (size_t a = 0; a < d; ++a) {
      const double av = qn[kk * d + a];
      double* orow = qt_dout + a * d;
      for (size_t b = 0; b < d; ++b) orow[b] += av * d_out[kk * d + b];
    }
  /* :408 dm = -ln(n) * s * <Q~^T dO, S> (matrix.cpp:230-237) */
  double dot = 0.0;
  for (size_t i = 0; i < d * d; ++i) dot += qt_dout[i] * S[i];
  *dm = -log_n * scale * dot;

  /* :410-411 d_qn = s * gemm_nt(d_out, S) — matrix.cpp:60-86 */
  for (size_t i = 0; i < n; ++i)
    for (size_t a = 0; a < d; ++a) {
      double acc = 0.0;
      for (size_t b = 0; b < d; ++b) acc += d_out[i * d + b] * S[a * d + b];
      d_qn[i * d + a] = 0.0 + acc;
    }
  for (size_t i = 0; i < n * d; ++i) d_qn[i] *= scale;
  /* :412-413 dA = s * Q~^T dO */
  for (size_t i = 0; i < d * d; ++i) qt_dout[i] *= scale;
  const double* da = qt_dout;

  /* :415 d_kn = gemm_nt(v, dA) */
  for (size_t i = 0; i < n; ++i)
    for (size_t a = 0; a < d; ++a) {
      double acc = 0.0;
      for (size_t b = 0; b < d; ++b) acc += v[i * d + b] * da[a * d + b];
      d_kn[i * d + a] = 0.0 + acc;
    }
  /* :416 dv = gemm(kn, dA) — matrix.cpp:33-58, ascending inner index */
  memset(dv, 0, n * d * sizeof(double));
  for (size_t i = 0; i < n; ++i)
    for (size_t a = 0; a < d; ++a) {
      const double av = kn[i * d + a];
      for (size_t b = 0; b < d; ++b) dv[i * d + b] += av * da[a * d + b];
    }

  /* :418-438 pull through x -> x / sqrt(|x|^2 + eps) */
  memset(dq, 0, n * d * sizeof(double));
  memset(dk, 0, n * d * sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    const double* gq = d_qn + i * d;
    const double* un = qn + i * d;
    double proj = 0.0;
    for (size_t j = 0; j < d; ++j) proj += gq[j] * un[j];
    const double inv = 1.0 / norm_q[i];
    for (size_t j = 0; j < d; ++j) dq[i * d + j] = (gq[j] - proj * un[j]) * inv;
    if (valid != NULL && !valid[i]) continue; /* :430 padded keys: dk stays 0 */
    const double* gk = d_kn + i * d;
    const double* kr = kn + i * d;
    proj = 0.0;
    for (size_t j = 0; j < d; ++j) proj += gk[j] * kr[j];
    const double invk = 1.0 / norm_k[i];
    for (size_t j = 0; j < d; ++j) dk[i * d + j] = (gk[j] - proj * kr[j]) * invk;
  }
  /* :439 zero_invalid_rows(dv) */
  if (valid != NULL)
    for (size_t i = 0; i < n; ++i)
      if (!valid[i])
        for (size_t j = 0; j < d; ++j) dv[i * d + j] = 0.0;
  free(qt_dout);
  free(d_qn);
  free(d_kn);
  return 0;
}

/* Convenience: forward + backward for one unit from raw inputs, the call
 * pattern of multi_head_attention(_backward) (attention.cpp:513,554). */
int cos_oracle_fwd_bwd(const double* q, const double* k, const double* v, const uint8_t* valid,
                       size_t n, size_t d, double m, double eps, const double* d_out,
                       double* out, double* dq, double* dk, double* dv, double* dm) {
  double* nq = (double*)malloc(n * sizeof(double));
  double* nk = (double*)malloc(n * sizeof(double));
  double* qn = (double*)malloc(n * d * sizeof(double));
  double* kn = (double*)malloc(n * d * sizeof(double));
  double* S = (double*)malloc(d * d * sizeof(double));
  int rc = cos_oracle_fwd(q, k, v, valid, n, d, m, eps, out, nq, nk, qn, kn, S);
  if (rc == 0)
    rc = cos_oracle_bwd(qn, kn, nq, nk, S, v, valid, cos_oracle_true_count(valid, n), n, d, m,
                        d_out, dq, dk, dv, dm);
  free(nq);
  free(nk);
  free(qn);
  free(kn);
  free(S);
  return rc;
}

/* attention.cpp:285-295 — the n x n route (no mask), the fused op's own oracle. */
int cos_oracle_naive(const double* q, const double* k, const double* v, size_t n, size_t d,
                     double m, double eps, double* out) {
  if (n == 0 || d == 0) return 2;
  double* qn = (double*)malloc(n * d * sizeof(double));
  double* kn = (double*)malloc(n * d * sizeof(double));
  double* sim = (double*)calloc(n * n, sizeof(double));
  for (size_t i = 0; i < n; ++i) { /* matrix.cpp:138-151 */
    const double iq = 1.0 / row_norm(q + i * d, d, eps);
    const double ik = 1.0 / row_norm(k + i * d, d, eps);
    for (size_t j = 0; j < d; ++j) {
      qn[i * d + j] = q[i * d + j] * iq;
      kn[i * d + j] = k[i * d + j] * ik;
    }
  }
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (size_t a = 0; a < d; ++a) acc += qn[i * d + a] * kn[j * d + a];
      sim[i * n + j] = acc;
    }
  memset(out, 0, n * d * sizeof(double));
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < n; ++j) {
      const double s = sim[i * n + j];
      for (size_t b = 0; b < d; ++b) out[i * d + b] += s * v[j * d + b];
    }
  const double scale = exp(-m * log((double)n));
  for (size_t i = 0; i < n * d; ++i) out[i] *= scale;
  free(qn);
  free(kn);
  free(sim);
  return 0;
}

/* Batched driver over a [B][H][N][D]-strided float32 layout (the device
 * layout of include/cotten.h), widening to float64 per unit so the oracle
 * sees exactly the values the GPU sees.  Units are processed in order; the
 * per-unit dm values are written to dm_unit[b*H+h]; outputs are float64 in the
 * same strided layout.  Used by the tests as the checker for whole batches. */
int cos_oracle_batched_f32(const float* q, const float* k, const float* v, const float* d_out,
                           const uint8_t* valid, int64_t B, int64_t H, int64_t N, int64_t D,
                           int64_t sb, int64_t sh, int64_t sn, int64_t mask_sb, double m,
                           double eps, double* out, double* dq, double* dk, double* dv,
                           double* dm_unit) {
  const size_t nd = (size_t)(N * D);
  double* buf = (double*)malloc(nd * 9 * sizeof(double));
  double *qd = buf, *kd = buf + nd, *vd = buf + 2 * nd, *gd = buf + 3 * nd, *od = buf + 4 * nd;
  double *dqd = buf + 5 * nd, *dkd = buf + 6 * nd, *dvd = buf + 7 * nd;
  int rc = 0;
  for (int64_t b = 0; b < B && rc == 0; ++b)
    for (int64_t h = 0; h < H && rc == 0; ++h) {
      const int64_t base = b * sb + h * sh;
      for (int64_t i = 0; i < N; ++i)
        for (int64_t j = 0; j < D; ++j) {
          const int64_t o = base + i * sn + j;
          qd[i * D + j] = q[o];
          kd[i * D + j] = k[o];
          vd[i * D + j] = v[o];
          gd[i * D + j] = d_out ? d_out[o] : 0.0;
        }
      const uint8_t* vm = valid ? valid + b * mask_sb : NULL;
      double dm = 0.0;
      if (d_out)
        rc = cos_oracle_fwd_bwd(qd, kd, vd, vm, (size_t)N, (size_t)D, m, eps, gd, od, dqd, dkd,
                                dvd, &dm);
      else
        rc = cos_oracle_fwd(qd, kd, vd, vm, (size_t)N, (size_t)D, m, eps, od, NULL, NULL, NULL,
                            NULL, NULL);
      if (rc != 0) break;
      if (dm_unit) dm_unit[b * H + h] = dm;
      for (int64_t i = 0; i < N; ++i)
        for (int64_t j = 0; j < D; ++j) {
          const int64_t o = base + i * sn + j;
          if (out) out[o] = od[i * D + j];
          if (d_out) {
            if (dq) dq[o] = dqd[i * D + j];
            if (dk) dk[o] = dkd[i * D + j];
            if (dv) dv[o] = dvd[i * D + j];
          }
        }
    }
  free(buf);
  return rc;
}
