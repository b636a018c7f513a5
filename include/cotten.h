/*
 * cotten.h — C-ABI of the B200 (sm_100a) cosine-attention operator.
 *
 * The drop-in boundary under the reference's C++ operator API
 *   Matrix cosine_attention_fused(q, k, v, m, cfg, cache, mask)
 *       /root/reference/proj/include/cosrec/attention.hpp:84-86
 *       (implementation /root/reference/proj/src/attention.cpp:297-395)
 *   AttentionGrads cosine_attention_backward(cache, d_out)
 *       attention.hpp:87 (attention.cpp:397-441)
 *   attention_forward / attention_backward (cosine dispatch)
 *       attention.hpp:90-93 (attention.cpp:443-468)
 * The reference has no operator-level FFI (its C API, cosrec.h, is
 * command-level), so these entry points are what a binding for this path
 * binds; paper_2602_06935_b200/host/cosrec_adapter.cpp implements the exact
 * C++ signatures above on top of them, and INTEGRATION.md shows the wiring.
 *
 * Conventions (mirroring cosrec.h:18-22 and capi.cpp:21-44):
 *   - every entry point returns COTTEN_OK (0) or an error code; the message
 *     of the most recent failure on the calling thread is cotten_last_error();
 *   - COTTEN_ERR_USAGE covers the reference's UsageError and its ShapeError
 *     subclass (empty/mismatched shapes, mask length, a sequence with no
 *     valid row, missing saved state);
 *   - no C++ types, no torch types: plain pointers, sizes and a cudaStream_t
 *     (passed as void*, NULL = the legacy default stream).
 *
 * Semantics per (sequence b, head h) unit, v_i = valid[b][i] (1 if no mask):
 *   true_n = sum_i v_i (> 0),  s = exp(-m * ln(true_n))
 *   K~_i = v_i ? K_i / sqrt(|K_i|^2 + eps) : 0,   S = sum_i K~_i^T V_i
 *   Q~_i = Q_i / sqrt(|Q_i|^2 + eps)  (all rows), O_i = s * Q~_i S
 * and the backward of attention.cpp:397-441 (dQ all rows; dK, dV exactly 0
 * on padded rows; dm = -ln(true_n) * s * <Q~^T dO, S>).
 *
 * Layout: element (b, h, i, j) of Q/K/V/O/dO/dQ/dK/dV lives at
 *   base[b*stride_b + h*stride_h + i*stride_n + j]        (j contiguous).
 * All-zero strides select the contiguous [B][H][N][D] layout.  The mask is
 * uint8 valid[b*mask_stride_b + i] (0 = padded row), shared by all heads.
 * Workspaces: the device entry points keep small grow-only device scratch per
 * (device, stream) — per-unit dm, a recomputed S, the in-kernel dm total's
 * CTA-completion counter — so concurrent calls on different streams never
 * share it; calls on one stream are ordered.  The first call on a stream (or
 * one needing more scratch) allocates, which CUDA-graph capture forbids: run
 * one eager call on the stream before capturing it.
 * Saved state (optional in the forward, required by the backward):
 *   saved_S     [B*H][D][D]  accumulation type (float for f32/bf16, double for f64)
 *   saved_norms [B*H][2][N]  accumulation type: sqrt(|Q_i|^2+eps), then
 *               sqrt(|K_i|^2+eps) (1.0 on padded rows, attention.cpp:336)
 */
#ifndef COTTEN_H
#define COTTEN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COTTEN_OK 0
#define COTTEN_ERR_INTERNAL 1 /* CUDA failure, no device, unsupported build */
#define COTTEN_ERR_USAGE 2    /* UsageError / ShapeError in the reference */
#define COTTEN_ERR_NUMERIC 4  /* reserved (the reference op never raises it) */

#define COTTEN_F32 0
#define COTTEN_BF16 1
#define COTTEN_F64 2

/* cotten_device_status() bits, set by kernels launched through the device
 * entry points (the host entry points check these conditions up front). */
#define COTTEN_STATUS_EMPTY_SEQUENCE 1 /* a unit had true_n == 0 (outputs are NaN) */

/* Kernel-path selection (cotten_desc.flags); default 0 = fastest available. */
#define COTTEN_FLAG_FORCE_GENERIC 1 /* always use the generic-D kernels */
#define COTTEN_FLAG_FP32_PIPE 2     /* d_h = 32 fp32: FP32-pipe kernels instead of tcgen05 */

typedef struct cotten_desc {
  int64_t batch;     /* B  sequences                       */
  int64_t heads;     /* H  heads per sequence              */
  int64_t seq_len;   /* N  rows per (sequence, head)        */
  int64_t head_dim;  /* D  columns (d_h)                     */
  int32_t dtype;     /* COTTEN_F32 | COTTEN_BF16 | COTTEN_F64 */
  int32_t flags;     /* COTTEN_FLAG_*                        */
  double eps;        /* AttentionConfig::eps (attention.hpp:18) */
  int64_t stride_b;  /* element strides; all three 0 = contiguous [B][H][N][D] */
  int64_t stride_h;
  int64_t stride_n;
  int64_t mask_stride_b; /* bytes between sequences in the mask; 0 = seq_len */
} cotten_desc;

const char* cotten_version(void);
const char* cotten_last_error(void);

/* ---- device entry points: all pointers are device pointers -------------- */

/* Forward.  valid may be NULL (all rows real).  saved_S / saved_norms may be
 * NULL (inference: nothing but O reaches HBM). */
int cotten_fwd(const cotten_desc* desc, const void* q, const void* k, const void* v,
               const uint8_t* valid, double m, void* out, void* saved_S, void* saved_norms,
               void* stream);

/* Backward.  saved_S must come from cotten_fwd on the same inputs (or be NULL
 * to recompute it).  dm_unit ([B*H] doubles) and dm_total (one double: the
 * fixed-order sum over all units, deterministic) are each optional. */
int cotten_bwd(const cotten_desc* desc, const void* q, const void* k, const void* v,
               const uint8_t* valid, double m, const void* d_out, const void* saved_S,
               void* dq, void* dk, void* dv, double* dm_unit, double* dm_total, void* stream);

/* The same two calls with the exponent m read from device memory (one double,
 * e.g. a learnable per-layer parameter that an on-device optimizer updates:
 * the encoder step in cotten_encoder.h never copies it to the host).  The
 * SURVEY §8(b) proposal's `const float* m` argument. */
int cotten_fwd_mdev(const cotten_desc* desc, const void* q, const void* k, const void* v,
                    const uint8_t* valid, const double* m_dev, void* out, void* saved_S,
                    void* saved_norms, void* stream);
int cotten_bwd_mdev(const cotten_desc* desc, const void* q, const void* k, const void* v,
                    const uint8_t* valid, const double* m_dev, const void* d_out,
                    const void* saved_S, void* dq, void* dk, void* dv, double* dm_unit,
                    double* dm_total, void* stream);

/* Per-device sticky status word (COTTEN_STATUS_* bits); synchronises the
 * device.  reset != 0 clears it after reading. */
int cotten_device_status(int device, int32_t* bits, int reset);

/* ---- host entry points: all pointers are host pointers ------------------ */
/* The reference-facing call (its Matrix data lives in host memory): checks the
 * mask on the host exactly like check_qkv (attention.cpp:37-46), stages the
 * buffers to the calling thread's device workspace, runs the kernels on that
 * thread's stream and copies the results back before returning.  Thread-safe:
 * every calling thread gets its own stream and workspace (the reference calls
 * the op concurrently from parallel_chunks workers, encoder.cpp:295,345); at
 * most COTTEN_HOST_MAX_CONCURRENT (environment, default 8) host-entry calls
 * stage and run at once per process, further callers wait their turn. */
int cotten_fwd_host(const cotten_desc* desc, const void* q, const void* k, const void* v,
                    const uint8_t* valid, double m, void* out, void* saved_S,
                    void* saved_norms);
int cotten_bwd_host(const cotten_desc* desc, const void* q, const void* k, const void* v,
                    const uint8_t* valid, double m, const void* d_out, const void* saved_S,
                    void* dq, void* dk, void* dv, double* dm_unit, double* dm_total);
/* One training step of the op (forward then backward) with host buffers. */
int cotten_fwd_bwd_host(const cotten_desc* desc, const void* q, const void* k, const void* v,
                        const uint8_t* valid, double m, const void* d_out, void* out, void* dq,
                        void* dk, void* dv, double* dm_total);

/* Device-resident AttentionCache (attention.hpp:35-54) for the host entry
 * points.  The reference's backward takes only the cache and dO
 * (cosine_attention_backward(cache, d_out), attention.cpp:397): the cached
 * forward keeps its staged Q, K, V, mask and state S on the device, so the
 * backward uploads dO alone (the uncached pair uploads Q, K, V twice).
 * Opaque and caller-owned; cotten_host_cache_free returns its device buffers
 * to a per-device pool, so a training loop that frees each step's caches
 * allocates nothing after its first step.  The backward may run on another
 * host thread than the forward (same device). */
typedef struct cotten_host_cache cotten_host_cache;
int cotten_fwd_host_cached(const cotten_desc* desc, const void* q, const void* k, const void* v,
                           const uint8_t* valid, double m, void* out, void* saved_norms,
                           cotten_host_cache** cache);
int cotten_bwd_host_cached(const cotten_host_cache* cache, const void* d_out, void* dq, void* dk,
                           void* dv, double* dm_unit, double* dm_total);
int cotten_host_cache_free(cotten_host_cache* cache);

/* Number of kernel launches the last device call on this thread issued. */
int cotten_last_launch_count(void);

/* Launch-duration profile (measurement plumbing, no reference counterpart).
 * After cotten_profile_begin(stamps, slots), the i-th device call
 * (cotten_fwd / cotten_bwd) of the calling thread makes each of its kernels
 * record, with atomics on the device buffer stamps[2*i .. 2*i+1] (uint64,
 * caller-initialised to {UINT64_MAX or INT64_MAX, 0}), the earliest CTA start
 * (after its programmatic dependency resolved) and the latest warp exit in
 * %globaltimer ns.  The slot pointers are launch parameters, so a CUDA graph
 * captured while profiling records into the same slots on every replay.
 * cotten_profile_end() stops assigning slots and returns how many were used. */
int cotten_profile_begin(void* stamps, int slots);
int cotten_profile_end(void);

#ifdef __cplusplus
}
#endif
#endif /* COTTEN_H */
