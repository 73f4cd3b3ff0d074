/*
 * mckernel_b200.h -- C ABI of the B200-native Fastfood (McKernel) hot path.
 *
 * The reference (mckernel 0.1.0, /root/reference/pkg/src/mckernel) is pure
 * Python; it has no FFI of its own.  Each entry point below replaces one
 * reference function on the hot path (cited file:line) and is what a
 * ctypes binding inside that package would call.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers (cudaMalloc / torch CUDA
 *    storage) unless the name says host_; sizes are element counts.
 *  - `stream` is a cudaStream_t passed as void*; every call is
 *    stream-ordered and asynchronous, re-entrant, and keeps no global
 *    mutable device state -- except the one-time table builders
 *    (mck_tables_build / mck_tables_from_factors), which synchronise the
 *    stream: the conflict-free permutation slots are an edge colouring
 *    computed on the host between two device phases.
 *  - Return value: MCK_OK, MCK_ERR_VALUE (bad argument; the Python layer
 *    raises ValueError with mck_last_error() text, whose wording follows the
 *    reference's messages) or MCK_ERR_CUDA (RuntimeError).
 *  - mck_last_error() is per host thread.
 */
#ifndef MCKERNEL_B200_H_
#define MCKERNEL_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCK_OK 0
#define MCK_ERR_VALUE 1
#define MCK_ERR_CUDA 2

#define MCK_KERNEL_RBF 0     /* fastfood.py:32-39  RBF(sigma)          */
#define MCK_KERNEL_MATERN 1  /* fastfood.py:42-53  RBFMatern(sigma, t) */

#define MCK_WHT_FAST 0    /* radix butterflies in registers (throughput path)   */
#define MCK_WHT_PARITY 1  /* base-256 sequential sums + (a+b,(a+b)-2b) combine:
                             bit-exact to wht.py:103-126 on OpenBLAS SkylakeX   */

/* ------------------------------------------------------------------ misc */
int mck_abi_version(void);
const char* mck_last_error(void);

/* ------------------------------------------------- randomness (detrand.py) */
/* detrand.py:78-83 -- (seed, label, block) -> 64-bit stream key (host). */
uint64_t mck_stream_key(uint64_t seed, const char* label, uint64_t block);

/* detrand.py:128-132 -- out[i] = fmix64(key + (counter0+i)*GAMMA). */
int mck_stream_hashes(uint64_t key, uint64_t counter0, int64_t count,
                      uint64_t* out, void* stream);
/* detrand.py:139-142 -- top 53 bits * 2^-53. */
int mck_stream_uniforms(uint64_t key, uint64_t counter0, int64_t count,
                        double* out, void* stream);
/* detrand.py:147-150 -- +1.0 if the top bit is set else -1.0. */
int mck_stream_signs(uint64_t key, uint64_t counter0, int64_t count,
                     double* out, void* stream);
/* detrand.py:173-183 -- `pairs` Box-Muller pairs from uniforms at
 * counter0, counter0+1, ...; out has 2*pairs doubles. */
int mck_stream_gaussian_pairs(uint64_t key, uint64_t counter0, int64_t pairs,
                              double* out, void* stream);
/* detrand.py:186-203 -- Fisher-Yates permutations of {0..n-1} for stream
 * (seed, label, block0 + b), b = 0..count-1; out is count x n int32
 * (used for Pi, fastfood.py:146, and the epoch shuffle,
 * linear_model.py:210-211). */
int mck_fisher_yates(uint64_t seed, const char* label, uint64_t block0,
                     int32_t count, int64_t n, int32_t* out, void* stream);

/* ------------------------------------------------ factor tables (fastfood) */
/* Bytes of the opaque device tables for an (n, E) feature map: the public
 * factors B, Pi, G, C (fastfood.py:82-93) followed by kernel-private derived
 * tables (sign masks, scatter addresses with G folded in, C*scale). */
int64_t mck_tables_bytes(int64_t n, int32_t expansions);

/* fastfood.py:133-166 build_blocks -- realise every block's factors on the
 * device from the seed, then derive the kernel tables.  `tables` must hold
 * mck_tables_bytes(n, E) bytes; n = next_pow2(input_dim) <= 2^20 (Matern:
 * <= 16384, its calibration costs t*n^2 gaussians per block).  Synchronous
 * (host edge-colouring step, see Conventions). */
int mck_tables_build(void* tables, int64_t input_dim, int32_t expansions,
                     int32_t kernel_kind, double sigma, int32_t t, uint64_t seed,
                     void* stream);

/* Same tables from caller-supplied factors (E x n each, device):
 * b_signs f32, permutation i32, g_diag f32, c_diag f32 -- e.g. blocks built
 * by the reference and uploaded.  Validates the permutation. */
int mck_tables_from_factors(void* tables, int64_t input_dim, int32_t expansions,
                            double sigma, const float* b_signs, const int32_t* perm,
                            const float* g_diag, const float* c_diag, void* stream);

/* Device pointers to the public factor arrays inside `tables`
 * (E x n each): b f32, perm i32, g f32, c f32. */
int mck_tables_factors(void* tables, int64_t n, int32_t expansions, float** b,
                       int32_t** perm, float** g, float** c);

/* ---------------------------------------------------- transforms (wht.py) */
/* wht.py:142-162 wht_fast_batch -- in-place unnormalised WHT of each of
 * `rows` contiguous rows of length n (power of two), fp32. */
int mck_fwht_f32(float* data, int64_t rows, int64_t n, int32_t variant, void* stream);
/* Same, fp64 (wht.py accepts any float dtype); MCK_WHT_FAST only. */
int mck_fwht_f64(double* data, int64_t rows, int64_t n, void* stream);

/* ------------------------------------------- feature map (fastfood.py) */
/* fastfood.py:179-198 apply_zhat_batch -- z (m x n*E, row stride ldz).
 * x: m rows of input_dim floats, row stride ldx; if row_index != NULL, row
 * r of the batch is x[row_index[r]] (fused gather of a mini-batch). */
int mck_zhat_f32(const void* tables, int64_t input_dim, int32_t expansions,
                 double sigma, const float* x, int64_t m, int64_t ldx,
                 const int32_t* row_index, float* z, int64_t ldz, int32_t variant,
                 void* stream);

/* fastfood.py:209-226 feature_map_batch -- [cos z | sin z] (m x 2nE, row
 * stride ldo), times float32(1/sqrt(nE)) when normalize != 0. */
int mck_features_f32(const void* tables, int64_t input_dim, int32_t expansions,
                     double sigma, const float* x, int64_t m, int64_t ldx,
                     const int32_t* row_index, int32_t normalize, float* out,
                     int64_t ldo, int32_t variant, void* stream);

/* ------------------------------------ softmax head (linear_model.py) */
/* Scratch bytes for the head kernels at (m rows, F features, C classes). */
int64_t mck_head_scratch_bytes(int64_t m, int64_t num_features, int32_t num_classes);

/* linear_model.py:95-131 forward_batch + loss + gradients' delta, in one pass:
 * logits = phi W^T + b (float64 accumulation over fp32 phi, W float64 C x F),
 * probs = softmax, delta = (probs - onehot(labels)) / m_total (m_total = global
 * batch size when rows are sharded), loss_sum = sum_r -log(max(p_r,y_r, 1e-300)).
 * Outputs (device): probs m x C f64 (may be NULL), delta m x C f64 (may be
 * NULL), loss_sum / hits scalars (may be NULL; hits = argmax matches).
 * The label of row r is labels[label_index[r]] when label_index != NULL
 * (the same index array that gathered the batch's input rows). */
int mck_head_forward(const float* phi, int64_t m, int64_t num_features, int64_t ldphi,
                     const double* w, const double* b, int32_t num_classes,
                     const int32_t* labels, const int32_t* label_index,
                     int64_t m_total, double* probs,
                     double* delta, double* loss_sum, int64_t* hits,
                     void* scratch, void* stream);

/* linear_model.py:126-131 gradients -- dW = delta^T phi (C x F, f64) and
 * db = sum_r delta_r (C).  Overwrites dw/db.  `scratch` as for
 * mck_head_forward (mck_head_scratch_bytes(m, F, C) bytes). */
int mck_head_backward(const float* phi, int64_t m, int64_t num_features, int64_t ldphi,
                      const double* delta, int32_t num_classes, double* dw,
                      double* db, void* scratch, void* stream);

/* linear_model.py:134-142 sgd_step -- W -= lr*(dW + 2*l2*W); b -= lr*db. */
int mck_head_sgd_update(double* w, double* b, const double* dw, const double* db,
                        int64_t num_features, int32_t num_classes, double lr,
                        double l2, void* stream);

/* Fused single-GPU backward + update: W -= lr*(delta^T phi + 2*l2*W),
 * b -= lr*sum(delta), without materialising dW. */
int mck_head_backward_sgd(const float* phi, int64_t m, int64_t num_features,
                          int64_t ldphi, const double* delta, int32_t num_classes,
                          double* w, double* b, double lr, double l2, void* scratch,
                          void* stream);

/* ----------------- fused expansion -> classifier (BASELINE config 4, K6) */
/* The softmax head of linear_model.py:95-142 applied to the feature map of
 * fastfood.py:209-226 (normalize=False) without materialising the features:
 * z is produced one block at a time into an L2-resident scratch and cos/sin
 * are formed inside the contraction.  W is float32 (C x 2nE); b, logits,
 * probs, delta and the loss are float64.  Scratch:
 * mck_fused_scratch_bytes(m, n, C). */
int64_t mck_fused_scratch_bytes(int64_t m, int64_t n, int32_t num_classes);

/* Scratch for E blocks; keep_z != 0 sizes it for variant bit 2 (z of all E
 * blocks kept by the forward, m * n * E floats, and reused by the backward
 * instead of recomputing the expansion). */
int64_t mck_fused_scratch_bytes_ex(int64_t m, int64_t n, int32_t expansions, int32_t num_classes,
                                   int32_t keep_z);

/* logits = phi W^T (+ b inside the softmax), softmax, loss_sum, hits and
 * delta = (probs - onehot) / m_total, as mck_head_forward.  delta required.
 * variant bits 0 and 2 select the contraction engine: neither (default):
 * packed-FFMA2 CUDA-core kernels (MUFU / HBM bound, fused_cc.cu); bit 2
 * (value 4): tcgen05 tensor cores (kind::tf32, 3xTF32 split, TMEM
 * accumulators); bit 0 (value 1): simple CUDA-core FMA kernels (cross-check).
 * variant bit 1 (value 2): keep z -- the forward leaves z of all E blocks in
 * scratch (sized by mck_fused_scratch_bytes_ex(..., keep_z = 1)) and the
 * following backward / backward_bucket calls on the SAME x, rows and m read
 * it instead of recomputing the expansion. */
int mck_fused_forward(const void* tables, int64_t input_dim, int32_t expansions, double sigma,
                      const float* x, int64_t m, int64_t ldx, const int32_t* row_index,
                      const float* w, const double* b, int32_t num_classes,
                      const int32_t* labels, const int32_t* label_index, int64_t m_total,
                      double* logits, double* probs, double* delta, double* loss_sum,
                      int64_t* hits, void* scratch, int32_t variant, void* stream);

/* dW = delta^T phi (recomputing phi) and db = sum_r delta_r.  If w != NULL
 * the SGD update W -= lr*(dW + 2*l2*W), b -= lr*db is applied in place and
 * dw/db may be NULL; otherwise dW (float32) and db are written. */
int mck_fused_backward(const void* tables, int64_t input_dim, int32_t expansions, double sigma,
                       const float* x, int64_t m, int64_t ldx, const int32_t* row_index,
                       const double* delta, int32_t num_classes, float* dw, double* db,
                       float* w, double* b, double lr, double l2, void* scratch,
                       int32_t variant, void* stream);

/* Multi-rank backward, one all-reduce bucket at a time (SURVEY.md 8(e) c4:
 * buckets by block, overlapped with the rest of the backward).  dW of the
 * blocks [e_begin, e_begin + e_count) is written to bucket as float32
 * [C][cos columns of the range | sin columns of the range]
 * (C * 2 * e_count * n floats, contiguous), to be summed over ranks and then
 * applied with mck_fused_apply_bucket.  Replaces the dW half of
 * linear_model.py:118-131 for a slice of W's columns. */
int mck_fused_backward_bucket(const void* tables, int64_t input_dim, int32_t expansions,
                              double sigma, const float* x, int64_t m, int64_t ldx,
                              const int32_t* row_index, const double* delta, int32_t num_classes,
                              int32_t e_begin, int32_t e_count, float* bucket, void* scratch,
                              int32_t variant, void* stream);

/* db = sum_r delta_r (float64, C values) -- linear_model.py:130. */
int mck_fused_bias_grad(const double* delta, int64_t m, int32_t num_classes, double* db,
                        void* stream);

/* W[:, columns of blocks e_begin..] -= lr * (bucket + 2*l2*W) (float32) and,
 * if b != NULL, b -= lr * db (float64) -- linear_model.py:134-142 applied to
 * an all-reduced bucket. */
int mck_fused_apply_bucket(float* w, int64_t input_dim, int32_t expansions, int32_t num_classes,
                           int32_t e_begin, int32_t e_count, const float* bucket, double lr,
                           double l2, double* b, const double* db, void* stream);

/* -------------------------------------------------------------- diagnostics */
/* tcgen05 self-test: D (128 x 16) = A (128 x K) * B (16 x K)^T, kind::tf32,
 * operands via shared memory, accumulator in TMEM (K % 8 == 0, K <= 256). */
int mck_diag_umma_tf32(const float* A, const float* B, float* D, int32_t K, void* stream);

/* Host-only (no GPU): the proper 32-edge-colouring used to lay out the
 * permutation Pi (fastfood.py:192) in shared memory without bank conflicts.
 * Edge e joins left node l[e] to right node r[e] (m nodes per side, every node
 * of degree 32); col[e] in [0, 32).  Returns 0, or 1 if not 32-regular. */
int mck_diag_edge_color32(int32_t m, const int32_t* l, const int32_t* r, uint8_t* col);

#ifdef __cplusplus
}
#endif

#endif /* MCKERNEL_B200_H_ */
