// K4/K5 -- softmax head on the expanded features (replaces
// linear_model.py:95-142: forward_batch, loss, gradients, sgd_step).
//
// The head is a 10-class contraction over 16,384 features -- a tall-skinny
// GEMM.  It computes in float64 like the reference (float64 W, logits and
// gradients over float32 features).  Both contractions run on the FP64
// tensor cores (mma.sync.m8n8k4.f64) when the feature rows are float4
// aligned: the forward with 8 rows per warp over 512-feature chunks whose W
// slice sits in shared memory, the backward with dW tiles of 8 classes x 8
// features over row splits with delta in shared memory.  CUDA-core fallbacks
// (k_head_fwd / k_head_bwd) cover unaligned inputs.  Every reduction
// (split-K logits, row splits of dW, db, loss, hits) runs in a fixed order,
// so training is bit-reproducible.
#include <type_traits>

#include "mck_common.cuh"
#include "async_copy.cuh"

namespace mck {

constexpr int kMaxClasses = 16;
constexpr int kFwdK = 1024;     // features per forward CTA (W slice in smem)
constexpr int kFwdRowsPerWarp = 4;
constexpr int kFwdWarps = 8;
constexpr int kFwdRows = kFwdRowsPerWarp * kFwdWarps;  // rows per forward CTA
constexpr int kBwdFeatPerThread = 4;
constexpr int kBwdThreads = 256;
constexpr int kBwdK = kBwdFeatPerThread * kBwdThreads;  // features per backward CTA
constexpr int kBwdRowChunk = 128;

struct HeadScratch {
  double* partial;  // [KS][m][C]   split-K logits (C > 16: one [KS][m][16] region per class group)
  double* rowloss;  // [m]
  int32_t* rowhit;  // [m]
  double* dwpart;   // [RS][C][F]   row-split dW (C > 16: of one class group)
  double* logits;   // [m][C]       C > 16 only: combined logits
  double* dgroup;   // [m][16]      C > 16 only: delta columns of one class group
};

// More than 16 classes (the reference accepts any C): the NC <= 16 kernels
// run once per group of <= 16 consecutive classes (W rows are contiguous);
// a single trailing class shares a 2-class group with its predecessor, whose
// results it does not write (cw = first class the group owns).
struct ClassGroup {
  int c0, nc, cw;
};
inline int class_groups(int C, ClassGroup* gs) {
  int k = 0;
  for (int c = 0; c < C; c += kMaxClasses) {
    const int nc = C - c < kMaxClasses ? C - c : kMaxClasses;
    gs[k++] = nc >= 2 ? ClassGroup{c, nc, c} : ClassGroup{C - 2, 2, c};
  }
  return k;
}

inline int64_t head_ksplits(int64_t F) { return (F + kFwdK - 1) / kFwdK; }
inline int64_t head_ksplits_max(int64_t F) { return (F + 511) / 512; }  // k_head_fwd_dmma (kDK)
#ifndef MCK_HEAD_RS_MAX
#define MCK_HEAD_RS_MAX 8
#endif
inline int64_t head_rsplits(int64_t m, int64_t F, int32_t C) {
  int64_t rs = (int64_t(1) << 22) / ((int64_t)C * F);  // keep dW partials <= 32 MB
  if (rs > MCK_HEAD_RS_MAX) rs = MCK_HEAD_RS_MAX;
  if (rs > (m + 63) / 64) rs = (m + 63) / 64;
  return rs < 1 ? 1 : rs;
}

inline int64_t head_layout(int64_t m, int64_t F, int32_t C, char* base, HeadScratch* hs) {
  auto al = [](int64_t x) { return (x + 255) & ~int64_t(255); };
  int64_t off = 0;
  HeadScratch h{};
  const bool grouped = C > kMaxClasses;
  const int32_t G = (C + kMaxClasses - 1) / kMaxClasses;
  const int32_t Cg = grouped ? kMaxClasses : C;  // classes per kernel launch
  h.partial = (double*)(base ? base + off : nullptr);
  off += al(head_ksplits_max(F) * m * Cg * 8 * (grouped ? G : 1));
  h.rowloss = (double*)(base ? base + off : nullptr);
  off += al(m * 8);
  h.rowhit = (int32_t*)(base ? base + off : nullptr);
  off += al(m * 4);
  h.dwpart = (double*)(base ? base + off : nullptr);
  off += al(head_rsplits(m, F, Cg) * Cg * F * 8);
  if (grouped) {
    h.logits = (double*)(base ? base + off : nullptr);
    off += al(m * C * 8);
    h.dgroup = (double*)(base ? base + off : nullptr);
    off += al(m * kMaxClasses * 8);
  }
  if (hs) *hs = h;
  return off;
}

// partial[ks][r][c] = sum_{f in chunk ks} phi[r][f] * W[c][f]
template <int NC>
__global__ void __launch_bounds__(kFwdWarps * 32) k_head_fwd(const float* __restrict__ phi,
                                                             int64_t m, int64_t F, int64_t ld,
                                                             const double* __restrict__ w,
                                                             double* __restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double ws[];  // [NC][kFwdK]
  __shared__ uint64_t wbar;
  const int ks = blockIdx.y;
  const int64_t f0 = (int64_t)ks * kFwdK;
  const int nf = (int)((F - f0) < kFwdK ? (F - f0) : kFwdK);
  // W slice: one TMA bulk copy per class row (contiguous in W) when the rows
  // are 16-byte aligned, else a plain loop; columns past F are zeroed.
  const bool bulk = (F % 2 == 0) && ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
  if (bulk) {
    if (threadIdx.x == 0) {
      mbar_init(&wbar, 1);
      fence_mbar_init();
      mbar_expect_tx(&wbar, (uint32_t)(NC * nf * 8));
      for (int c = 0; c < NC; ++c) bulk_g2s(ws + c * kFwdK, w + (int64_t)c * F + f0, (uint32_t)nf * 8, &wbar);
    }
    for (int t = threadIdx.x; t < NC * kFwdK; t += blockDim.x)
      if (t % kFwdK >= nf) ws[t] = 0.0;
  } else {
    for (int t = threadIdx.x; t < NC * kFwdK; t += blockDim.x) {
      const int c = t / kFwdK, f = t % kFwdK;
      ws[t] = f < nf ? w[(int64_t)c * F + f0 + f] : 0.0;
    }
  }
  __syncthreads();
  if (bulk) mbar_wait(&wbar, 0u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * kFwdRows + warp * kFwdRowsPerWarp;
  double acc[kFwdRowsPerWarp][NC];
#pragma unroll
  for (int q = 0; q < kFwdRowsPerWarp; ++q)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[q][c] = 0.0;
  const float* pr[kFwdRowsPerWarp];
#pragma unroll
  for (int q = 0; q < kFwdRowsPerWarp; ++q) {
    const int64_t r = r0 + q < m ? r0 + q : m - 1;  // clamp: duplicates are discarded
    pr[q] = phi + r * ld + f0;
  }
  for (int f = lane; f < nf; f += 32) {
    double x[kFwdRowsPerWarp];
#pragma unroll
    for (int q = 0; q < kFwdRowsPerWarp; ++q) x[q] = (double)__ldg(pr[q] + f);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double wc = ws[c * kFwdK + f];
#pragma unroll
      for (int q = 0; q < kFwdRowsPerWarp; ++q) acc[q][c] = fma(x[q], wc, acc[q][c]);
    }
  }
#pragma unroll
  for (int q = 0; q < kFwdRowsPerWarp; ++q) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double v = acc[q][c];
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      acc[q][c] = v;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < kFwdRowsPerWarp; ++q)
      if (r0 + q < m)
#pragma unroll
        for (int c = 0; c < NC; ++c) partial[((int64_t)ks * m + r0 + q) * NC + c] = acc[q][c];
  }
}

// Same contraction on the FP64 tensor cores (mma.sync.m8n8k4.f64): a warp
// owns 8 rows, a CTA 64 rows x 512 features; classes are padded to N tiles of
// 8.  Per 16-feature group each lane loads one float4 of its row (the K order
// inside the group is permuted so that lane k of the fragment owns features
// 16u + 4k .. 16u + 4k + 3), and per k-step one W value per N tile from shared
// memory (row stride 513 doubles: conflict-free fragments).  float64 products
// and sums as before, in a different (fixed) order.
constexpr int kDK = 512;  // (head_ksplits_max sizes the partials for it)
constexpr int kDRows = 64;
constexpr int kDStride = kDK + 1;

__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int NC>
__global__ void __launch_bounds__(256) k_head_fwd_dmma(const float* __restrict__ phi, int64_t m,
                                                       int64_t F, int64_t ld,
                                                       const double* __restrict__ w,
                                                       double* __restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  constexpr int NT = (NC + 7) / 8;
  extern __shared__ __align__(16) double wsd[];  // [NT*8][kDStride]
  const int ks = blockIdx.y;
  const int64_t f0 = (int64_t)ks * kDK;
  const int nf = (int)((F - f0) < kDK ? (F - f0) : kDK);  // multiple of 16 (host check)
#pragma unroll 4
  for (int t = threadIdx.x; t < NT * 8 * kDK; t += blockDim.x) {
    const int c = t / kDK, f = t % kDK;
    wsd[c * kDStride + f] = (c < NC && f < nf) ? w[(int64_t)c * F + f0 + f] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kc = lane & 3, n = lane >> 2;
  const int64_t r0 = (int64_t)blockIdx.x * kDRows + warp * 8;
  const int64_t row = r0 + n < m ? r0 + n : m - 1;  // clamp: duplicates are discarded
  const float* pr = phi + row * ld + f0 + 4 * kc;
  const double* wb = wsd + n * kDStride + 4 * kc;
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  // eight float4 loads in flight per lane (nf / 16 is a multiple of 8 except
  // for a short last chunk, handled by the remainder loop)
  const int groups = nf / 16;
  int u = 0;
  for (; u + 8 <= groups; u += 8) {
    float4 a4[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) a4[v] = __ldg(reinterpret_cast<const float4*>(pr + 16 * (u + v)));
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double a[4] = {(double)a4[v].x, (double)a4[v].y, (double)a4[v].z, (double)a4[v].w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma_m8n8k4(acc[t], a[j], wb[t * 8 * kDStride + 16 * (u + v) + j]);
    }
  }
  for (; u < groups; ++u) {
    const float4 a4 = __ldg(reinterpret_cast<const float4*>(pr + 16 * u));
    const double a[4] = {(double)a4.x, (double)a4.y, (double)a4.z, (double)a4.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int t = 0; t < NT; ++t) dmma_m8n8k4(acc[t], a[j], wb[t * 8 * kDStride + 16 * u + j]);
  }
  const int64_t r = r0 + n;
  if (r < m)
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int c = 8 * t + 2 * kc + i;
        if (c < NC) partial[((int64_t)ks * m + r) * NC + c] = acc[t][i];
      }
}

// logits -> stable softmax (linear_model.py:79-83) -> loss / delta / argmax.
// One CTA per kSmRows rows: thread (row, class) sums the split-K partials of
// its logit in ascending split order (loads of all splits in flight), then one
// thread per row finishes the softmax from shared memory.
#ifndef MCK_SM_ROWS
#define MCK_SM_ROWS 4
#endif
constexpr int kSmRows = MCK_SM_ROWS;
__global__ void __launch_bounds__(kSmRows * kMaxClasses)
k_head_softmax(const double* __restrict__ partial, int64_t KS, int64_t m, int C,
               const double* __restrict__ b, const int32_t* __restrict__ labels,
               const int32_t* __restrict__ label_index, int64_t m_total, double* probs,
               double* delta, double* rowloss, int32_t* rowhit) {
  pdl_wait();
  pdl_trigger();
  __shared__ double zs[kSmRows][kMaxClasses];
  const int rr = threadIdx.x / kMaxClasses, c = threadIdx.x % kMaxClasses;
  const int64_t r = (int64_t)blockIdx.x * kSmRows + rr;
  if (r < m && c < C) {
    double sum = 0.0;
#pragma unroll 8
    for (int64_t k = 0; k < KS; ++k) sum += partial[(k * m + r) * C + c];
    zs[rr][c] = sum + b[c];
  }
  __syncthreads();
  if (c != 0 || r >= m) return;
  double* z = zs[rr];
  double mx = z[0];
  for (int j = 1; j < C; ++j) mx = fmax(mx, z[j]);
  for (int j = 0; j < C; ++j) z[j] = exp(z[j] - mx);
  const double sum = pairwise_serial([&](int64_t i) { return z[i]; }, 0, C);
  int arg = 0;
  for (int j = 0; j < C; ++j) {
    z[j] /= sum;
    if (z[j] > z[arg]) arg = j;  // first maximum, as numpy argmax
  }
  const int y = labels ? labels[label_index ? label_index[r] : r] : -1;
  if (probs)
    for (int j = 0; j < C; ++j) probs[r * C + j] = z[j];
  if (y >= 0) {
    rowloss[r] = -log(fmax(z[y], 1e-300));
    rowhit[r] = (arg == y) ? 1 : 0;
    if (delta)
      for (int j = 0; j < C; ++j) delta[r * C + j] = (z[j] - (j == y ? 1.0 : 0.0)) / (double)m_total;
  }
}


// fixed-order reduction of per-row loss / hits (one CTA)
__global__ void k_head_reduce(const double* rowloss, const int32_t* rowhit, int64_t m,
                              double* loss_sum, int64_t* hits) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sl[1024];
  __shared__ long long sh[1024];
  double a = 0.0;
  long long h = 0;
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) {
    a += rowloss[r];
    h += rowhit[r];
  }
  sl[threadIdx.x] = a;
  sh[threadIdx.x] = h;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sl[threadIdx.x] += sl[threadIdx.x + s];
      sh[threadIdx.x] += sh[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (loss_sum) *loss_sum = sl[0];
    if (hits) *hits = (int64_t)sh[0];
  }
}

template <int NC>
int launch_fwd(const float* phi, int64_t m, int64_t F, int64_t ld, const double* w,
               double* partial, cudaStream_t st, int64_t* ksplits) {
  // tensor-core path when rows load as float4 and 16-feature groups tile F
  const bool dmma = (F % 16 == 0) && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(phi) & 15) == 0);
  if (dmma) {
    constexpr int NT = (NC + 7) / 8;
    const size_t smem = (size_t)NT * 8 * kDStride * sizeof(double);
    auto kern = k_head_fwd_dmma<NC>;
    static PerDevice pd;
    const DeviceSlot* ds = nullptr;
    MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot&) {
      return check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem), "head fwd dmma smem");
    }));
    *ksplits = (F + kDK - 1) / kDK;
    dim3 grid((unsigned)((m + kDRows - 1) / kDRows), (unsigned)*ksplits);
    return launch_pdl(kern, grid, dim3(256), smem, st, "k_head_fwd_dmma", phi, m, F, ld, w, partial);
  }
  const size_t smem = (size_t)NC * kFwdK * sizeof(double);
  auto kern = k_head_fwd<NC>;
  if (smem > 48 * 1024)
    MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem), "head fwd smem"));
  *ksplits = head_ksplits(F);
  dim3 grid((unsigned)((m + kFwdRows - 1) / kFwdRows), (unsigned)*ksplits);
  return launch_pdl(kern, grid, dim3(kFwdWarps * 32), smem, st, "k_head_fwd", phi, m, F, ld, w, partial);
}

// logits[r][c] (c in [cw, c0+nc)) = sum_k partial[k][r][c - c0], k ascending
__global__ void k_head_combine(const double* __restrict__ partial, int64_t KS, int64_t m, int nc, int c0,
                               int cw, int C, double* __restrict__ logits) {
  pdl_wait();
  pdl_trigger();
  const int own = c0 + nc - cw;
  const int64_t total = m * own;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / own;
    const int c = cw + (int)(t - r * own);
    double sum = 0.0;
    for (int64_t k = 0; k < KS; ++k) sum += partial[(k * m + r) * nc + (c - c0)];
    logits[r * C + c] = sum;
  }
}

// k_head_softmax for any C: one thread per row over its logits in place
// (the same operation order as k_head_softmax).
__global__ void k_head_softmax_any(double* __restrict__ z_all, int64_t m, int C, const double* __restrict__ b,
                                   const int32_t* __restrict__ labels, const int32_t* __restrict__ label_index,
                                   int64_t m_total, double* probs, double* delta, double* rowloss,
                                   int32_t* rowhit) {
  pdl_wait();
  pdl_trigger();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  double* z = z_all + r * C;
  for (int j = 0; j < C; ++j) z[j] += b[j];
  double mx = z[0];
  for (int j = 1; j < C; ++j) mx = fmax(mx, z[j]);
  for (int j = 0; j < C; ++j) z[j] = exp(z[j] - mx);
  const double sum = pairwise_serial([&](int64_t i) { return z[i]; }, 0, C);
  int arg = 0;
  for (int j = 0; j < C; ++j) {
    z[j] /= sum;
    if (z[j] > z[arg]) arg = j;
  }
  const int y = labels ? labels[label_index ? label_index[r] : r] : -1;
  if (probs)
    for (int j = 0; j < C; ++j) probs[r * C + j] = z[j];
  if (y >= 0) {
    rowloss[r] = -log(fmax(z[y], 1e-300));
    rowhit[r] = (arg == y) ? 1 : 0;
    if (delta)
      for (int j = 0; j < C; ++j) delta[r * C + j] = (z[j] - (j == y ? 1.0 : 0.0)) / (double)m_total;
  }
}

// dg[r][j] = delta[r][c0 + j], j < nc
__global__ void k_head_pack_delta(const double* __restrict__ delta, int64_t m, int C, int c0, int nc,
                                  double* __restrict__ dg) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = m * nc;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / nc;
    dg[t] = delta[r * C + c0 + (int)(t - r * nc)];
  }
}

// Like k_head_dw_finish over a slice [off, off + count) of a [RS][stride] partial.
__global__ void k_head_dw_finish_slice(const double* __restrict__ dwpart, int64_t RS, int64_t stride,
                                       int64_t off, int64_t count, double* dw, double* w, double lr,
                                       double l2) {
  pdl_wait();
  pdl_trigger();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    double g = 0.0;
    for (int64_t s = 0; s < RS; ++s) g += dwpart[s * stride + off + t];
    if (w) {
      const double wv = w[t];
      if (l2 != 0.0) g += 2.0 * l2 * wv;
      w[t] = wv - lr * g;
    } else {
      dw[t] = g;
    }
  }
}

template <class Fn>
static int dispatch_classes(int C, Fn fn) {
  switch (C) {
#define MCK_D(N) case N: return fn(std::integral_constant<int, N>{});
    MCK_D(2) MCK_D(3) MCK_D(4) MCK_D(5) MCK_D(6) MCK_D(7) MCK_D(8) MCK_D(9) MCK_D(10)
    MCK_D(11) MCK_D(12) MCK_D(13) MCK_D(14) MCK_D(15) MCK_D(16)
#undef MCK_D
    default: return fail_value("internal: class group of %d", C);
  }
}

static int head_forward_grouped(const float* phi, int64_t m, int64_t F, int64_t ld, const double* w,
                                const double* b, int32_t C, const int32_t* labels,
                                const int32_t* label_index, int64_t m_total, double* probs,
                                double* delta, double* loss_sum, int64_t* hits, const HeadScratch& hs,
                                cudaStream_t st) {
  ClassGroup gs[4096];
  if (C > 16 * 4096) return fail_value("num_classes must be <= %d", 16 * 4096);
  const int G = class_groups(C, gs);
  const int64_t region = head_ksplits_max(F) * m * kMaxClasses;
  for (int g = 0; g < G; ++g) {
    double* part = hs.partial + (int64_t)g * region;
    int64_t ks = 0;
    MCK_TRY(dispatch_classes(gs[g].nc, [&](auto nc) {
      return launch_fwd<decltype(nc)::value>(phi, m, F, ld, w + (int64_t)gs[g].c0 * F, part, st, &ks);
    }));
    const int64_t own = m * (gs[g].c0 + gs[g].nc - gs[g].cw);
    MCK_TRY(launch_pdl(k_head_combine, dim3((unsigned)((own + 255) / 256 < 148 * 8 ? (own + 255) / 256 : 148 * 8)),
                       dim3(256), 0, st, "k_head_combine", (const double*)part, ks, m, gs[g].nc, gs[g].c0,
                       gs[g].cw, (int)C, hs.logits));
  }
  MCK_TRY(launch_pdl(k_head_softmax_any, dim3((unsigned)((m + 127) / 128)), dim3(128), 0, st,
                     "k_head_softmax_any", hs.logits, m, (int)C, b, labels, label_index, m_total, probs,
                     delta, hs.rowloss, hs.rowhit));
  if (labels && (loss_sum || hits))
    MCK_TRY(launch_pdl(k_head_reduce, dim3(1), dim3(1024), 0, st, "k_head_reduce",
                       (const double*)hs.rowloss, (const int32_t*)hs.rowhit, m, loss_sum, hits));
  return MCK_OK;
}

int head_forward(const float* phi, int64_t m, int64_t F, int64_t ld, const double* w,
                 const double* b, int32_t C, const int32_t* labels, const int32_t* label_index,
                 int64_t m_total, double* probs, double* delta, double* loss_sum, int64_t* hits,
                 void* scratch, cudaStream_t st) {
  if (C < 2) return fail_value("need at least two classes");
  if (m == 0) return MCK_OK;
  HeadScratch hs;
  head_layout(m, F, C, (char*)scratch, &hs);
  if (C > kMaxClasses)
    return head_forward_grouped(phi, m, F, ld, w, b, C, labels, label_index, m_total, probs, delta,
                                loss_sum, hits, hs, st);
  int64_t ksplits = 0;
  auto fwd = [&](auto nc) {
    return launch_fwd<decltype(nc)::value>(phi, m, F, ld, w, hs.partial, st, &ksplits);
  };
  int rc;
  switch (C) {
#define MCK_F(N) case N: rc = fwd(std::integral_constant<int, N>{}); break;
    MCK_F(2) MCK_F(3) MCK_F(4) MCK_F(5) MCK_F(6) MCK_F(7) MCK_F(8) MCK_F(9) MCK_F(10)
    MCK_F(11) MCK_F(12) MCK_F(13) MCK_F(14) MCK_F(15) MCK_F(16)
#undef MCK_F
    default: return fail_value("num_classes must be in 2..%d", kMaxClasses);
  }
  MCK_TRY(rc);
  MCK_TRY(launch_pdl(k_head_softmax, dim3((unsigned)((m + kSmRows - 1) / kSmRows)),
                     dim3(kSmRows * kMaxClasses), 0, st, "k_head_softmax", (const double*)hs.partial,
                     ksplits, m, (int)C, b, labels, label_index, m_total, probs, delta,
                     hs.rowloss, hs.rowhit));
  if (labels && (loss_sum || hits)) {
    MCK_TRY(launch_pdl(k_head_reduce, dim3(1), dim3(1024), 0, st, "k_head_reduce",
                       (const double*)hs.rowloss, (const int32_t*)hs.rowhit, m, loss_sum, hits));
  }
  return MCK_OK;
}

// dwpart[rs][c][f] = sum_{r in split rs} delta[r][c] * phi[r][f]
template <int NC>
__global__ void __launch_bounds__(kBwdThreads) k_head_bwd(const float* __restrict__ phi,
                                                          int64_t m, int64_t F, int64_t ld,
                                                          const double* __restrict__ delta,
                                                          int64_t rows_per_split,
                                                          double* __restrict__ dwpart) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sd[kBwdRowChunk][NC];
  const int rs = blockIdx.y;
  const int64_t rbeg = (int64_t)rs * rows_per_split;
  const int64_t rend = rbeg + rows_per_split < m ? rbeg + rows_per_split : m;
  const int64_t fb = (int64_t)blockIdx.x * kBwdK + threadIdx.x;
  double acc[kBwdFeatPerThread][NC];
#pragma unroll
  for (int j = 0; j < kBwdFeatPerThread; ++j)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[j][c] = 0.0;
  for (int64_t r0 = rbeg; r0 < rend; r0 += kBwdRowChunk) {
    const int nr = (int)(rend - r0 < kBwdRowChunk ? rend - r0 : kBwdRowChunk);
    __syncthreads();
    for (int t = threadIdx.x; t < nr * NC; t += blockDim.x) sd[t / NC][t % NC] = delta[r0 * NC + t];
    __syncthreads();
    const float* pp = phi + r0 * ld;
#pragma unroll 4
    for (int rr = 0; rr < nr; ++rr) {
      double x[kBwdFeatPerThread];
#pragma unroll
      for (int j = 0; j < kBwdFeatPerThread; ++j) {
        const int64_t f = fb + j * kBwdThreads;
        x[j] = f < F ? (double)__ldg(pp + (int64_t)rr * ld + f) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double d = sd[rr][c];
#pragma unroll
        for (int j = 0; j < kBwdFeatPerThread; ++j) acc[j][c] = fma(d, x[j], acc[j][c]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kBwdFeatPerThread; ++j) {
    const int64_t f = fb + j * kBwdThreads;
    if (f < F)
#pragma unroll
      for (int c = 0; c < NC; ++c) dwpart[((int64_t)rs * NC + c) * F + f] = acc[j][c];
  }
}

// dW = sum over row splits (fixed order); optionally W -= lr*(dW + 2*l2*W)
__global__ void k_head_dw_finish(const double* __restrict__ dwpart, int64_t RS, int64_t total,
                                 double* dw, double* w, double lr, double l2) {
  pdl_wait();
  pdl_trigger();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    double g = 0.0;
    for (int64_t s = 0; s < RS; ++s) g += dwpart[s * total + t];
    if (w) {
      const double wv = w[t];
      if (l2 != 0.0) g += 2.0 * l2 * wv;
      w[t] = wv - lr * g;
    } else {
      dw[t] = g;
    }
  }
}

// db[c] = sum_r delta[r][c] in a fixed order; optionally b -= lr*db.  One CTA per class.
__global__ void k_head_db(const double* delta, int64_t m, int C, double* db, double* b, double lr) {
  pdl_wait();
  pdl_trigger();
  __shared__ double s[256];
  const int c = blockIdx.x;
  double a = 0.0;
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) a += delta[r * C + c];
  s[threadIdx.x] = a;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) s[threadIdx.x] += s[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (db) db[c] = s[0];
    if (b) b[c] -= lr * s[0];
  }
}

// dW on the FP64 tensor cores: D (classes x features) = delta^T (classes x
// rows) * phi (rows x features), mma.sync.m8n8k4.f64 with M = classes (tiles
// of 8), K = 4 rows per step, N = features.  A warp owns 32 features as four
// N tiles whose columns are the features base + 4n + j (n = 0..7, tile j), so
// every lane loads one float4 of a row per k-step; delta comes from a shared
// tile with row stride 20 doubles (conflict-free A fragments).
constexpr int kBDF = 256;  // features per CTA (8 warps x 32)
constexpr int kBDS = 20;   // delta tile row stride (doubles)

template <int NC>
__global__ void __launch_bounds__(256) k_head_bwd_dmma(const float* __restrict__ phi, int64_t m,
                                                       int64_t F, int64_t ld,
                                                       const double* __restrict__ delta,
                                                       int64_t rows_per_split,
                                                       double* __restrict__ dwpart) {
  pdl_wait();
  pdl_trigger();
  constexpr int MT = (NC + 7) / 8;
  __shared__ double sd[kBwdRowChunk][kBDS];
  const int rs = blockIdx.y;
  const int64_t rbeg = (int64_t)rs * rows_per_split;
  const int64_t rend = rbeg + rows_per_split < m ? rbeg + rows_per_split : m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kc = lane & 3, n = lane >> 2;
  const int64_t base = (int64_t)blockIdx.x * kBDF + warp * 32;
  const int64_t fl = base + 4 * n;  // this lane's float4 of every row
  double acc[MT][4][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[t][j][0] = acc[t][j][1] = 0.0;
  for (int64_t r0 = rbeg; r0 < rend; r0 += kBwdRowChunk) {
    const int nr = (int)(rend - r0 < kBwdRowChunk ? rend - r0 : kBwdRowChunk);
    __syncthreads();
    for (int t = threadIdx.x; t < kBwdRowChunk * 16; t += blockDim.x) {
      const int rr = t >> 4, c = t & 15;
      sd[rr][c] = (rr < nr && c < NC) ? delta[(r0 + rr) * NC + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int k0 = 0; k0 < nr; k0 += 4) {
      const int64_t row = r0 + k0 + kc < rend ? r0 + k0 + kc : rend - 1;  // padded rows: delta 0
      float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (fl < F) b4 = __ldg(reinterpret_cast<const float4*>(phi + row * ld + fl));
      const double b[4] = {(double)b4.x, (double)b4.y, (double)b4.z, (double)b4.w};
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const double a = sd[k0 + kc][t * 8 + n];
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[t][j], a, b[j]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int c = t * 8 + n;
        const int64_t f = base + 4 * (2 * kc + i) + j;
        if (c < NC && f < F) dwpart[((int64_t)rs * NC + c) * F + f] = acc[t][j][i];
      }
}

template <int NC>
int launch_bwd(const float* phi, int64_t m, int64_t F, int64_t ld, const double* delta,
               const HeadScratch& hs, int64_t RS, cudaStream_t st) {
  const int64_t rows_per_split = (m + RS - 1) / RS;
  if ((F % 4 == 0) && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(phi) & 15) == 0)) {
    dim3 grid((unsigned)((F + kBDF - 1) / kBDF), (unsigned)RS);
    return launch_pdl(k_head_bwd_dmma<NC>, grid, dim3(256), 0, st, "k_head_bwd_dmma", phi, m, F, ld,
                      delta, rows_per_split, hs.dwpart);
  }
  dim3 grid((unsigned)((F + kBwdK - 1) / kBwdK), (unsigned)RS);
  MCK_TRY(launch_pdl(k_head_bwd<NC>, grid, dim3(kBwdThreads), 0, st, "k_head_bwd", phi, m, F, ld, delta,
                     rows_per_split, hs.dwpart));
  return check_launch("k_head_bwd");
}

static int head_bwd_grouped(const float* phi, int64_t m, int64_t F, int64_t ld, const double* delta,
                            int32_t C, double* dw, double* db, double* w, double* b, double lr,
                            double l2, const HeadScratch& hs, cudaStream_t st) {
  ClassGroup gs[4096];
  if (C > 16 * 4096) return fail_value("num_classes must be <= %d", 16 * 4096);
  const int G = class_groups(C, gs);
  const int64_t RS = head_rsplits(m, F, kMaxClasses);
  for (int g = 0; g < G; ++g) {
    const ClassGroup cg = gs[g];
    const int64_t pk = m * cg.nc;
    MCK_TRY(launch_pdl(k_head_pack_delta, dim3((unsigned)((pk + 255) / 256 < 148 * 4 ? (pk + 255) / 256 : 148 * 4)),
                       dim3(256), 0, st, "k_head_pack_delta", delta, m, (int)C, cg.c0, cg.nc, hs.dgroup));
    MCK_TRY(dispatch_classes(cg.nc, [&](auto nc) {
      return launch_bwd<decltype(nc)::value>(phi, m, F, ld, hs.dgroup, hs, RS, st);
    }));
    const int64_t off = (int64_t)(cg.cw - cg.c0) * F, count = (int64_t)(cg.c0 + cg.nc - cg.cw) * F;
    int64_t grid = (count + 255) / 256;
    if (grid > 148 * 8) grid = 148 * 8;
    MCK_TRY(launch_pdl(k_head_dw_finish_slice, dim3((unsigned)grid), dim3(256), 0, st,
                       "k_head_dw_finish_slice", (const double*)hs.dwpart, RS, (int64_t)cg.nc * F, off,
                       count, dw ? dw + (int64_t)cg.cw * F : nullptr, w ? w + (int64_t)cg.cw * F : nullptr,
                       lr, l2));
  }
  return launch_pdl(k_head_db, dim3(C), dim3(256), 0, st, "k_head_db", delta, m, (int)C, db, b, lr);
}

static int head_bwd_common(const float* phi, int64_t m, int64_t F, int64_t ld,
                           const double* delta, int32_t C, double* dw, double* db, double* w,
                           double* b, double lr, double l2, void* scratch, cudaStream_t st) {
  if (C < 2) return fail_value("need at least two classes");
  if (m == 0) return MCK_OK;
  HeadScratch hs;
  head_layout(m, F, C, (char*)scratch, &hs);
  if (C > kMaxClasses) return head_bwd_grouped(phi, m, F, ld, delta, C, dw, db, w, b, lr, l2, hs, st);
  const int64_t RS = head_rsplits(m, F, C);
  auto bwd = [&](auto nc) {
    return launch_bwd<decltype(nc)::value>(phi, m, F, ld, delta, hs, RS, st);
  };
  int rc;
  switch (C) {
#define MCK_B(N) case N: rc = bwd(std::integral_constant<int, N>{}); break;
    MCK_B(2) MCK_B(3) MCK_B(4) MCK_B(5) MCK_B(6) MCK_B(7) MCK_B(8) MCK_B(9) MCK_B(10)
    MCK_B(11) MCK_B(12) MCK_B(13) MCK_B(14) MCK_B(15) MCK_B(16)
#undef MCK_B
    default: return fail_value("num_classes must be in 2..%d", kMaxClasses);
  }
  MCK_TRY(rc);
  const int64_t total = (int64_t)C * F;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 8) grid = 148 * 8;
  MCK_TRY(launch_pdl(k_head_dw_finish, dim3((unsigned)grid), dim3(256), 0, st, "k_head_dw_finish",
                     (const double*)hs.dwpart, RS, total, dw, w, lr, l2));
  return launch_pdl(k_head_db, dim3(C), dim3(256), 0, st, "k_head_db", delta, m, (int)C, db, b, lr);
}

int head_backward(const float* phi, int64_t m, int64_t F, int64_t ld, const double* delta,
                  int32_t C, double* dw, double* db, void* scratch, cudaStream_t st) {
  return head_bwd_common(phi, m, F, ld, delta, C, dw, db, nullptr, nullptr, 0.0, 0.0, scratch, st);
}

int head_backward_sgd(const float* phi, int64_t m, int64_t F, int64_t ld, const double* delta,
                      int32_t C, double* w, double* b, double lr, double l2, void* scratch,
                      cudaStream_t st) {
  return head_bwd_common(phi, m, F, ld, delta, C, nullptr, nullptr, w, b, lr, l2, scratch, st);
}

__global__ void k_sgd(double* w, double* b, const double* dw, const double* db, int64_t F, int C,
                      double lr, double l2) {
  const int64_t total = F * C;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    double g = dw[t];
    if (l2 != 0.0) g += 2.0 * l2 * w[t];
    w[t] = w[t] - lr * g;
  }
  if (blockIdx.x == 0 && threadIdx.x < C) b[threadIdx.x] = b[threadIdx.x] - lr * db[threadIdx.x];
}

int head_sgd_update(double* w, double* b, const double* dw, const double* db, int64_t F,
                    int32_t C, double lr, double l2, cudaStream_t st) {
  k_sgd<<<148 * 4, 256, 0, st>>>(w, b, dw, db, F, C, lr, l2);
  return check_launch("k_sgd");
}

int64_t head_scratch_bytes(int64_t m, int64_t F, int32_t C) { return head_layout(m, F, C, nullptr, nullptr); }

// Softmax / loss / delta / hits from finished logits (without bias), used by
// the fused config-4 path (fused_head.cu).
int head_softmax_from_logits(const double* logits, int64_t m, int32_t C, const double* b,
                             const int32_t* labels, const int32_t* label_index, int64_t m_total,
                             double* probs, double* delta, double* loss_sum, int64_t* hits,
                             double* rowloss, int32_t* rowhit, cudaStream_t st) {
  if (C < 2 || C > kMaxClasses) return fail_value("num_classes must be in 2..%d", kMaxClasses);
  if (m == 0) return MCK_OK;
  MCK_TRY(launch_pdl(k_head_softmax, dim3((unsigned)((m + kSmRows - 1) / kSmRows)),
                     dim3(kSmRows * kMaxClasses), 0, st, "k_head_softmax", logits, (int64_t)1, m, (int)C,
                     b, labels, label_index, m_total, probs, delta, rowloss, rowhit));
  if (labels && (loss_sum || hits)) {
    MCK_TRY(launch_pdl(k_head_reduce, dim3(1), dim3(1024), 0, st, "k_head_reduce",
                       (const double*)rowloss, (const int32_t*)rowhit, m, loss_sum, hits));
  }
  return MCK_OK;
}

}  // namespace mck
