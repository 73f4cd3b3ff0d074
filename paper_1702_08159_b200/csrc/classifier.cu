// K4/K5 -- softmax head on the expanded features (replaces
// linear_model.py:95-142: forward_batch, loss, gradients, sgd_step).
//
// The head is a 10-class contraction over 16,384 features: ~5 FLOP per byte
// of phi, i.e. bound by reading phi (which the training step keeps L2
// resident), not by math.  It is written for CUDA cores in float64 like the
// reference (float64 W, logits and gradients over float32 features) and all
// reductions run in a fixed order, so training is bit-reproducible.
#include "mck_common.cuh"

namespace mck {

constexpr int kMaxClasses = 16;
constexpr int kFwdFeat = 256;   // features per split in the forward pass
constexpr int kFwdRows = 32;    // rows per CTA in the forward pass
constexpr int kBwdFeat = 128;   // features per CTA in the backward pass
constexpr int kBwdRowChunk = 256;

struct HeadScratch {
  double* partial;  // [KS][m][C]
  double* rowloss;  // [m]
  int32_t* rowhit;  // [m]
};

inline int64_t head_splits(int64_t F) { return (F + kFwdFeat - 1) / kFwdFeat; }

inline int64_t head_layout(int64_t m, int64_t F, int32_t C, char* base, HeadScratch* hs) {
  const int64_t KS = head_splits(F);
  auto al = [](int64_t x) { return (x + 255) & ~int64_t(255); };
  int64_t off = 0;
  HeadScratch h{};
  h.partial = (double*)(base ? base + off : nullptr);
  off += al(KS * m * C * 8);
  h.rowloss = (double*)(base ? base + off : nullptr);
  off += al(m * 8);
  h.rowhit = (int32_t*)(base ? base + off : nullptr);
  off += al(m * 4);
  if (hs) *hs = h;
  return off;
}

// partial[ks][r][c] = sum_{f in split ks} phi[r][f] * W[c][f]
__global__ void __launch_bounds__(256) k_head_fwd_partial(const float* __restrict__ phi, int64_t m,
                                                          int64_t F, int64_t ld,
                                                          const double* __restrict__ w, int C,
                                                          double* __restrict__ partial) {
  __shared__ double ws[kMaxClasses][kFwdFeat];
  const int ks = blockIdx.y;
  const int64_t f0 = (int64_t)ks * kFwdFeat;
  const int nf = (int)((F - f0) < kFwdFeat ? (F - f0) : kFwdFeat);
  for (int t = threadIdx.x; t < C * kFwdFeat; t += blockDim.x) {
    const int c = t / kFwdFeat, f = t % kFwdFeat;
    ws[c][f] = f < nf ? w[(int64_t)c * F + f0 + f] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int rr = warp; rr < kFwdRows; rr += 8) {
    const int64_t r = (int64_t)blockIdx.x * kFwdRows + rr;
    if (r >= m) break;
    double acc[kMaxClasses];
#pragma unroll
    for (int c = 0; c < kMaxClasses; ++c) acc[c] = 0.0;
    const float* pr = phi + r * ld + f0;
    for (int f = lane; f < nf; f += 32) {
      const double x = (double)pr[f];
#pragma unroll
      for (int c = 0; c < kMaxClasses; ++c)
        if (c < C) acc[c] = fma(x, ws[c][f], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < kMaxClasses; ++c) {
      if (c < C) {
        double v = acc[c];
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (lane == 0) partial[((int64_t)ks * m + r) * C + c] = v;
      }
    }
  }
}

// logits -> stable softmax (linear_model.py:79-83) -> loss / delta / argmax
__global__ void k_head_softmax(const double* __restrict__ partial, int64_t KS, int64_t m, int C,
                               const double* __restrict__ b, const int32_t* __restrict__ labels,
                               const int32_t* __restrict__ label_index, int64_t m_total, double* probs, double* delta, double* rowloss,
                               int32_t* rowhit) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  double z[kMaxClasses];
  for (int c = 0; c < C; ++c) {
    double s = 0.0;
    for (int64_t k = 0; k < KS; ++k) s += partial[(k * m + r) * C + c];
    z[c] = s + b[c];
  }
  double mx = z[0];
  for (int c = 1; c < C; ++c) mx = fmax(mx, z[c]);
  for (int c = 0; c < C; ++c) z[c] = exp(z[c] - mx);
  const double sum = pairwise_serial([&](int64_t i) { return z[i]; }, 0, C);
  int arg = 0;
  for (int c = 0; c < C; ++c) {
    z[c] /= sum;
    if (z[c] > z[arg]) arg = c;  // first maximum, as numpy argmax
  }
  const int y = labels ? labels[label_index ? label_index[r] : r] : -1;
  if (probs)
    for (int c = 0; c < C; ++c) probs[r * C + c] = z[c];
  if (y >= 0) {
    rowloss[r] = -log(fmax(z[y], 1e-300));
    rowhit[r] = (arg == y) ? 1 : 0;
    if (delta)
      for (int c = 0; c < C; ++c) delta[r * C + c] = (z[c] - (c == y ? 1.0 : 0.0)) / (double)m_total;
  }
}

// fixed-order reduction of per-row loss / hits (one CTA)
__global__ void k_head_reduce(const double* rowloss, const int32_t* rowhit, int64_t m,
                              double* loss_sum, int64_t* hits) {
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

int head_forward(const float* phi, int64_t m, int64_t F, int64_t ld, const double* w,
                 const double* b, int32_t C, const int32_t* labels, const int32_t* label_index,
                 int64_t m_total, double* probs, double* delta, double* loss_sum, int64_t* hits, void* scratch,
                 cudaStream_t st) {
  if (C < 2 || C > kMaxClasses) return fail_value("num_classes must be in 2..%d", kMaxClasses);
  if (m == 0) return MCK_OK;
  HeadScratch hs;
  head_layout(m, F, C, (char*)scratch, &hs);
  const int64_t KS = head_splits(F);
  dim3 grid((unsigned)((m + kFwdRows - 1) / kFwdRows), (unsigned)KS);
  k_head_fwd_partial<<<grid, 256, 0, st>>>(phi, m, F, ld, w, C, hs.partial);
  MCK_TRY(check_launch("k_head_fwd_partial"));
  k_head_softmax<<<(unsigned)((m + 127) / 128), 128, 0, st>>>(hs.partial, KS, m, C, b, labels,
                                                              label_index, m_total, probs, delta, hs.rowloss,
                                                              hs.rowhit);
  MCK_TRY(check_launch("k_head_softmax"));
  if (labels && (loss_sum || hits)) {
    k_head_reduce<<<1, 1024, 0, st>>>(hs.rowloss, hs.rowhit, m, loss_sum, hits);
    MCK_TRY(check_launch("k_head_reduce"));
  }
  return MCK_OK;
}

// dW[c][f] = sum_r delta[r][c] * phi[r][f]; optionally fused SGD update.
template <bool UPDATE>
__global__ void __launch_bounds__(kBwdFeat) k_head_bwd(const float* __restrict__ phi, int64_t m,
                                                       int64_t F, int64_t ld,
                                                       const double* __restrict__ delta, int C,
                                                       double* dw, double* w, double lr,
                                                       double l2) {
  __shared__ double sd[kBwdRowChunk][kMaxClasses];
  const int64_t f = (int64_t)blockIdx.x * kBwdFeat + threadIdx.x;
  double acc[kMaxClasses];
#pragma unroll
  for (int c = 0; c < kMaxClasses; ++c) acc[c] = 0.0;
  for (int64_t r0 = 0; r0 < m; r0 += kBwdRowChunk) {
    const int nr = (int)(m - r0 < kBwdRowChunk ? m - r0 : kBwdRowChunk);
    __syncthreads();
    for (int t = threadIdx.x; t < nr * kMaxClasses; t += blockDim.x) {
      const int rr = t / kMaxClasses, c = t % kMaxClasses;
      sd[rr][c] = c < C ? delta[(r0 + rr) * C + c] : 0.0;
    }
    __syncthreads();
    if (f < F) {
      const float* pp = phi + r0 * ld + f;
#pragma unroll 4
      for (int rr = 0; rr < nr; ++rr) {
        const double x = (double)pp[(int64_t)rr * ld];
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c)
          if (c < C) acc[c] = fma(sd[rr][c], x, acc[c]);
      }
    }
  }
  if (f >= F) return;
#pragma unroll
  for (int c = 0; c < kMaxClasses; ++c) {
    if (c < C) {
      if constexpr (UPDATE) {
        double g = acc[c];
        const double wv = w[(int64_t)c * F + f];
        if (l2 != 0.0) g += 2.0 * l2 * wv;
        w[(int64_t)c * F + f] = wv - lr * g;
      } else {
        dw[(int64_t)c * F + f] = acc[c];
      }
    }
  }
}

// db[c] = sum_r delta[r][c] (fixed order), optional update b -= lr*db
__global__ void k_head_db(const double* delta, int64_t m, int C, double* db, double* b, double lr) {
  const int c = threadIdx.x;
  if (c >= C) return;
  double s = 0.0;
  for (int64_t r = 0; r < m; ++r) s += delta[r * C + c];
  if (db) db[c] = s;
  if (b) b[c] -= lr * s;
}

int head_backward(const float* phi, int64_t m, int64_t F, int64_t ld, const double* delta,
                  int32_t C, double* dw, double* db, cudaStream_t st) {
  if (C < 2 || C > kMaxClasses) return fail_value("num_classes must be in 2..%d", kMaxClasses);
  const unsigned grid = (unsigned)((F + kBwdFeat - 1) / kBwdFeat);
  k_head_bwd<false><<<grid, kBwdFeat, 0, st>>>(phi, m, F, ld, delta, C, dw, nullptr, 0.0, 0.0);
  MCK_TRY(check_launch("k_head_bwd"));
  k_head_db<<<1, 32, 0, st>>>(delta, m, C, db, nullptr, 0.0);
  return check_launch("k_head_db");
}

int head_backward_sgd(const float* phi, int64_t m, int64_t F, int64_t ld, const double* delta,
                      int32_t C, double* w, double* b, double lr, double l2, cudaStream_t st) {
  if (C < 2 || C > kMaxClasses) return fail_value("num_classes must be in 2..%d", kMaxClasses);
  const unsigned grid = (unsigned)((F + kBwdFeat - 1) / kBwdFeat);
  k_head_bwd<true><<<grid, kBwdFeat, 0, st>>>(phi, m, F, ld, delta, C, nullptr, w, lr, l2);
  MCK_TRY(check_launch("k_head_bwd_sgd"));
  k_head_db<<<1, 32, 0, st>>>(delta, m, C, nullptr, b, lr);
  return check_launch("k_head_db");
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

}  // namespace mck
