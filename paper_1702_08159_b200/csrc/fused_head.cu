// K6 -- fused expansion -> softmax classifier for the largest configuration
// (BASELINE config 4: d = n = 16384, E = 32, 2^20 features per row, 10
// classes).  Features are never written to HBM:
//
//   for each group of 16 blocks: k_fastfood (z of those blocks only,
//                         fastfood_z_blocks) -> z tile (m x 16n fp32, scratch)
//                       k_fused_fwd_tc: cos/sin computed on chip from z,
//                         contracted with the group's W columns on the
//                         tensor cores into per-chunk partial logits
//                       k_fused_fold: partial logits -> float64 logits
//                         (fixed order: groups ascending, chunks in order)
//   softmax / loss / delta (classifier.cu, k_head_softmax)
//   for each group of 16 blocks: k_fastfood again (recompute z; cheaper than
//                         storing 2^20 features per row)
//                       k_fused_bwd_tc: dW columns of the group = delta^T
//                         [cos z | sin z] with cos/sin on chip, written or
//                         applied as the SGD update in place.
// (k_fused_fwd / k_fused_bwd / k_fused_dw_finish: the CUDA-core cross-check
// variant of the two contractions.)
//
// W is float32 (C x 2nE; 41.9 MB at config 4, the all-reduce payload named in
// SURVEY.md section 2.1), logits and loss float64, contraction accumulators
// float32 within a chunk of features.
#include <type_traits>

#include "mck_common.cuh"
#include "tables.cuh"

namespace mck {

int fastfood_z_blocks(const TablesView&, int32_t, double, const float*, int64_t, int64_t,
                      const int32_t*, int32_t, int32_t, float*, int64_t, bool, cudaStream_t);
int head_softmax_from_logits(const double* logits, int64_t m, int32_t C, const double* b,
                             const int32_t* labels, const int32_t* label_index, int64_t m_total,
                             double* probs, double* delta, double* loss_sum, int64_t* hits,
                             double* rowloss, int32_t* rowhit, cudaStream_t st);

constexpr int kFzChunk = 256;     // z values (512 features) per forward CTA
// Blocks whose z the producer computes per launch.  (row, block) items fill
// the producer's waves (1,024 rows x 16 blocks over 296 CTA slots: 55.4 of 56
// waves), one contraction launch covers the group (2,048 CTAs: 6.9 of 7
// waves) and launches drop 16x.  The z tile (m x 16n fp32: 1 GiB at m =
// 1,024, n = 16,384) is scratch in HBM; the features themselves (twice the
// size of z) are never written.  Measured c4 step: 1 block 6.42 ms, 4 blocks
// 5.02, 8 blocks 4.80, 16 blocks 4.70, 32 blocks 6.07.
constexpr int kFusedZBlocks = 16;
int64_t fused_tc_ksplits(int64_t n);  // fused_tc.cu
int64_t fused_cc_ksplits(int64_t nz);  // fused_cc.cu
int fused_fwd_cc(const float*, int64_t, int64_t, int64_t, int64_t, const float*, int64_t, int, int64_t,
                 int64_t, float*, float*, cudaStream_t);
int fused_bwd_cc(const float*, int64_t, int64_t, int64_t, int64_t, const float*, int, int64_t, int64_t,
                 int64_t, float*, float*, float, float, cudaStream_t);
constexpr int kFwarps = 8;
constexpr int kFrowsPerWarp = 4;
constexpr int kFrows = kFwarps * kFrowsPerWarp;
constexpr int kBzPerThread = 4;
constexpr int kBthreads = 256;
constexpr int kBz = kBzPerThread * kBthreads;  // z values per backward CTA
constexpr int kBrowChunk = 128;
constexpr int kFusedMaxClasses = 16;

// Variant bits of mck_fused_forward/backward.
constexpr int32_t kVarCudaCores = 1;  // simple CUDA-core contractions (cross-check)
constexpr int32_t kVarKeepZ = 2;      // forward keeps z of all E blocks; backward reuses it
constexpr int32_t kVarTc = 4;         // tcgen05 contractions (kind::tf32, 3xTF32)
// neither bit 0 nor bit 2: packed-FFMA2 contractions (fused_cc.cu), the default

struct FusedScratch {
  float* z;          // [groups][m][kFusedZBlocks n]: all E blocks (kept z) or one group
  float* lpart;      // [KS][m][C]     partial logits of the current block group
  double* logits;    // [m][C]
  double* rowloss;   // [m]
  int32_t* rowhit;   // [m]
  double* delta64;   // [m][C]
  float* delta32;    // [m][C]
  float* delta32p;   // [m rounded up to 8][16]  zero padded (FFMA2 backward)
  float* dwpart;     // [RS][C][2 nz]  backward partials of the current block group
  float* wt;         // [16 n][2][16]   W of the group, transposed (FFMA2 forward)
};

inline int64_t fused_rsplits(int64_t m) {
  int64_t rs = (m + 63) / 64;
  return rs > 16 ? 16 : (rs < 1 ? 1 : rs);
}

inline int64_t fused_zgroups(int32_t E, bool keep) {
  return keep ? (E + kFusedZBlocks - 1) / kFusedZBlocks : 1;
}

inline int64_t fused_mpad(int64_t m) { return (m + 127) & ~int64_t(127); }

// Group tile holding block e's z and the block's first column in it: tile
// (e / 16) at column (e % 16) n when kept; the single tile at column 0 when
// recomputed per chunk.  Tiles hold mpad rows of 16 n columns, row-major
// (reference engine) or tiled (zt_offset: FFMA2 and tcgen05 engines).
inline float* fused_ztile(float* z, int64_t m, int64_t n, int32_t e, bool keep, int64_t* col0) {
  *col0 = keep ? (int64_t)(e % kFusedZBlocks) * n : 0;
  return keep ? z + (int64_t)(e / kFusedZBlocks) * fused_mpad(m) * n * kFusedZBlocks : z;
}

inline int64_t fused_layout(int64_t m, int64_t n, int32_t E, int32_t C, bool keep, char* base,
                            FusedScratch* fs) {
  auto al = [](int64_t x) { return (x + 255) & ~int64_t(255); };
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    char* p = base ? base + off : nullptr;
    off += al(bytes);
    return p;
  };
  const int64_t nz = n * kFusedZBlocks;  // z columns handled per launch group
  const int64_t KS_cc = (nz + kFzChunk - 1) / kFzChunk, KS_tc = fused_tc_ksplits(nz);
  const int64_t KS = KS_cc > KS_tc ? KS_cc : KS_tc;   // partial-logit chunks of either variant
  FusedScratch s{};
  s.z = (float*)take(fused_zgroups(E, keep) * fused_mpad(m) * n * kFusedZBlocks * 4);
  s.lpart = (float*)take(KS * m * C * 4);
  s.logits = (double*)take(m * C * 8);
  s.rowloss = (double*)take(m * 8);
  s.rowhit = (int32_t*)take(m * 4);
  s.delta64 = (double*)take(m * C * 8);
  s.delta32 = (float*)take(m * C * 4);
  s.delta32p = (float*)take(((m + 7) & ~int64_t(7)) * 16 * 4);
  s.dwpart = (float*)take(fused_rsplits(m) * C * 2 * nz * 4);
  s.wt = (float*)take(nz * 2 * 16 * 4);
  if (fs) *fs = s;
  return off;
}

// lpart[ks][r][c] = sum_{i in chunk ks} cos(z[r][i]) W[c][e n + i] + sin(z[r][i]) W[c][D + e n + i]
template <int NC>
__global__ void __launch_bounds__(kFwarps * 32) k_fused_fwd(const float* __restrict__ z, int64_t m,
                                                            int64_t n, int64_t ldz,
                                                            const float* __restrict__ w,
                                                            int64_t F, int64_t col_cos,
                                                            int64_t col_sin, float* __restrict__ lpart) {
  __shared__ __align__(16) float wc[NC][kFzChunk];
  __shared__ __align__(16) float wsn[NC][kFzChunk];
  const int ks = blockIdx.y;
  const int64_t i0 = (int64_t)ks * kFzChunk;
  const int ni = (int)(n - i0 < kFzChunk ? n - i0 : kFzChunk);
  for (int t = threadIdx.x; t < NC * kFzChunk; t += blockDim.x) {
    const int c = t / kFzChunk, i = t % kFzChunk;
    wc[c][i] = i < ni ? w[(int64_t)c * F + col_cos + i0 + i] : 0.f;
    wsn[c][i] = i < ni ? w[(int64_t)c * F + col_sin + i0 + i] : 0.f;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * kFrows + warp * kFrowsPerWarp;
  float acc[kFrowsPerWarp][NC];
#pragma unroll
  for (int q = 0; q < kFrowsPerWarp; ++q)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[q][c] = 0.f;
  const float* zr[kFrowsPerWarp];
#pragma unroll
  for (int q = 0; q < kFrowsPerWarp; ++q) zr[q] = z + (r0 + q < m ? r0 + q : m - 1) * ldz + i0;
  for (int i = lane; i < ni; i += 32) {
    float cs[kFrowsPerWarp], sn[kFrowsPerWarp];
#pragma unroll
    for (int q = 0; q < kFrowsPerWarp; ++q) __sincosf(__ldg(zr[q] + i), &sn[q], &cs[q]);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const float a = wc[c][i], b = wsn[c][i];
#pragma unroll
      for (int q = 0; q < kFrowsPerWarp; ++q) acc[q][c] = fmaf(cs[q], a, fmaf(sn[q], b, acc[q][c]));
    }
  }
#pragma unroll
  for (int q = 0; q < kFrowsPerWarp; ++q)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      float v = acc[q][c];
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      acc[q][c] = v;
    }
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < kFrowsPerWarp; ++q)
      if (r0 + q < m)
#pragma unroll
        for (int c = 0; c < NC; ++c) lpart[((int64_t)ks * m + r0 + q) * NC + c] = acc[q][c];
}

// logits[r][c] (+)= sum_ks lpart[ks][r][c]   (float64, chunk order)
// 32 outputs per CTA; warp w sums the partials k = w, w+32, ... and the 32
// warp sums are combined in a fixed order (deterministic, independent loads).
constexpr int kFoldWarps = 32;
__global__ void __launch_bounds__(kFoldWarps * 32)
k_fused_fold(const float* __restrict__ lpart, int64_t KS, int64_t m, int C, double* logits,
             int first) {
  __shared__ double part[kFoldWarps][32];
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t mc = m * C;
  const int64_t t = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (t < mc) {
    // sixteen loads in flight per thread, summed in ascending k
    int64_t k = w;
    for (; k + 15 * kFoldWarps < KS; k += 16 * kFoldWarps) {
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = lpart[(k + i * kFoldWarps) * mc + t];
#pragma unroll
      for (int i = 0; i < 16; ++i) s += (double)v[i];
    }
    for (; k < KS; k += kFoldWarps) s += (double)lpart[k * mc + t];
  }
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && t < mc) {
    double r = first ? 0.0 : logits[t];
#pragma unroll
    for (int i = 0; i < kFoldWarps; ++i) r += part[i][lane];
    logits[t] = r;
  }
}

// padded float32 copy of delta: out[r][c] for r < rows (multiple of 8), c < ncp
__global__ void k_to_f32_pad(const double* a, int64_t m, int C, int ncp, int64_t rows, float* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * ncp) return;
  const int64_t r = t / ncp;
  const int c = (int)(t - r * ncp);
  out[t] = (r < m && c < C) ? (float)a[r * C + c] : 0.f;
}

__global__ void k_to_f32(const double* a, float* b, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) b[t] = (float)a[t];
}

// dwpart[rs][c][i]      = sum_{r in split} delta[r][c] cos(z[r][i])
// dwpart[rs][c][n + i]  = sum_{r in split} delta[r][c] sin(z[r][i])
template <int NC>
__global__ void __launch_bounds__(kBthreads) k_fused_bwd(const float* __restrict__ z, int64_t m,
                                                         int64_t n, int64_t ldz,
                                                         const float* __restrict__ delta,
                                                         int64_t rows_per_split,
                                                         float* __restrict__ dwpart) {
  __shared__ float sd[kBrowChunk][NC];
  const int rs = blockIdx.y;
  const int64_t rbeg = (int64_t)rs * rows_per_split;
  const int64_t rend = rbeg + rows_per_split < m ? rbeg + rows_per_split : m;
  const int64_t ib = (int64_t)blockIdx.x * kBz + threadIdx.x;
  float ac[kBzPerThread][NC], as[kBzPerThread][NC];
#pragma unroll
  for (int j = 0; j < kBzPerThread; ++j)
#pragma unroll
    for (int c = 0; c < NC; ++c) ac[j][c] = as[j][c] = 0.f;
  for (int64_t r0 = rbeg; r0 < rend; r0 += kBrowChunk) {
    const int nr = (int)(rend - r0 < kBrowChunk ? rend - r0 : kBrowChunk);
    __syncthreads();
    for (int t = threadIdx.x; t < nr * NC; t += blockDim.x) sd[t / NC][t % NC] = delta[r0 * NC + t];
    __syncthreads();
#pragma unroll 2
    for (int rr = 0; rr < nr; ++rr) {
      const float* zr = z + (r0 + rr) * ldz;
      float cs[kBzPerThread], sn[kBzPerThread];
#pragma unroll
      for (int j = 0; j < kBzPerThread; ++j) {
        const int64_t i = ib + j * kBthreads;
        const float zz = i < n ? __ldg(zr + i) : 0.f;
        __sincosf(zz, &sn[j], &cs[j]);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const float d = sd[rr][c];
#pragma unroll
        for (int j = 0; j < kBzPerThread; ++j) {
          ac[j][c] = fmaf(d, cs[j], ac[j][c]);
          as[j][c] = fmaf(d, sn[j], as[j][c]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kBzPerThread; ++j) {
    const int64_t i = ib + j * kBthreads;
    if (i < n)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        dwpart[((int64_t)rs * NC + c) * 2 * n + i] = ac[j][c];
        dwpart[((int64_t)rs * NC + c) * 2 * n + n + i] = as[j][c];
      }
  }
}

// For block e: g = sum_rs dwpart (fixed order); dw[c][col] = g, or
// w[c][col] -= lr*(g + 2*l2*w) in place.  col = e n + i (cos) / D + e n + i (sin).
__global__ void k_fused_dw_finish(const float* __restrict__ dwpart, int64_t RS, int C, int64_t n,
                                  int64_t F, int64_t col_cos, int64_t col_sin, float* dw, float* w,
                                  float lr, float l2) {
  const int64_t per = 2 * n;
  const int64_t total = (int64_t)C * per;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / per, k = t % per;
    float g = 0.f;
    for (int64_t s = 0; s < RS; ++s) g += dwpart[s * total + t];
    const int64_t col = c * F + (k < n ? col_cos + k : col_sin + (k - n));
    if (w) {
      const float wv = w[col];
      w[col] = wv - lr * (l2 != 0.f ? g + 2.f * l2 * wv : g);
    } else {
      dw[col] = g;
    }
  }
}

__global__ void k_fused_db(const double* delta, int64_t m, int C, double* db, double* b, double lr) {
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

template <class Fn>
static int dispatch_nc(int C, Fn fn) {
  switch (C) {
#define MCK_D(N) case N: return fn(std::integral_constant<int, N>{});
    MCK_D(2) MCK_D(3) MCK_D(4) MCK_D(5) MCK_D(6) MCK_D(7) MCK_D(8) MCK_D(9) MCK_D(10)
    MCK_D(11) MCK_D(12) MCK_D(13) MCK_D(14) MCK_D(15) MCK_D(16)
#undef MCK_D
    default: return fail_value("num_classes must be in 2..%d", kFusedMaxClasses);
  }
}

int64_t fused_scratch_bytes(int64_t m, int64_t n, int32_t E, int32_t C, bool keep) {
  return fused_layout(m, n, E, C, keep, nullptr, nullptr);
}

int fused_fwd_tc(const float*, int64_t, int64_t, int64_t, int64_t, const float*, int64_t, int, int64_t,
                 int64_t, float*, cudaStream_t);
int fused_bwd_tc(const float*, int64_t, int64_t, int64_t, int64_t, const float*, int, int64_t, int64_t,
                 int64_t, float*, float*, float, float, cudaStream_t);
int64_t fused_tc_ksplits(int64_t n);

int fused_forward(const TablesView& tv, int32_t d, double sigma, const float* x, int64_t m,
                  int64_t ldx, const int32_t* rows, const float* w, const double* b, int32_t C,
                  const int32_t* labels, const int32_t* label_index, int64_t m_total,
                  double* logits_out, double* probs, double* delta, double* loss_sum,
                  int64_t* hits, void* scratch, int32_t variant, cudaStream_t st) {
  const bool cuda_cores = variant & kVarCudaCores, keep = variant & kVarKeepZ, tc = variant & kVarTc;
  const bool tile8 = !cuda_cores;  // the FFMA2 and tcgen05 engines read tiled z
  if (m == 0) return MCK_OK;
  const int64_t n = tv.n, E = tv.E, D = n * E, F = 2 * D;
  FusedScratch fs;
  fused_layout(m, n, (int32_t)E, C, keep, (char*)scratch, &fs);
  // Blocks e .. e+nb-1 are contiguous in z (tile columns), in W (cos and
  // sin columns) and in the partial-logit chunks: one contraction and one
  // fold per group, over nb*n z values.
  const int64_t ldz = n * kFusedZBlocks;
  for (int32_t e = 0; e < E; e += kFusedZBlocks) {
    const int32_t nb = (int32_t)(E - e < kFusedZBlocks ? E - e : kFusedZBlocks);
    const int64_t nz = (int64_t)nb * n;
    const int64_t KS = tc ? fused_tc_ksplits(nz)
                          : cuda_cores ? (nz + kFzChunk - 1) / kFzChunk : fused_cc_ksplits(nz);
    int64_t col0 = 0;
    float* const zt = fused_ztile(fs.z, m, n, e, keep, &col0);  // col0 = 0: e is a group start
    float* const zg = zt + col0;
    MCK_TRY(fastfood_z_blocks(tv, d, sigma, x, m, ldx, rows, e, nb, zg, ldz, tile8, st));
    if (tc)
      MCK_TRY(fused_fwd_tc(zt, m, nz, ldz, col0, w, F, C, (int64_t)e * n, D + (int64_t)e * n, fs.lpart, st));
    else if (!cuda_cores)
      MCK_TRY(fused_fwd_cc(zt, m, nz, ldz, col0, w, F, C, (int64_t)e * n, D + (int64_t)e * n, fs.wt,
                           fs.lpart, st));
    else MCK_TRY(dispatch_nc(C, [&](auto nc) {
      constexpr int NC = decltype(nc)::value;
      dim3 grid((unsigned)((m + kFrows - 1) / kFrows), (unsigned)KS);
      k_fused_fwd<NC><<<grid, kFwarps * 32, 0, st>>>(zg, m, nz, ldz, w, F, (int64_t)e * n,
                                                     D + (int64_t)e * n, fs.lpart);
      return check_launch("k_fused_fwd");
    }));
    MCK_TRY(launch_pdl(k_fused_fold, dim3((unsigned)((m * C + 31) / 32)), dim3(kFoldWarps * 32), 0, st,
                       "k_fused_fold", (const float*)fs.lpart, KS, m, (int)C, fs.logits, e == 0 ? 1 : 0));
  }
  if (logits_out)
    MCK_TRY(check_cuda(cudaMemcpyAsync(logits_out, fs.logits, m * C * 8, cudaMemcpyDeviceToDevice, st),
                       "logits copy"));
  return head_softmax_from_logits(fs.logits, m, C, b, labels, label_index, m_total, probs,
                                  delta ? delta : fs.delta64, loss_sum, hits, fs.rowloss,
                                  fs.rowhit, st);
}

// Backward of blocks [e_begin, e_begin + e_count) only.  dW of those blocks
// goes to dw with row stride ldw; block e_begin + k's cos columns start at
// cos0 + k n and its sin columns at sin0 + k n.  The plain layout is
// (ldw, cos0, sin0) = (F, e_begin n, D + e_begin n); an all-reduce bucket
// uses (2 e_count n, 0, e_count n), i.e. [C][cos | sin] of the range,
// contiguous.  With w != NULL the update is applied in place instead
// (plain layout only).
int fused_backward_range(const TablesView& tv, int32_t d, double sigma, const float* x, int64_t m,
                         int64_t ldx, const int32_t* rows, const double* delta, int32_t C,
                         int32_t e_begin, int32_t e_count, float* dw, int64_t ldw, int64_t cos0,
                         int64_t sin0, float* w, double lr, double l2, void* scratch,
                         int32_t variant, cudaStream_t st) {
  if (m == 0) return MCK_OK;
  const bool cuda_cores = variant & kVarCudaCores, keep = variant & kVarKeepZ, tc = variant & kVarTc;
  const bool tile8 = !cuda_cores;
  const int64_t n = tv.n;
  FusedScratch fs;
  fused_layout(m, n, (int32_t)tv.E, C, keep, (char*)scratch, &fs);
  const int64_t RS = fused_rsplits(m);
  const int64_t rps = (m + RS - 1) / RS;
  k_to_f32<<<(unsigned)((m * C + 255) / 256), 256, 0, st>>>(delta, fs.delta32, m * C);
  MCK_TRY(check_launch("k_to_f32"));
  if (!tc && !cuda_cores) {
    const int ncp = (C + 1) & ~1;
    const int64_t rows8 = (m + 7) & ~int64_t(7);
    k_to_f32_pad<<<(unsigned)((rows8 * ncp + 255) / 256), 256, 0, st>>>(delta, m, C, ncp, rows8,
                                                                       fs.delta32p);
    MCK_TRY(check_launch("k_to_f32_pad"));
  }
  const int64_t ldz = n * kFusedZBlocks;
  const int32_t e_end = e_begin + e_count;
  for (int32_t e = e_begin, nb = 0; e < e_end; e += nb) {
    // chunks never cross a 16-block boundary (the forward's z groups)
    const int32_t room = kFusedZBlocks - e % kFusedZBlocks;
    nb = e_end - e < room ? e_end - e : room;
    const int64_t nz = (int64_t)nb * n;
    const int64_t cc = cos0 + (int64_t)(e - e_begin) * n, cs = sin0 + (int64_t)(e - e_begin) * n;
    // kept z: the forward's tile, read as is; otherwise recompute this group
    int64_t col0 = 0;
    float* const zt = fused_ztile(fs.z, m, n, e, keep, &col0);
    float* const zg = zt + col0;  // row-major engines
    if (!keep) MCK_TRY(fastfood_z_blocks(tv, d, sigma, x, m, ldx, rows, e, nb, zt, ldz, tile8, st));
    if (tc) {
      MCK_TRY(fused_bwd_tc(zt, m, nz, ldz, col0, fs.delta32, C, ldw, cc, cs, dw, w, (float)lr, (float)l2,
                           st));
      continue;
    }
    if (!cuda_cores) {
      MCK_TRY(fused_bwd_cc(zt, m, nz, ldz, col0, fs.delta32p, C, ldw, cc, cs, dw, w, (float)lr, (float)l2,
                           st));
      continue;
    }
    MCK_TRY(dispatch_nc(C, [&](auto nc) {
      constexpr int NC = decltype(nc)::value;
      dim3 grid((unsigned)((nz + kBz - 1) / kBz), (unsigned)RS);
      k_fused_bwd<NC><<<grid, kBthreads, 0, st>>>(zg, m, nz, ldz, fs.delta32, rps, fs.dwpart);
      return check_launch("k_fused_bwd");
    }));
    int64_t grid = ((int64_t)C * 2 * nz + 255) / 256;
    if (grid > 148 * 8) grid = 148 * 8;
    k_fused_dw_finish<<<(unsigned)grid, 256, 0, st>>>(fs.dwpart, RS, C, nz, ldw, cc, cs, dw, w,
                                                      (float)lr, (float)l2);
    MCK_TRY(check_launch("k_fused_dw_finish"));
  }
  return MCK_OK;
}

int fused_backward(const TablesView& tv, int32_t d, double sigma, const float* x, int64_t m,
                   int64_t ldx, const int32_t* rows, const double* delta, int32_t C, float* dw,
                   double* db, float* w, double* b, double lr, double l2, void* scratch,
                   int32_t variant, cudaStream_t st) {
  if (m == 0) return MCK_OK;
  const int64_t n = tv.n, D = n * tv.E, F = 2 * D;
  MCK_TRY(fused_backward_range(tv, d, sigma, x, m, ldx, rows, delta, C, 0, (int32_t)tv.E, dw, F, 0, D,
                               w, lr, l2, scratch, variant, st));
  k_fused_db<<<C, 256, 0, st>>>(delta, m, C, db, b, lr);
  return check_launch("k_fused_db");
}

int fused_bias_grad(const double* delta, int64_t m, int32_t C, double* db, cudaStream_t st) {
  k_fused_db<<<C, 256, 0, st>>>(delta, m, C, db, nullptr, 0.0);
  return check_launch("k_fused_db");
}

// W[c][block columns] -= lr * (g + 2 l2 W) for the bucket of blocks
// [e_begin, e_begin + e_count) (layout of fused_backward_range's bucket), and
// b -= lr * db when b is given.  Same float32 arithmetic as the fused update
// of the single-rank backward (k_fused_bwd_tc / k_fused_dw_finish).
__global__ void k_fused_apply_bucket(float* __restrict__ w, int64_t F, int64_t D, int64_t n,
                                     int32_t e_begin, int64_t nz, int C,
                                     const float* __restrict__ bucket, float lr, float l2,
                                     double* __restrict__ b, const double* __restrict__ db,
                                     double lr64) {
  const int64_t total = (int64_t)C * 2 * nz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / (2 * nz), k = i - c * 2 * nz;
    const int64_t col = c * F + (k < nz ? (int64_t)e_begin * n + k : D + (int64_t)e_begin * n + (k - nz));
    const float g = bucket[i];
    const float wv = w[col];
    w[col] = wv - lr * (l2 != 0.f ? g + 2.f * l2 * wv : g);
  }
  if (b && blockIdx.x == 0 && threadIdx.x < C) b[threadIdx.x] -= lr64 * db[threadIdx.x];
}

int fused_apply_bucket(float* w, int64_t n, int32_t E, int32_t C, int32_t e_begin, int32_t e_count,
                       const float* bucket, double lr, double l2, double* b, const double* db,
                       cudaStream_t st) {
  const int64_t D = n * E, nz = (int64_t)e_count * n;
  int64_t grid = ((int64_t)C * 2 * nz + 255) / 256;
  if (grid > 148 * 8) grid = 148 * 8;
  if (grid < 1) grid = 1;
  k_fused_apply_bucket<<<(unsigned)grid, 256, 0, st>>>(w, 2 * D, D, n, e_begin, nz, C, bucket,
                                                       (float)lr, (float)l2, b, db, lr);
  return check_launch("k_fused_apply_bucket");
}

}  // namespace mck
