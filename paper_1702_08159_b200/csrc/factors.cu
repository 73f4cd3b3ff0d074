// K2 -- on-device factor generation (replaces fastfood.py:96-166 and the
// detrand.py streams it draws from), plus the stream-level kernels exported
// through the C ABI.
//
// Bit-exactness: B signs and the Fisher-Yates permutation are integer /
// IEEE-multiply derived and reproduce the reference exactly.  G and C are
// float64 Box-Muller / norms with numpy's pairwise summation order restated
// (mck_common.cuh); CUDA's libdevice log/sin/cos/pow may differ from numpy's
// by an ulp in float64, which the cast to float32 almost always absorbs --
// the GPU tests count mismatches against the reference's own values.
#include "mck_common.cuh"
#include "tables.cuh"

namespace mck {

__device__ __forceinline__ uint64_t block_key(uint64_t seed, uint64_t label_hash, uint64_t block) {
  uint64_t k = fmix64(seed);
  k = fmix64(k ^ label_hash);
  return fmix64(k ^ (block * kGamma));
}

// ---------------------------------------------------------------- streams
__global__ void k_hashes(uint64_t key, uint64_t c0, int64_t count, uint64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = draw(key, c0 + i);
}
__global__ void k_uniforms(uint64_t key, uint64_t c0, int64_t count, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = uniform01(key, c0 + i);
}
__global__ void k_signs(uint64_t key, uint64_t c0, int64_t count, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (draw(key, c0 + i) >> 63) ? 1.0 : -1.0;
}
__global__ void k_gauss_pairs(uint64_t key, uint64_t c0, int64_t pairs, double* out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < pairs;
       p += (int64_t)gridDim.x * blockDim.x) {
    double z0, z1;
    gauss_pair(key, c0 + 2 * p, z0, z1);
    out[2 * p] = z0;
    out[2 * p + 1] = z1;
  }
}

static unsigned grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return (unsigned)g;
}

int stream_hashes(uint64_t key, uint64_t c0, int64_t count, uint64_t* out, cudaStream_t st) {
  if (count <= 0) return MCK_OK;
  k_hashes<<<grid_for(count), 256, 0, st>>>(key, c0, count, out);
  return check_launch("k_hashes");
}
int stream_uniforms(uint64_t key, uint64_t c0, int64_t count, double* out, cudaStream_t st) {
  if (count <= 0) return MCK_OK;
  k_uniforms<<<grid_for(count), 256, 0, st>>>(key, c0, count, out);
  return check_launch("k_uniforms");
}
int stream_signs(uint64_t key, uint64_t c0, int64_t count, double* out, cudaStream_t st) {
  if (count <= 0) return MCK_OK;
  k_signs<<<grid_for(count), 256, 0, st>>>(key, c0, count, out);
  return check_launch("k_signs");
}
int stream_gaussian_pairs(uint64_t key, uint64_t c0, int64_t pairs, double* out, cudaStream_t st) {
  if (pairs <= 0) return MCK_OK;
  k_gauss_pairs<<<grid_for(pairs), 256, 0, st>>>(key, c0, pairs, out);
  return check_launch("k_gauss_pairs");
}

// ---------------------------------------------------------------- Fisher-Yates
// detrand.py:186-203.  One CTA per permutation; the swap chain is serial
// (thread 0) over a shared-memory array; the uniforms are recomputed inline
// (counter k for step i = n-1-k).
template <class IDX>
__global__ void k_fisher_yates(uint64_t seed, uint64_t label_hash, uint64_t block0, int64_t n,
                               int32_t* out) {
  extern __shared__ __align__(16) unsigned char fy_smem[];
  IDX* p = reinterpret_cast<IDX*>(fy_smem);
  const uint64_t key = block_key(seed, label_hash, block0 + blockIdx.x);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) p[i] = (IDX)i;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t k = 0; k < n - 1; ++k) {
      const int64_t i = n - 1 - k;
      const double u = uniform01(key, (uint64_t)k);
      int64_t j = (int64_t)(u * (double)(i + 1));
      if (j > i) j = i;
      const IDX a = p[i];
      p[i] = p[j];
      p[j] = a;
    }
  }
  __syncthreads();
  int32_t* o = out + (int64_t)blockIdx.x * n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) o[i] = (int32_t)p[i];
}

// large n: in place in global memory
__global__ void k_fisher_yates_global(uint64_t seed, uint64_t label_hash, uint64_t block0,
                                      int64_t n, int32_t* out) {
  int32_t* p = out + (int64_t)blockIdx.x * n;
  const uint64_t key = block_key(seed, label_hash, block0 + blockIdx.x);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) p[i] = (int32_t)i;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t k = 0; k < n - 1; ++k) {
      const int64_t i = n - 1 - k;
      const double u = uniform01(key, (uint64_t)k);
      int64_t j = (int64_t)(u * (double)(i + 1));
      if (j > i) j = i;
      const int32_t a = p[i];
      p[i] = p[j];
      p[j] = a;
    }
  }
}

int fisher_yates(uint64_t seed, uint64_t label_hash, uint64_t block0, int32_t count, int64_t n,
                 int32_t* out, cudaStream_t st) {
  if (count <= 0) return MCK_OK;
  if (n <= 65536) {
    const size_t smem = (size_t)n * 2;
    auto kern = k_fisher_yates<uint16_t>;
    if (smem > 48 * 1024)
      MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem), "fy smem"));
    kern<<<count, 256, smem, st>>>(seed, label_hash, block0, n, out);
  } else {
    k_fisher_yates_global<<<count, 256, 0, st>>>(seed, label_hash, block0, n, out);
  }
  return check_launch("k_fisher_yates");
}

// ---------------------------------------------------------------- B, G
__global__ void k_block_signs(uint64_t seed, uint64_t lh, int64_t n, int32_t E, float* b) {
  const int64_t total = n * E;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / n, i = t % n;
    const uint64_t key = block_key(seed, lh, (uint64_t)e);
    b[t] = (draw(key, (uint64_t)i) >> 63) ? 1.0f : -1.0f;
  }
}

// G: gaussians(n) from a fresh stream (pairs 0..ceil(n/2)-1), float64 kept
// for |g|, float32 cast for the table; then |g| = sqrt(pairwise sum g^2)
// (fastfood.py:103 / :152).  One CTA per block.
__global__ void k_block_gauss(uint64_t seed, uint64_t lh, int64_t n, float* g, double* g64,
                              double* gnorm) {
  const int e = blockIdx.x;
  const uint64_t key = block_key(seed, lh, (uint64_t)e);
  double* G = g64 + (int64_t)e * n;
  for (int64_t p = threadIdx.x; 2 * p < n; p += blockDim.x) {
    double z0, z1;
    gauss_pair(key, 2 * (uint64_t)p, z0, z1);
    G[2 * p] = z0;
    g[(int64_t)e * n + 2 * p] = (float)z0;
    if (2 * p + 1 < n) {
      G[2 * p + 1] = z1;
      g[(int64_t)e * n + 2 * p + 1] = (float)z1;
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double s;
    if (n >= 1024) {
      s = pairwise_warp_pow2(
          [&](int64_t p, double& a, double& b) {
            a = G[2 * p] * G[2 * p];
            b = G[2 * p + 1] * G[2 * p + 1];
          },
          n, threadIdx.x);
    } else {
      s = pairwise_serial([&](int64_t i) { return G[i] * G[i]; }, 0, n);
    }
    if (threadIdx.x == 0) gnorm[e] = sqrt(s);
  }
}

// ---------------------------------------------------------------- C (RBF)
// fastfood.py:96-107: entry i = |gaussians[i*n : (i+1)*n]| of stream "C",
// divided by |g|.  One warp per entry.
__global__ void k_c_rbf(uint64_t seed, uint64_t lh, int64_t n, int32_t E, const double* gnorm,
                        float* c) {
  const int lane = threadIdx.x & 31;
  const int64_t entry = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (entry >= n * E) return;
  const int64_t e = entry / n, i = entry % n;
  const uint64_t key = block_key(seed, lh, (uint64_t)e);
  double s;
  if (n >= 1024) {
    const uint64_t pbase = (uint64_t)i * (uint64_t)n / 2;  // n even
    s = pairwise_warp_pow2(
        [&](int64_t p, double& a, double& b) {
          double z0, z1;
          gauss_pair(key, 2 * (pbase + (uint64_t)p), z0, z1);
          a = z0 * z0;
          b = z1 * z1;
        },
        n, lane);
  } else {
    if (lane != 0) return;
    s = pairwise_serial(
        [&](int64_t j) {
          const uint64_t gi = (uint64_t)i * (uint64_t)n + (uint64_t)j;
          double z0, z1;
          gauss_pair(key, 2 * (gi >> 1), z0, z1);
          const double z = (gi & 1) ? z1 : z0;
          return z * z;
        },
        0, n);
  }
  if (lane == 0) c[entry] = (float)(sqrt(s) / gnorm[e]);
}

// ---------------------------------------------------------------- C (Matern)
// fastfood.py:110-130 + detrand.py:216-254 (even-n fast path): entry i,
// sample s uses uniforms at counters (i*t+s)*(n+1) + [0, n] -- n gaussians
// then U.  point = x * (U^(1/n) / |x|); sums over s in order; c = |sum|/|g|.
// One CTA per entry; thread owns VPT consecutive coordinates.
template <int VPT>
__global__ void k_c_matern(uint64_t seed, uint64_t lh, int64_t n, int32_t t, const double* gnorm,
                           float* c) {
  extern __shared__ __align__(16) double msq[];  // n squares
  __shared__ double red;
  const int64_t e = blockIdx.y, i = blockIdx.x;
  const uint64_t key = block_key(seed, lh, (uint64_t)e);
  const int64_t c0 = (int64_t)threadIdx.x * VPT;
  double acc[VPT];
  const double inv_n = 1.0 / (double)n;
  for (int s = 0; s < t; ++s) {
    const uint64_t base = ((uint64_t)i * (uint64_t)t + (uint64_t)s) * (uint64_t)(n + 1);
    double x[VPT];
#pragma unroll
    for (int q = 0; q < VPT; q += 2) {
      gauss_pair(key, base + (uint64_t)(c0 + q), x[q], x[q + 1]);
      msq[c0 + q] = x[q] * x[q];
      msq[c0 + q + 1] = x[q + 1] * x[q + 1];
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      double sq;
      if (n >= 1024)
        sq = pairwise_warp_pow2(
            [&](int64_t p, double& a, double& b) {
              a = msq[2 * p];
              b = msq[2 * p + 1];
            },
            n, threadIdx.x);
      else
        sq = pairwise_serial([&](int64_t j) { return msq[j]; }, 0, n);
      if (threadIdx.x == 0) red = sq;
    }
    __syncthreads();
    const double U = uniform01(key, base + (uint64_t)n);
    const double scale = (1.0 * pow(U, inv_n)) / sqrt(red);
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const double pt = x[q] * scale;
      acc[q] = (s == 0) ? pt : acc[q] + pt;
    }
    __syncthreads();  // msq / red reused next sample
  }
#pragma unroll
  for (int q = 0; q < VPT; ++q) msq[c0 + q] = acc[q] * acc[q];
  __syncthreads();
  if (threadIdx.x < 32) {
    double sq;
    if (n >= 1024)
      sq = pairwise_warp_pow2(
          [&](int64_t p, double& a, double& b) {
            a = msq[2 * p];
            b = msq[2 * p + 1];
          },
          n, threadIdx.x);
    else
      sq = pairwise_serial([&](int64_t j) { return msq[j]; }, 0, n);
    if (threadIdx.x == 0) c[e * n + i] = (float)(sqrt(sq) / gnorm[e]);
  }
}

// n == 1 (odd n: the reference's per-sample slow path with the cached
// second Box-Muller variate, detrand.py:242-246).
__global__ void k_c_matern_n1(uint64_t seed, uint64_t lh, int32_t E, int32_t t,
                              const double* gnorm, float* c) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const uint64_t key = block_key(seed, lh, (uint64_t)e);
  uint64_t ctr = 0;
  bool has_pending = false;
  double pending = 0.0, acc = 0.0;
  for (int s = 0; s < t; ++s) {
    double gval;
    if (has_pending) {
      gval = pending;
      has_pending = false;
    } else {
      double z0, z1;
      gauss_pair(key, ctr, z0, z1);
      ctr += 2;
      gval = z0;
      pending = z1;
      has_pending = true;
    }
    const double U = uniform01(key, ctr++);
    const double nrm = sqrt(gval * gval);
    const double pt = gval * ((1.0 * pow(U, 1.0)) / nrm);
    acc = (s == 0) ? pt : acc + pt;
  }
  c[e] = (float)(sqrt(acc * acc) / gnorm[e]);
}

int build_factors(const TablesView& tv, uint64_t seed, int32_t kind, int32_t t, cudaStream_t st) {
  const int64_t n = tv.n;
  const int32_t E = tv.E;
  const uint64_t hB = fnv1a64("B"), hPi = fnv1a64("Pi"), hG = fnv1a64("G"), hC = fnv1a64("C");
  k_block_signs<<<grid_for(n * E), 256, 0, st>>>(seed, hB, n, E, tv.b);
  MCK_TRY(check_launch("k_block_signs"));
  MCK_TRY(fisher_yates(seed, hPi, 0, E, n, tv.perm, st));
  k_block_gauss<<<E, 256, 0, st>>>(seed, hG, n, tv.g, tv.g64, tv.gnorm);
  MCK_TRY(check_launch("k_block_gauss"));
  if (kind == MCK_KERNEL_RBF) {
    const int64_t entries = n * E;
    const int warps = 8;
    k_c_rbf<<<(unsigned)((entries + warps - 1) / warps), 32 * warps, 0, st>>>(seed, hC, n, E,
                                                                              tv.gnorm, tv.c);
    MCK_TRY(check_launch("k_c_rbf"));
  } else {
    if (n == 1) {
      k_c_matern_n1<<<(E + 127) / 128, 128, 0, st>>>(seed, hC, E, t, tv.gnorm, tv.c);
      return check_launch("k_c_matern_n1");
    }
    const int64_t threads = n / 2 < 1024 ? n / 2 : 1024;
    const int vpt = (int)(n / threads);
    const size_t smem = (size_t)n * 8;
    dim3 grid((unsigned)n, (unsigned)E);
#define MCK_MAT(V)                                                                            \
  case V: {                                                                                   \
    auto kern = k_c_matern<V>;                                                                \
    if (smem > 48 * 1024)                                                                     \
      MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                              (int)smem), "matern smem"));                   \
    kern<<<grid, (unsigned)threads, smem, st>>>(seed, hC, n, t, tv.gnorm, tv.c);               \
    break;                                                                                    \
  }
    switch (vpt) {
      MCK_MAT(2) MCK_MAT(4) MCK_MAT(8) MCK_MAT(16)
      default:
        return fail_value("Matern calibration supports padded_dim <= 16384 (its cost grows as "
                          "t * n^2 gaussians per block; the reference needs ~12 CPU-minutes per "
                          "block at 16384)");
    }
#undef MCK_MAT
    MCK_TRY(check_launch("k_c_matern"));
  }
  return MCK_OK;
}

}  // namespace mck
