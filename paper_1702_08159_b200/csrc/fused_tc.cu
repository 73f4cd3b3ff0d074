// K6 tensor-core contractions for the fused config-4 classifier (tcgen05,
// kind::tf32, 3xTF32 split so the result carries ~fp32 accuracy):
//
//   forward : partial logits (128 rows x 16 classes, TMEM) +=
//             [cos z | sin z] (128 rows x 2*256 features, produced on chip
//             from the L2-resident z tile) * W slice^T
//   backward: dW tile (128 features = 64 z x {cos, sin}, 16 classes, TMEM) +=
//             [cos z ; sin z]^T (features x rows) * delta (rows x classes)
//
// Features exist only in shared memory.  Producer warps compute sin/cos, split
// each value x into tf32 hi = x & ~0x1fff and lo = x - hi, and store both in the
// interleaved K-major layout (umma.cuh); one thread issues A_hi*B_hi +
// A_hi*B_lo + A_lo*B_hi per K step and commits to an mbarrier that releases
// the double-buffered stage.  Accumulation is fp32 in TMEM.
#include "mck_common.cuh"
#include "umma.cuh"

namespace mck {

constexpr int kTcM = 128;
constexpr int kTcN = 16;            // classes padded to the MMA's N
constexpr int kTcThreads = 256;
constexpr int kFzCta = 128;         // forward: z values (K = 2 * 128 features) per CTA
constexpr int kFzStage = 16;        // forward: z values per pipeline stage
constexpr int kBzCta = 64;          // backward: z values per CTA (M = 128 features)
constexpr int kBrowStage = 32;      // backward: rows (K) per pipeline stage

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

__device__ __forceinline__ void sts128(void* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}

// ---------------------------------------------------------------- forward
struct FwdSmem {
  // B: W slice, rows = 16 classes, K = kFzCta, interleaved; [cos_hi, cos_lo, sin_hi, sin_lo]
  float b[4][kTcN * kFzCta];
  // A stages: rows = 128, K = kFzStage; [stage][cos_hi, cos_lo, sin_hi, sin_lo]
  float a[2][4][kTcM * kFzStage];
  uint64_t bar[2];
  uint32_t tslot;
};

__global__ void __launch_bounds__(kTcThreads, 2)
k_fused_fwd_tc(const float* __restrict__ z, int64_t m, int64_t n, const float* __restrict__ w,
               int64_t F, int C, int64_t col_cos, int64_t col_sin, float* __restrict__ lpart) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  FwdSmem& S = *reinterpret_cast<FwdSmem*>(smraw);
  const int t = threadIdx.x, warp = t >> 5;
  const int ks = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * kTcM;
  const int64_t z0 = (int64_t)ks * kFzCta;
  const int nz = (int)(n - z0 < kFzCta ? n - z0 : kFzCta);

  const int row = t & (kTcM - 1), half = t >> 7;  // 2 threads per row, 8 z each per stage
  const int64_t gr = r0 + row < m ? r0 + row : m - 1;
  const float* zr = z + gr * n + z0;
  // z prefetch ring: stage s+P is requested while stage s is consumed (the z
  // tile comes from L2/HBM; a 4-deep ring hides its latency)
  constexpr int SF = kFzCta / kFzStage, P = 4;
  float4 ring[P][2];
  auto load_stage = [&](int st, float4 (&dst)[2]) {
    const int zi = st * kFzStage + half * 8;
    if (zi + 8 <= nz) {
      dst[0] = __ldcs(reinterpret_cast<const float4*>(zr + zi));
      dst[1] = __ldcs(reinterpret_cast<const float4*>(zr + zi + 4));
    } else {
      float tmp[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) tmp[j] = zi + j < nz ? __ldcs(zr + zi + j) : 0.f;
      dst[0] = make_float4(tmp[0], tmp[1], tmp[2], tmp[3]);
      dst[1] = make_float4(tmp[4], tmp[5], tmp[6], tmp[7]);
    }
  };
#pragma unroll
  for (int p = 0; p < P; ++p) load_stage(p, ring[p]);

  // W slice -> B tiles (hi/lo), zero for padded classes / z beyond n
  for (int idx = t; idx < kTcN * kFzCta; idx += kTcThreads) {
    const int c = idx / kFzCta, k = idx % kFzCta;
    float wc = 0.f, wsn = 0.f;
    if (c < C && k < nz) {
      wc = w[(int64_t)c * F + col_cos + z0 + k];
      wsn = w[(int64_t)c * F + col_sin + z0 + k];
    }
    const uint32_t off = umma::tile_off(c, k, kTcN) / 4;
    split_tf32(wc, S.b[0][off], S.b[1][off]);
    split_tf32(wsn, S.b[2][off], S.b[3][off]);
  }
  if (t == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc<32>(&S.tslot);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = S.tslot;
  constexpr uint32_t idesc = umma::idesc_tf32(kTcM, kTcN);

  // stages beyond nz multiply zero W columns: always run all SF stages
#pragma unroll
  for (int s = 0; s < SF; ++s) {
    const int buf = s & 1;
    float zv[8] = {ring[s % P][0].x, ring[s % P][0].y, ring[s % P][0].z, ring[s % P][0].w,
                   ring[s % P][1].x, ring[s % P][1].y, ring[s % P][1].z, ring[s % P][1].w};
    if (s + P < SF) load_stage(s + P, ring[s % P]);
    if (s >= 2) mbar_wait(&S.bar[buf], (uint32_t)(((s - 2) >> 1) & 1));
    const int kb = half * 8;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float c[4], sn[4], ch[4], cl[4], sh[4], sl[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __sincosf(zv[4 * q + j], &sn[j], &c[j]);
        split_tf32(c[j], ch[j], cl[j]);
        split_tf32(sn[j], sh[j], sl[j]);
      }
      const uint32_t off = umma::tile_off(row, kb + 4 * q, kTcM);
      unsigned char* base = reinterpret_cast<unsigned char*>(S.a[buf][0]);
      constexpr uint32_t AS = kTcM * kFzStage * 4;
      sts128(base + 0 * AS + off, ch[0], ch[1], ch[2], ch[3]);
      sts128(base + 1 * AS + off, cl[0], cl[1], cl[2], cl[3]);
      sts128(base + 2 * AS + off, sh[0], sh[1], sh[2], sh[3]);
      sts128(base + 3 * AS + off, sl[0], sl[1], sl[2], sl[3]);
    }
    umma::fence_smem_to_async();
    __syncthreads();
    if (t == 0) {
      umma::fence_after();
#pragma unroll
      for (int part = 0; part < 2; ++part) {         // cos, sin
#pragma unroll
        for (int k0 = 0; k0 < kFzStage; k0 += 8) {
          const unsigned char* ab = reinterpret_cast<const unsigned char*>(S.a[buf][2 * part]);
          const unsigned char* al = reinterpret_cast<const unsigned char*>(S.a[buf][2 * part + 1]);
          const unsigned char* bb = reinterpret_cast<const unsigned char*>(S.b[2 * part]);
          const unsigned char* bl = reinterpret_cast<const unsigned char*>(S.b[2 * part + 1]);
          const uint32_t aoff = (k0 / 4) * kTcM * 16;
          const uint32_t boff = ((s * kFzStage + k0) / 4) * kTcN * 16;
          const uint64_t dah = umma::smem_desc(ab + aoff, kTcM * 16, 128);
          const uint64_t dal = umma::smem_desc(al + aoff, kTcM * 16, 128);
          const uint64_t dbh = umma::smem_desc(bb + boff, kTcN * 16, 128);
          const uint64_t dbl = umma::smem_desc(bl + boff, kTcN * 16, 128);
          const uint32_t acc0 = (s > 0 || part > 0 || k0 > 0) ? 1u : 0u;
          umma::mma_tf32(tm, dah, dbh, idesc, acc0);
          umma::mma_tf32(tm, dah, dbl, idesc, 1u);
          umma::mma_tf32(tm, dal, dbh, idesc, 1u);
        }
      }
      umma::commit(&S.bar[buf]);
    }
  }
  const int stages = SF;
  // all MMAs done: the last commit covers every earlier MMA of thread 0
  if (stages > 0) mbar_wait(&S.bar[(stages - 1) & 1], (uint32_t)(((stages - 1) >> 1) & 1));
  umma::fence_after();
  if (warp < 4) {
    float v[16];
    umma::tmem_ld16(tm + ((uint32_t)(32 * warp) << 16), v);
    const int64_t r = r0 + 32 * warp + (t & 31);
    if (r < m)
      for (int c = 0; c < C; ++c) lpart[((int64_t)ks * m + r) * C + c] = stages > 0 ? v[c] : 0.f;
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<32>(tm);
}

// ---------------------------------------------------------------- backward
struct BwdSmem {
  // A stages: rows = 128 features (64 cos, 64 sin), K = 32 rows; [stage][hi, lo]
  float a[2][2][kTcM * kBrowStage];
  // B stages: rows = 16 classes, K = 32 rows; [stage][hi, lo]
  float b[2][2][kTcN * kBrowStage];
  uint64_t bar[2];
  uint32_t tslot;
};

__global__ void __launch_bounds__(kTcThreads, 3)
k_fused_bwd_tc(const float* __restrict__ z, int64_t m, int64_t n, const float* __restrict__ delta,
               int C, int64_t F, int64_t col_cos, int64_t col_sin, float* dw, float* w, float lr,
               float l2) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  BwdSmem& S = *reinterpret_cast<BwdSmem*>(smraw);
  const int t = threadIdx.x, warp = t >> 5;
  const int64_t z0 = (int64_t)blockIdx.x * kBzCta;
  if (t == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc<32>(&S.tslot);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = S.tslot;
  constexpr uint32_t idesc = umma::idesc_tf32(kTcM, kTcN);
  constexpr uint32_t AS = kTcM * kBrowStage * 4, BS = kTcN * kBrowStage * 4;

  const int zi = t & 63, q0 = t >> 6;  // A items: (z, row quad q0) and (z, q0 + 4)
  const bool zok = z0 + zi < n;
  const int stages = (int)((m + kBrowStage - 1) / kBrowStage);
  // z prefetch ring (4 stages deep) hides the L2/HBM latency of the z tile
  constexpr int P = 4;
  float ring[P][8];
  auto load_stage = [&](int st, float (&dst)[8]) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t r = (int64_t)st * kBrowStage + 4 * (q0 + 4 * h) + j;
        dst[4 * h + j] = (zok && r < m) ? __ldcs(z + r * n + z0 + zi) : 0.f;
      }
  };
#pragma unroll
  for (int p = 0; p < P; ++p)
    if (p < stages) load_stage(p, ring[p]);
  for (int s0 = 0; s0 < stages; s0 += P)
#pragma unroll
  for (int u = 0; u < P; ++u) {
    const int s = s0 + u;
    if (s >= stages) break;
    float zv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) zv[j] = ring[u][j];
    if (s + P < stages) load_stage(s + P, ring[u]);
    const int buf = s & 1;
    if (s >= 2) mbar_wait(&S.bar[buf], (uint32_t)(((s - 2) >> 1) & 1));
    const int64_t rb = (int64_t)s * kBrowStage;
    unsigned char* A = reinterpret_cast<unsigned char*>(S.a[buf][0]);
    unsigned char* B = reinterpret_cast<unsigned char*>(S.b[buf][0]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = q0 + 4 * h;
      float cs[4], sn[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) __sincosf(zv[4 * h + j], &sn[j], &cs[j]);
      float ch[4], cl[4], sh[4], sl[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        split_tf32(cs[j], ch[j], cl[j]);
        split_tf32(sn[j], sh[j], sl[j]);
      }
      const uint32_t oc = umma::tile_off(zi, 4 * q, kTcM), os = umma::tile_off(64 + zi, 4 * q, kTcM);
      sts128(A + oc, ch[0], ch[1], ch[2], ch[3]);
      sts128(A + AS + oc, cl[0], cl[1], cl[2], cl[3]);
      sts128(A + os, sh[0], sh[1], sh[2], sh[3]);
      sts128(A + AS + os, sl[0], sl[1], sl[2], sl[3]);
    }
    if (t < kTcN * (kBrowStage / 4)) {           // B = delta^T: (class c, row quad q)
      const int c = t % kTcN, q = t / kTcN;
      float d[4], dh[4], dl[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t r = rb + 4 * q + j;
        d[j] = (c < C && r < m) ? delta[r * C + c] : 0.f;
        split_tf32(d[j], dh[j], dl[j]);
      }
      const uint32_t ob = umma::tile_off(c, 4 * q, kTcN);
      sts128(B + ob, dh[0], dh[1], dh[2], dh[3]);
      sts128(B + BS + ob, dl[0], dl[1], dl[2], dl[3]);
    }
    umma::fence_smem_to_async();
    __syncthreads();
    if (t == 0) {
      umma::fence_after();
#pragma unroll
      for (int k0 = 0; k0 < kBrowStage; k0 += 8) {
        const uint32_t aoff = (k0 / 4) * kTcM * 16, boff = (k0 / 4) * kTcN * 16;
        const uint64_t dah = umma::smem_desc(A + aoff, kTcM * 16, 128);
        const uint64_t dal = umma::smem_desc(A + AS + aoff, kTcM * 16, 128);
        const uint64_t dbh = umma::smem_desc(B + boff, kTcN * 16, 128);
        const uint64_t dbl = umma::smem_desc(B + BS + boff, kTcN * 16, 128);
        umma::mma_tf32(tm, dah, dbh, idesc, (s > 0 || k0 > 0) ? 1u : 0u);
        umma::mma_tf32(tm, dah, dbl, idesc, 1u);
        umma::mma_tf32(tm, dal, dbh, idesc, 1u);
      }
      umma::commit(&S.bar[buf]);
    }
  }
  if (stages > 0) mbar_wait(&S.bar[(stages - 1) & 1], (uint32_t)(((stages - 1) >> 1) & 1));
  umma::fence_after();
  if (warp < 4) {
    float v[16];
    umma::tmem_ld16(tm + ((uint32_t)(32 * warp) << 16), v);
    const int f = 32 * warp + (t & 31);   // feature row of the tile
    const int zz = f & 63;
    if (z0 + zz < n) {
      const int64_t col = (f < 64 ? col_cos : col_sin) + z0 + zz;
      for (int c = 0; c < C; ++c) {
        const float g = stages > 0 ? v[c] : 0.f;
        if (w) {
          const float wv = w[(int64_t)c * F + col];
          w[(int64_t)c * F + col] = wv - lr * (l2 != 0.f ? g + 2.f * l2 * wv : g);
        } else {
          dw[(int64_t)c * F + col] = g;
        }
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<32>(tm);
}

int fused_fwd_tc(const float* z, int64_t m, int64_t n, const float* w, int64_t F, int C,
                 int64_t col_cos, int64_t col_sin, float* lpart, cudaStream_t st) {
  if (C > kTcN) return fail_value("num_classes must be <= %d", kTcN);
  const size_t smem = sizeof(FwdSmem);
  static bool init = false;
  if (!init) {
    MCK_TRY(check_cuda(cudaFuncSetAttribute(k_fused_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem), "fwd tc smem"));
    init = true;
  }
  dim3 grid((unsigned)((m + kTcM - 1) / kTcM), (unsigned)((n + kFzCta - 1) / kFzCta));
  k_fused_fwd_tc<<<grid, kTcThreads, smem, st>>>(z, m, n, w, F, C, col_cos, col_sin, lpart);
  return check_launch("k_fused_fwd_tc");
}

int fused_bwd_tc(const float* z, int64_t m, int64_t n, const float* delta, int C, int64_t F,
                 int64_t col_cos, int64_t col_sin, float* dw, float* w, float lr, float l2,
                 cudaStream_t st) {
  if (C > kTcN) return fail_value("num_classes must be <= %d", kTcN);
  const size_t smem = sizeof(BwdSmem);
  static bool init = false;
  if (!init) {
    MCK_TRY(check_cuda(cudaFuncSetAttribute(k_fused_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem), "bwd tc smem"));
    init = true;
  }
  const unsigned grid = (unsigned)((n + kBzCta - 1) / kBzCta);
  k_fused_bwd_tc<<<grid, kTcThreads, smem, st>>>(z, m, n, delta, C, F, col_cos, col_sin, dw, w,
                                                 lr, l2);
  return check_launch("k_fused_bwd_tc");
}

int64_t fused_tc_ksplits(int64_t n) { return (n + kFzCta - 1) / kFzCta; }

}  // namespace mck
