// K6 tensor-core contractions for the fused config-4 classifier (tcgen05,
// kind::tf32, 3xTF32 split so the result carries ~fp32 accuracy):
//
//   forward : partial logits (128 rows x 16 classes per row tile, TMEM) +=
//             [cos z | sin z] (128 rows x 2*128 features, produced on chip
//             from the L2-resident z tile) * W slice^T
//   backward: dW tile (128 features = 64 z x {cos, sin}, 16 classes, TMEM) +=
//             [cos z ; sin z]^T (features x rows) * delta (rows x classes)
//
// Features exist only on chip.  Each CTA runs three warp roles: a loader warp
// streams z (and delta) blocks into shared rings with cp.async, completion
// signalled on mbarriers; producer warps compute sin/cos, split each value x
// into tf32 hi = x & ~0x1fff and lo = x - hi and store both in the
// interleaved K-major layout (umma.cuh); one thread issues A_hi*B_hi +
// A_hi*B_lo + A_lo*B_hi per K step and commits to the stage's "empty"
// mbarrier.  Accumulation is fp32 in TMEM.  The producers never hold
// outstanding global loads, so the proxy fence before each hand-off (a
// CTA-scope memory barrier) does not wait on memory latency.
#include "mck_common.cuh"
#include "umma.cuh"

namespace mck {

constexpr int kTcM = 128;
constexpr int kTcN = 16;            // classes padded to the MMA's N
constexpr int kFzCta = 128;         // forward: z values (K = 2 * 128 features) per CTA
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
// One CTA per (128-z chunk, group of RTG row tiles of 128 rows): the W slice
// of the chunk is split into tf32 hi/lo B tiles (shared memory) once and
// reused for every row tile; partial logits of row tile j accumulate in TMEM
// columns 16j..16j+15.  Pipeline over stages of 16 z x 128 rows:
//   8 producer warps: each thread streams its own 8 z of the stage (one row,
//     two z quads) into a private kFwdZD-deep shared ring with cp.async
//     (cp.async.wait_group, no cross-thread hand-off), computes sincos and the
//     tf32 hi/lo split, and writes the four A tiles (cos/sin x hi/lo; row =
//     TMEM lane, k = column) into the stage's TMEM buffer with tcgen05.st,
//     then arrives on full[];
//   MMA thread: wait full[], 12 MMAs with A from TMEM (3xTF32, cos and sin,
//     two K = 8 steps), commit to empty[].
// The A operand never touches shared memory.
constexpr int kFwdStageZ = 16;                      // z per stage (two K=8 MMAs per part)
constexpr int kFwdBuf = 3;                          // A buffers (TMEM)
constexpr int kFwdZD = 8;                           // z prefetch depth (stages)
constexpr int kFwdProducers = 256;
constexpr int kFwdThreads = kFwdProducers + 32;     // + MMA warp
constexpr int kFwdMaxRTG = 4;                       // accumulators: TMEM columns 0..63
constexpr uint32_t kFwdAcol = 64;                   // A buffers: columns 64 + 64 b + 16 sub + k
constexpr uint32_t kFwdTmemCols = 256;

struct FwdSmem {
  // B: W slice, rows = 16 classes, K = kFzCta, interleaved; [cos_hi, cos_lo, sin_hi, sin_lo]
  float b[4][kTcN * kFzCta];
  // per-thread z ring: [stage slot][quad j][thread] float4
  float4 zr[kFwdZD][2][kFwdProducers];
  uint64_t full[kFwdBuf], empty[kFwdBuf], done;
  uint32_t tslot;
};

__global__ void __launch_bounds__(kFwdThreads, 2)
k_fused_fwd_tc(const float* __restrict__ z, int64_t m, int64_t n, int64_t ldz, int64_t zc0,
               const float* __restrict__ w, int64_t F, int C, int64_t col_cos, int64_t col_sin, int rtg,
               float* __restrict__ lpart) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  FwdSmem& S = *reinterpret_cast<FwdSmem*>(smraw);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int ks = blockIdx.y;
  const int64_t z0 = (int64_t)ks * kFzCta;
  const int nz = (int)(n - z0 < kFzCta ? n - z0 : kFzCta);
  const int64_t rt0 = (int64_t)blockIdx.x * rtg;
  const int64_t rts = (m + kTcM - 1) / kTcM;
  const int nrt = (int)(rts - rt0 < rtg ? rts - rt0 : rtg);
  constexpr int SPR = kFzCta / kFwdStageZ;            // stages per row tile
  const int stages = nrt * SPR;
  constexpr int kMmaWarp = kFwdProducers / 32;

  if (t == 0) {
    for (int b = 0; b < kFwdBuf; ++b) {
      mbar_init(&S.full[b], kFwdProducers);
      mbar_init(&S.empty[b], 1);
    }
    mbar_init(&S.done, 1);
    fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc<kFwdTmemCols>(&S.tslot);
  // producer mapping: warp w writes TMEM lanes 32*(w%4).. (rows) and the
  // columns of z quads q, q+1 with q = 2*(w/4)
  const int q = 2 * (warp >> 2), prow = 32 * (warp & 3) + lane;
  // rows clamped into the tile, z beyond n meets zero W columns
  auto issue = [&](int s) {
    if (s < stages) {
      const int64_t r = (rt0 + s / SPR) * kTcM + prow;
      const int64_t rr = r < m ? r : m - 1;
      const int zi = (s % SPR) * kFwdStageZ + 4 * q;
      const int slot = s % kFwdZD;
      // tiled z: lanes = consecutive rows of one unit
      cp_async16(&S.zr[slot][0][t], z + zt_offset(ldz, rr, zc0 + z0 + (zi < nz ? zi : 0)));
      cp_async16(&S.zr[slot][1][t], z + zt_offset(ldz, rr, zc0 + z0 + (zi + 4 < nz ? zi + 4 : 0)));
    }
    cp_async_commit();  // one group per stage (possibly empty)
  };
  // W slice -> B tiles (hi/lo), zero for padded classes / z beyond n (W is
  // not written by the z producer this kernel follows: read before pdl_wait)
  for (int idx = t; idx < kTcN * kFzCta; idx += blockDim.x) {
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
  pdl_wait();  // z tile complete
  pdl_trigger();
  if (warp < kMmaWarp)
    for (int d = 0; d < kFwdZD; ++d) issue(d);
  umma::fence_smem_to_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = S.tslot;
  if (warp < kMmaWarp) {
    // ---------------- producers
    const uint32_t lane_base = tm + ((uint32_t)(32 * (warp & 3)) << 16);
    for (int s = 0; s < stages; ++s) {
      const int b = s % kFwdBuf, slot = s % kFwdZD;
      cp_async_wait<kFwdZD - 1>();  // stage s (this thread's own copies) landed
      const float4 za = S.zr[slot][0][t], zc = S.zr[slot][1][t];
      const float zv[8] = {za.x, za.y, za.z, za.w, zc.x, zc.y, zc.z, zc.w};
      float c[8], sn[8], ch[8], cl[8], sh[8], sl[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        __sincosf(zv[j], &sn[j], &c[j]);
        split_tf32(c[j], ch[j], cl[j]);
        split_tf32(sn[j], sh[j], sl[j]);
      }
      issue(s + kFwdZD);  // the slot's values are consumed above
      if (s >= kFwdBuf) {
        mbar_wait(&S.empty[b], (uint32_t)((s / kFwdBuf - 1) & 1));
        umma::fence_after();
      }
      const uint32_t col = lane_base + kFwdAcol + (uint32_t)(64 * b + 4 * q);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        umma::tmem_st4(col + 4 * h + 0, ch[4 * h], ch[4 * h + 1], ch[4 * h + 2], ch[4 * h + 3]);
        umma::tmem_st4(col + 4 * h + 16, cl[4 * h], cl[4 * h + 1], cl[4 * h + 2], cl[4 * h + 3]);
        umma::tmem_st4(col + 4 * h + 32, sh[4 * h], sh[4 * h + 1], sh[4 * h + 2], sh[4 * h + 3]);
        umma::tmem_st4(col + 4 * h + 48, sl[4 * h], sl[4 * h + 1], sl[4 * h + 2], sl[4 * h + 3]);
      }
      umma::tmem_wait_st();
      umma::fence_before();
      mbar_arrive(&S.full[b]);
    }
    cp_async_wait<0>();
  } else if (lane == 0) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = umma::idesc_tf32(kTcM, kTcN);
    for (int s = 0; s < stages; ++s) {
      const int b = s % kFwdBuf, rt = s / SPR, k8 = s % SPR;
      mbar_wait(&S.full[b], (uint32_t)((s / kFwdBuf) & 1));
      umma::fence_after();
      const uint32_t acc = tm + (uint32_t)(rt * kTcN);
      const uint32_t abuf = tm + kFwdAcol + (uint32_t)(64 * b);
#pragma unroll
      for (int part = 0; part < 2; ++part) {  // cos, sin
#pragma unroll
        for (int kk = 0; kk < kFwdStageZ; kk += 8) {
          const unsigned char* bb = reinterpret_cast<const unsigned char*>(S.b[2 * part]);
          const unsigned char* bl = reinterpret_cast<const unsigned char*>(S.b[2 * part + 1]);
          const uint32_t boff = ((k8 * kFwdStageZ + kk) / 4) * kTcN * 16;
          const uint64_t dbh = umma::smem_desc(bb + boff, kTcN * 16, 128);
          const uint64_t dbl = umma::smem_desc(bl + boff, kTcN * 16, 128);
          const uint32_t ah = abuf + (uint32_t)(32 * part + kk), al = ah + 16;
          umma::mma_tf32_ts(acc, ah, dbh, idesc, (k8 > 0 || part > 0 || kk > 0) ? 1u : 0u);
          umma::mma_tf32_ts(acc, ah, dbl, idesc, 1u);
          umma::mma_tf32_ts(acc, al, dbh, idesc, 1u);
        }
      }
      umma::commit(&S.empty[b]);
    }
    umma::commit(&S.done);
  }
  // ---------------- epilogue: TMEM -> partial logits.  Rows rt0*128 ..
  // of chunk ks are one contiguous [rows][C] block of lpart: stage it in
  // shared memory (the z ring is idle now) and store it coalesced.
  __syncwarp();
  float* stage_out = reinterpret_cast<float*>(&S.zr[0][0][0]);  // nrt*128*C <= 4*128*16 floats
  if (warp < 4) {
    mbar_wait(&S.done, 0u);
    umma::fence_after();
    for (int rt = 0; rt < nrt; ++rt) {
      float v[16];
      umma::tmem_ld16(tm + ((uint32_t)(32 * warp) << 16) + (uint32_t)(rt * kTcN), v);
      float* o = stage_out + (rt * kTcM + 32 * warp + lane) * C;
      for (int c = 0; c < C; ++c) o[c] = v[c];
    }
  }
  __syncthreads();
  {
    const int64_t r0 = rt0 * kTcM;
    const int64_t nrows = m - r0 < (int64_t)nrt * kTcM ? m - r0 : (int64_t)nrt * kTcM;
    float* dst = lpart + ((int64_t)ks * m + r0) * C;
    for (int64_t i = t; i < nrows * C; i += blockDim.x) dst[i] = stage_out[i];
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<kFwdTmemCols>(tm);
}

// ---------------------------------------------------------------- backward
// One CTA per 64-z slice (M = 128 features: 64 cos, 64 sin), K = all rows in
// stages of 32 rows.  A cp.async loader warp streams the stage's z block
// (32 rows x 64 z) and delta rows into shared rings; 8 producer warps write
// the A operand (feature = TMEM lane, row = column; tf32 hi/lo) with
// tcgen05.st -- warp w owns lanes 32*(w%4).. (cos for the first 64 features,
// sin for the rest) and rows 16*(w/4)..+15 of the stage -- and 4 of them
// build the small B tiles (delta^T hi/lo) in shared memory; one thread
// issues 12 MMAs per stage with A from TMEM.
constexpr int kBwdBuf = 3;
constexpr int kBwdZBuf = 4;
constexpr int kBwdProducers = 256;
constexpr int kBwdThreads = kBwdProducers + 64;
constexpr uint32_t kBwdAcol = 32;                 // A buffers: columns 32 + 64 b + {0: hi, 32: lo} + k
constexpr uint32_t kBwdTmemCols = 256;

struct BwdSmem {
  // B stages: rows = 16 classes, K = 32 rows; [buf][hi, lo]
  float b[kBwdBuf][2][kTcN * kBrowStage];
  float zr[kBwdZBuf][kBrowStage * kBzCta];      // [stage][row][64 z]
  float dr[kBwdZBuf][kBrowStage * kTcN];        // [stage][row][C] (C <= 16)
  uint64_t full[kBwdBuf], empty[kBwdBuf], zfull[kBwdZBuf], zempty[kBwdZBuf], done;
  uint32_t tslot;
};

__global__ void __launch_bounds__(kBwdThreads, 2)
k_fused_bwd_tc(const float* __restrict__ z, int64_t m, int64_t n, int64_t ldz, int64_t zc0,
               const float* __restrict__ delta, int C, int64_t F, int64_t col_cos, int64_t col_sin,
               float* dw, float* w, float lr, float l2) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  BwdSmem& S = *reinterpret_cast<BwdSmem*>(smraw);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int64_t z0 = (int64_t)blockIdx.x * kBzCta;
  const int stages = (int)((m + kBrowStage - 1) / kBrowStage);
  constexpr int kMmaWarp = kBwdProducers / 32, kLoadWarp = kMmaWarp + 1;
  pdl_wait();
  pdl_trigger();
  if (t == 0) {
    for (int b = 0; b < kBwdBuf; ++b) {
      mbar_init(&S.full[b], kBwdProducers);
      mbar_init(&S.empty[b], 1);
    }
    for (int b = 0; b < kBwdZBuf; ++b) {
      mbar_init(&S.zfull[b], 32);
      mbar_init(&S.zempty[b], kBwdProducers / 32);
    }
    mbar_init(&S.done, 1);
    fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc<kBwdTmemCols>(&S.tslot);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = S.tslot;
  constexpr uint32_t BS = kTcN * kBrowStage * 4;

  if (warp == kLoadWarp) {
    // ---------------- loader: 32 rows x 64 z (512 chunks of 16 B, 16 per
    // lane; rows and z clamped into the tile) + the stage's delta rows
    // (contiguous, 32*C floats; a chunk may run past m*C into the scratch
    // allocation's 256-byte alignment padding, those values are never used)
    const int64_t dchunks = (m * C + 3) / 4;
    for (int s = 0; s < stages; ++s) {
      const int zb = s % kBwdZBuf;
      if (s >= kBwdZBuf) mbar_wait(&S.zempty[zb], (uint32_t)((s / kBwdZBuf - 1) & 1));
      const int64_t rb = (int64_t)s * kBrowStage;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        // chunk -> (column quad zq, row): one instruction covers 16
        // rows x 32 B of one unit, i.e. 512 contiguous bytes
        const int ch = lane + 32 * j, row = (ch >> 1) & 31, zq = ((ch >> 6) << 1) | (ch & 1);
        const int64_t r = rb + row < m ? rb + row : m - 1;
        const int64_t zi = z0 + 4 * zq < n ? z0 + 4 * zq : 0;
        cp_async16(&S.zr[zb][row * kBzCta + 4 * zq], z + zt_offset(ldz, r, zc0 + zi));  // tiled z
      }
      const int64_t c0 = rb * C / 4;  // 16-byte chunk index of the stage's first delta
      for (int j = lane; j < kBrowStage * C / 4; j += 32)
        if (c0 + j < dchunks) cp_async16(&S.dr[zb][4 * j], delta + 4 * (c0 + j));
      cp_async_arrive(&S.zfull[zb]);
    }
  } else if (warp < kMmaWarp) {
    // ---------------- producers
    const int lq = warp & 3, rh = warp >> 2;
    const int f = 32 * lq + lane, zi = f & 63;
    const bool is_cos = lq < 2;
    const uint32_t lane_base = tm + ((uint32_t)(32 * lq) << 16);
    const int bc = t % kTcN, bq = t / kTcN;   // B items on threads < 128
    for (int s = 0; s < stages; ++s) {
      const int zb = s % kBwdZBuf, buf = s % kBwdBuf;
      const int64_t rb = (int64_t)s * kBrowStage;
      mbar_wait(&S.zfull[zb], (uint32_t)((s / kBwdZBuf) & 1));
      float hi[16], lo[16], d[4];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float zz = S.zr[zb][(16 * rh + j) * kBzCta + zi];
        const float v = is_cos ? __cosf(zz) : __sinf(zz);
        split_tf32(v, hi[j], lo[j]);
      }
      if (t < kTcN * (kBrowStage / 4)) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t r = rb + 4 * bq + j;
          d[j] = (bc < C && r < m) ? S.dr[zb][(4 * bq + j) * C + bc] : 0.f;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.zempty[zb]);
      if (s >= kBwdBuf) {
        mbar_wait(&S.empty[buf], (uint32_t)((s / kBwdBuf - 1) & 1));
        umma::fence_after();
      }
      const uint32_t col = lane_base + kBwdAcol + (uint32_t)(64 * buf + 16 * rh);
      umma::tmem_st16(col, hi);
      umma::tmem_st16(col + 32, lo);
      if (t < kTcN * (kBrowStage / 4)) {  // B = delta^T: (class c, row quad q); zero rows >= m
        unsigned char* B = reinterpret_cast<unsigned char*>(S.b[buf][0]);
        float dh[4], dl[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) split_tf32(d[j], dh[j], dl[j]);
        const uint32_t ob = umma::tile_off(bc, 4 * bq, kTcN);
        sts128(B + ob, dh[0], dh[1], dh[2], dh[3]);
        sts128(B + BS + ob, dl[0], dl[1], dl[2], dl[3]);
        umma::fence_smem_to_async();
      }
      umma::tmem_wait_st();
      umma::fence_before();
      mbar_arrive(&S.full[buf]);
    }
  } else if (lane == 0) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = umma::idesc_tf32(kTcM, kTcN);
    for (int s = 0; s < stages; ++s) {
      const int buf = s % kBwdBuf;
      mbar_wait(&S.full[buf], (uint32_t)((s / kBwdBuf) & 1));
      umma::fence_after();
      const unsigned char* B = reinterpret_cast<const unsigned char*>(S.b[buf][0]);
      const uint32_t abuf = tm + kBwdAcol + (uint32_t)(64 * buf);
#pragma unroll
      for (int k0 = 0; k0 < kBrowStage; k0 += 8) {
        const uint32_t boff = (k0 / 4) * kTcN * 16;
        const uint64_t dbh = umma::smem_desc(B + boff, kTcN * 16, 128);
        const uint64_t dbl = umma::smem_desc(B + BS + boff, kTcN * 16, 128);
        const uint32_t ah = abuf + (uint32_t)k0, al = ah + 32;
        umma::mma_tf32_ts(tm, ah, dbh, idesc, (s > 0 || k0 > 0) ? 1u : 0u);
        umma::mma_tf32_ts(tm, ah, dbl, idesc, 1u);
        umma::mma_tf32_ts(tm, al, dbh, idesc, 1u);
      }
      umma::commit(&S.empty[buf]);
    }
    umma::commit(&S.done);
  }
  __syncwarp();
  if (warp < 4) {
    if (stages > 0) mbar_wait(&S.done, 0u);
    umma::fence_after();
    float v[16];
    umma::tmem_ld16(tm + ((uint32_t)(32 * warp) << 16), v);
    const int f = 32 * warp + lane;   // feature row of the tile
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
  if (warp == 0) umma::tmem_free<kBwdTmemCols>(tm);
}

int fused_fwd_tc(const float* z, int64_t m, int64_t n, int64_t ldz, int64_t zc0, const float* w, int64_t F,
                 int C, int64_t col_cos, int64_t col_sin, float* lpart, cudaStream_t st) {
  if (C > kTcN) return fail_value("num_classes must be <= %d", kTcN);
  const size_t smem = sizeof(FwdSmem);
  static PerDevice pd;
  const DeviceSlot* ds = nullptr;
  MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot&) {
    return check_cuda(cudaFuncSetAttribute(k_fused_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem), "fwd tc smem");
  }));
  const int64_t KS = (n + kFzCta - 1) / kFzCta, RT = (m + kTcM - 1) / kTcM;
  // row tiles per CTA: enough CTAs for one wave of 2 per SM, W slice reused
  int64_t per = 296 / KS;
  if (per < 1) per = 1;
  int64_t rtg = (RT + per - 1) / per;
  if (rtg > kFwdMaxRTG) rtg = kFwdMaxRTG;
  if (rtg < 1) rtg = 1;
  dim3 grid((unsigned)((RT + rtg - 1) / rtg), (unsigned)KS);
  return launch_pdl(k_fused_fwd_tc, grid, dim3(kFwdThreads), smem, st, "k_fused_fwd_tc", z, m, n, ldz,
                    zc0, w, F, C, col_cos, col_sin, (int)rtg, lpart);
}

int fused_bwd_tc(const float* z, int64_t m, int64_t n, int64_t ldz, int64_t zc0, const float* delta, int C,
                 int64_t F,
                 int64_t col_cos, int64_t col_sin, float* dw, float* w, float lr, float l2,
                 cudaStream_t st) {
  if (C > kTcN) return fail_value("num_classes must be <= %d", kTcN);
  const size_t smem = sizeof(BwdSmem);
  static PerDevice pd;
  const DeviceSlot* ds = nullptr;
  MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot&) {
    return check_cuda(cudaFuncSetAttribute(k_fused_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem), "bwd tc smem");
  }));
  const unsigned grid = (unsigned)((n + kBzCta - 1) / kBzCta);
  return launch_pdl(k_fused_bwd_tc, dim3(grid), dim3(kBwdThreads), smem, st, "k_fused_bwd_tc", z, m, n,
                    ldz, zc0, delta, C, F, col_cos, col_sin, dw, w, lr, l2);
}

int64_t fused_tc_ksplits(int64_t n) { return (n + kFzCta - 1) / kFzCta; }

}  // namespace mck
