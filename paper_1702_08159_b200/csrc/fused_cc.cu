// K6 contractions on the FP32 pipes with packed f32x2 FMAs (FFMA2): the
// default engine of the config-4 fused classifier.
//
// With 10 classes the contraction is a skinny GEMM (N = 10): per z value and
// row it needs one sin and one cos (MUFU) and 20 FMAs.  Packed FFMA2 does
// two of those FMAs per lane-instruction, so per 128 (row, z) pairs a warp
// issues 8 MUFU + 40 FFMA2 + a few loads: the MUFU pipe (16 results per
// clock per SM) and the HBM read of z are the bounds, not the FMA pipe.
//
// Both kernels are persistent (one CTA of kWarps warps per SM) and every
// warp works on its own items with its own cp.async ring (no CTA barriers):
//
// * forward  (k_fused_fwd_cc): item = 128 rows x kZW z values.  Lane l holds
//   rows l, l+32, l+64, l+96; a stage brings a [128 rows][8 z] slice of a z-tile unit
//   (4 KB contiguous; rows XOR-swizzled in shared memory so the per-row
//   16-byte reads are conflict free) and
//   the 8 z values' W (transposed per group to [z][cos classes | sin classes],
//   read as broadcasts).  Accumulators: class pairs as f32x2, 4 rows x 8.
//   Output: partial logits lpart[ks][r][c] of the item's z chunk, folded in
//   float64 by k_fused_fold (fixed order).
// * backward (k_fused_bwd_cc): item = 128 z columns x all rows.  Lane l holds
//   columns 4l..4l+3; a stage brings [8 rows][128 z] of z (16 runs of 256 B
//   of whole 128-byte lines) and the 8 rows' delta (float32).  dW of the 128 columns is complete at the end of the
//   item: written (plain or all-reduce bucket layout) or applied as the SGD
//   update in place -- no partial buffers, no second pass.
//
// Semantics: linear_model.py:95-131 (logits = phi W^T, dW = delta^T phi) with
// phi = [cos z | sin z] never stored (fastfood.py:209-226).
#include <cstdint>

#include "async_copy.cuh"
#include "mck_common.cuh"

namespace mck {

namespace {

#ifndef MCK_FWD_WARPS
#define MCK_FWD_WARPS 14
#endif
#ifndef MCK_FWD_STAGES
#define MCK_FWD_STAGES 3
#endif
constexpr int kCcWarps = MCK_FWD_WARPS;    // forward: warps per CTA (one CTA per SM)
constexpr int kCcStages = MCK_FWD_STAGES;  // forward: cp.async ring depth per warp
constexpr int kFRows = 128;     // forward: rows per item (4 per lane)
constexpr int kFZ = 8;          // forward: z per stage
constexpr int kZW = 1024;       // forward: z per item (one partial-logit chunk)
#ifndef MCK_BWD_WARPS
#define MCK_BWD_WARPS 14
#endif
#ifndef MCK_BWD_STAGES
#define MCK_BWD_STAGES 3
#endif
constexpr int kBWarps = MCK_BWD_WARPS;    // backward: warps per CTA
constexpr int kBStages = MCK_BWD_STAGES;  // backward: ring depth per warp
constexpr int kBRows = 8;       // backward: rows per stage
constexpr int kBCols = 128;     // backward: z columns per item (4 per lane)

__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
// d = a * b + d, two lanes' worth (sm_100 FFMA2)
__device__ __forceinline__ void ffma2(uint64_t& d, uint64_t a, uint64_t b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

template <int NCP>
struct FwdStage {
  float z[kFRows * kFZ];        // row r: 8 z, two 16-byte halves swapped when (r >> 2) & 1
  float w[kFZ * 2 * NCP];       // [k][cos classes | sin classes]
};

template <int NCP>
struct BwdStage {
  float z[kBRows * kBCols];     // [row][128 z]
  float d[kBRows * NCP];        // [row][classes], zero padded
};

}  // namespace

// wt[i][c] = W[c][col_cos + i], wt[i][NCP + c] = W[c][col_sin + i] (0 for c >= C).
// A CTA transposes 256 z indices through shared memory: coalesced reads of
// each class row, then the [256][2*NCP] block written linearly.
__global__ void __launch_bounds__(256) k_fused_wt(const float* __restrict__ w, int64_t F, int C, int NCP,
                                                  int64_t col_cos, int64_t col_sin, int64_t nz,
                                                  float* __restrict__ wt) {
  __shared__ float tile[256 * 33];
  pdl_wait();
  pdl_trigger();
  const int t = threadIdx.x;
  for (int64_t i0 = (int64_t)blockIdx.x * 256; i0 < nz; i0 += (int64_t)gridDim.x * 256) {
    const int ni = nz - i0 < 256 ? (int)(nz - i0) : 256;
    for (int k = 0; k < 2 * NCP; ++k) {
      const int c = k < NCP ? k : k - NCP;
      tile[t * 33 + k] = (c < C && t < ni) ? w[(int64_t)c * F + (k < NCP ? col_cos : col_sin) + i0 + t] : 0.f;
    }
    __syncthreads();
    const int total = ni * 2 * NCP;
    for (int e = t; e < total; e += 256) {
      const int i = e / (2 * NCP), k = e - i * (2 * NCP);
      wt[i0 * 2 * NCP + e] = tile[i * 33 + k];
    }
    __syncthreads();
  }
}

template <int NCP>
__global__ void __launch_bounds__(kCcWarps * 32, 1)
k_fused_fwd_cc(const float* __restrict__ z, int64_t m, int64_t nz, int64_t zcols, int64_t col0,
               const float* __restrict__ wt, int C, float* __restrict__ lpart) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  FwdStage<NCP>* ring = reinterpret_cast<FwdStage<NCP>*>(smraw) + warp * kCcStages;
  const int64_t RT = (m + kFRows - 1) / kFRows, KS = (nz + kZW - 1) / kZW;
  const int64_t items = RT * KS;
  const int64_t nwarps = (int64_t)gridDim.x * kCcWarps;
  pdl_wait();
  pdl_trigger();
  for (int64_t it = (int64_t)blockIdx.x * kCcWarps + warp; it < items; it += nwarps) {
    const int64_t rt = it % RT, ks = it / RT;
    const int64_t r0 = rt * kFRows, zb = ks * kZW;
    const int64_t ze = zb + kZW < nz ? zb + kZW : nz;
    const int nst = (int)((ze - zb + kFZ - 1) / kFZ);
    auto load = [&](int s) {
      if (s < nst) {
        FwdStage<NCP>& st = ring[s % kCcStages];
        const int64_t c0 = zb + (int64_t)s * kFZ;
        // [128 rows][8 z] of the z tile (one contiguous unit when MCK_ZT_LOG == 3;
        // rows >= m are never output)
        const float* unit = z + zt_offset(zcols, r0, col0 + c0);
#pragma unroll
        for (int t = 0; t < (kFRows * 2) / 32; ++t) {
          const int idx = lane + 32 * t, r = idx >> 1, j = idx & 1;
          cp_async16(&st.z[r * kFZ + ((j ^ ((r >> 2) & 1)) << 2)], unit + (r << MCK_ZT_LOG) + 4 * j);
        }
        for (int idx = lane; idx < kFZ * 2 * NCP / 4; idx += 32)
          cp_async16(&st.w[idx * 4], wt + c0 * 2 * NCP + idx * 4);
      }
      cp_async_commit();
    };
#pragma unroll
    for (int s = 0; s < kCcStages - 1; ++s) load(s);
    uint64_t acc[4][NCP / 2];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int p = 0; p < NCP / 2; ++p) acc[q][p] = 0ull;
    for (int s = 0; s < nst; ++s) {
      cp_async_wait<kCcStages - 2>();
      __syncwarp();
      const FwdStage<NCP>& st = ring[s % kCcStages];
      float zv[4][kFZ];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = lane + 32 * q, sw = (r >> 2) & 1;
        const float4 a = *reinterpret_cast<const float4*>(&st.z[r * kFZ + (sw << 2)]);
        const float4 b = *reinterpret_cast<const float4*>(&st.z[r * kFZ + ((sw ^ 1) << 2)]);
        zv[q][0] = a.x; zv[q][1] = a.y; zv[q][2] = a.z; zv[q][3] = a.w;
        zv[q][4] = b.x; zv[q][5] = b.y; zv[q][6] = b.z; zv[q][7] = b.w;
      }
#pragma unroll
      for (int k = 0; k < kFZ; ++k) {
        uint64_t wc[NCP / 2], ws[NCP / 2];
        const uint64_t* wk = reinterpret_cast<const uint64_t*>(&st.w[k * 2 * NCP]);
#pragma unroll
        for (int p = 0; p < NCP / 2; ++p) {
          wc[p] = wk[p];
          ws[p] = wk[NCP / 2 + p];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float sn, cs;
#ifdef MCK_EXP_NOMUFU
          cs = zv[q][k]; sn = zv[q][k] * 0.5f;
#else
          __sincosf(zv[q][k], &sn, &cs);
#endif
          const uint64_t cc = pk(cs, cs), ss = pk(sn, sn);
#pragma unroll
#ifdef MCK_EXP_NOFMA
          ffma2(acc[q][0], cc, wc[0]);
          ffma2(acc[q][1], ss, ws[1]);
#else
          for (int p = 0; p < NCP / 2; ++p) {
            ffma2(acc[q][p], cc, wc[p]);
            ffma2(acc[q][p], ss, ws[p]);
          }
#endif
        }
      }
      __syncwarp();
      load(s + kCcStages - 1);
    }
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t r = r0 + lane + 32 * q;
      if (r < m) {
        float* o = lpart + (ks * m + r) * C;
#pragma unroll
        for (int p = 0; p < NCP / 2; ++p) {
          const float2 v = upk(acc[q][p]);
          if (2 * p < C) o[2 * p] = v.x;
          if (2 * p + 1 < C) o[2 * p + 1] = v.y;
        }
      }
    }
  }
}

// dW of columns i in [0, nz): g[c][i] = sum_r delta[r][c] cos(z[r][i]) (cos
// half) / sin (sin half); delta is the zero-padded float32 [rows8][NCP] copy.
// (cos
// half) / sin (sin half); written to dw[c*ldw + cos0 + i] / [c*ldw + sin0 + i]
// or applied as w -= lr*(g + 2*l2*w) at the same positions.
template <int NCP>
__global__ void __launch_bounds__(kBWarps * 32, 1)
k_fused_bwd_cc(const float* __restrict__ z, int64_t m, int64_t nz, int64_t zcols, int64_t col0,
               const float* __restrict__ delta, int C, int64_t ldw, int64_t cos0, int64_t sin0,
               float* __restrict__ dw, float* __restrict__ w, float lr, float l2) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  BwdStage<NCP>* ring = reinterpret_cast<BwdStage<NCP>*>(smraw) + warp * kBStages;
  const int64_t items = (nz + kBCols - 1) / kBCols;
  const int64_t nwarps = (int64_t)gridDim.x * kBWarps;
  const int nst = (int)((m + kBRows - 1) / kBRows);
  pdl_wait();
  pdl_trigger();
  for (int64_t it = (int64_t)blockIdx.x * kBWarps + warp; it < items; it += nwarps) {
    const int64_t c0 = it * kBCols;
    const int64_t col = c0 + 4 * lane;
    const bool live = col < nz;  // nz is a multiple of 8, so 4 columns are all in or all out
    auto load = [&](int s) {
      if (s < nst) {
        BwdStage<NCP>& st = ring[s % kBStages];
        const int64_t rb = (int64_t)s * kBRows;
        // lane: 4 columns of a tile row piece (8 lanes = one 128-byte line).
        // Rows >= m are zero-filled (delta is zero there too, and the tile's
        // padding rows are never written).
        const float* unit = z + zt_offset(zcols, rb, col0 + c0 + 4 * lane);
#pragma unroll
        for (int rr = 0; rr < kBRows; ++rr)
          if (live) cp_async16_zfill(&st.z[rr * kBCols + 4 * lane], unit + (rr << MCK_ZT_LOG), rb + rr < m);
        // delta: 8 padded rows of NCP floats, contiguous (zero beyond m and C)
        if (lane < kBRows * NCP / 4) cp_async16(&st.d[4 * lane], delta + rb * NCP + 4 * lane);
      }
      cp_async_commit();
    };
#pragma unroll
    for (int s = 0; s < kBStages - 1; ++s) load(s);
    uint64_t ac[4][NCP / 2], as[4][NCP / 2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int p = 0; p < NCP / 2; ++p) ac[j][p] = as[j][p] = 0ull;
    for (int s = 0; s < nst; ++s) {
      cp_async_wait<kBStages - 2>();
      __syncwarp();
      const BwdStage<NCP>& st = ring[s % kBStages];
#pragma unroll 2
      for (int rr = 0; rr < kBRows; ++rr) {
        const float4 zq = live ? *reinterpret_cast<const float4*>(&st.z[rr * kBCols + 4 * lane])
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        uint64_t d[NCP / 2];
        const uint64_t* dr = reinterpret_cast<const uint64_t*>(&st.d[rr * NCP]);
#pragma unroll
        for (int p = 0; p < NCP / 2; ++p) d[p] = dr[p];
        const float zz[4] = {zq.x, zq.y, zq.z, zq.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float sn, cs;
          __sincosf(zz[j], &sn, &cs);
          const uint64_t cc = pk(cs, cs), ss = pk(sn, sn);
#pragma unroll
          for (int p = 0; p < NCP / 2; ++p) {
            ffma2(ac[j][p], cc, d[p]);
            ffma2(as[j][p], ss, d[p]);
          }
        }
      }
      __syncwarp();
      load(s + kBStages - 1);
    }
    cp_async_wait<0>();
    __syncwarp();
    if (!live) continue;
#pragma unroll
    for (int p = 0; p < NCP / 2; ++p) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 2 * p + h;
        if (c >= C) continue;
        float gc[4], gs[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 a = upk(ac[j][p]), b = upk(as[j][p]);
          gc[j] = h ? a.y : a.x;
          gs[j] = h ? b.y : b.x;
        }
        const int64_t oc = (int64_t)c * ldw + cos0 + col, os = (int64_t)c * ldw + sin0 + col;
        if (w) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float wc = w[oc + j], wsn = w[os + j];
            w[oc + j] = wc - lr * (l2 != 0.f ? gc[j] + 2.f * l2 * wc : gc[j]);
            w[os + j] = wsn - lr * (l2 != 0.f ? gs[j] + 2.f * l2 * wsn : gs[j]);
          }
        } else {
          *reinterpret_cast<float4*>(dw + oc) = make_float4(gc[0], gc[1], gc[2], gc[3]);
          *reinterpret_cast<float4*>(dw + os) = make_float4(gs[0], gs[1], gs[2], gs[3]);
        }
      }
    }
  }
}

namespace {

template <class Fn>
int dispatch_ncp(int C, Fn fn) {
  switch ((C + 1) & ~1) {
    case 2: return fn(std::integral_constant<int, 2>{});
    case 4: return fn(std::integral_constant<int, 4>{});
    case 6: return fn(std::integral_constant<int, 6>{});
    case 8: return fn(std::integral_constant<int, 8>{});
    case 10: return fn(std::integral_constant<int, 10>{});
    case 12: return fn(std::integral_constant<int, 12>{});
    case 14: return fn(std::integral_constant<int, 14>{});
    case 16: return fn(std::integral_constant<int, 16>{});
    default: return fail_value("num_classes must be in 2..16");
  }
}

}  // namespace

int64_t fused_cc_ksplits(int64_t nz) { return (nz + kZW - 1) / kZW; }
int64_t fused_cc_wt_floats(int64_t nz) { return nz * 2 * 16; }

// Partial logits of the group's nz z columns: lpart[ks][r][c], ks < fused_cc_ksplits(nz).
int fused_fwd_cc(const float* z, int64_t m, int64_t nz, int64_t zcols, int64_t col0, const float* w,
                 int64_t F, int C, int64_t col_cos, int64_t col_sin, float* wt, float* lpart,
                 cudaStream_t st) {
  if (nz % 8 || zcols % 8 || col0 % 8 || (reinterpret_cast<uintptr_t>(z) & 15))
    return fail_value("internal: fused forward needs 8-aligned z columns");
  return dispatch_ncp(C, [&](auto ncp) {
    constexpr int NCP = decltype(ncp)::value;
    MCK_TRY(launch_pdl(k_fused_wt, dim3(148 * 4), dim3(256), 0, st, "k_fused_wt", w, F, C, NCP, col_cos,
                       col_sin, nz, wt));
    const size_t smem = sizeof(FwdStage<NCP>) * kCcStages * kCcWarps;
    auto kern = k_fused_fwd_cc<NCP>;
    static PerDevice pd;
    const DeviceSlot* ds = nullptr;
    MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot&) {
      return check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "fwd cc smem");
    }));
    const int64_t items = ((m + kFRows - 1) / kFRows) * ((nz + kZW - 1) / kZW);
    int64_t grid = (items + kCcWarps - 1) / kCcWarps;
    if (grid > ds->sms) grid = ds->sms;
    return launch_pdl(kern, dim3((unsigned)grid), dim3(kCcWarps * 32), smem, st, "k_fused_fwd_cc", z, m,
                      nz, zcols, col0, (const float*)wt, C, lpart);
  });
}

int fused_bwd_cc(const float* z, int64_t m, int64_t nz, int64_t zcols, int64_t col0, const float* delta,
                 int C, int64_t ldw, int64_t cos0, int64_t sin0, float* dw, float* w, float lr, float l2,
                 cudaStream_t st) {
  if (nz % 8 || zcols % 8 || col0 % 8 || (reinterpret_cast<uintptr_t>(z) & 15))
    return fail_value("internal: fused backward needs 8-aligned z columns");
  if (!w && ((ldw % 4) || (cos0 % 4) || (sin0 % 4) || (reinterpret_cast<uintptr_t>(dw) & 15)))
    return fail_value("internal: fused backward needs 16-byte aligned dW rows");
  return dispatch_ncp(C, [&](auto ncp) {
    constexpr int NCP = decltype(ncp)::value;
    const size_t smem = sizeof(BwdStage<NCP>) * kBStages * kBWarps;
    auto kern = k_fused_bwd_cc<NCP>;
    static PerDevice pd;
    const DeviceSlot* ds = nullptr;
    MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot&) {
      return check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "bwd cc smem");
    }));
    const int64_t items = (nz + kBCols - 1) / kBCols;
    int64_t grid = (items + kBWarps - 1) / kBWarps;
    if (grid > ds->sms) grid = ds->sms;
    return launch_pdl(kern, dim3((unsigned)grid), dim3(kBWarps * 32), smem, st, "k_fused_bwd_cc", z, m,
                      nz, zcols, col0, delta, C, ldw, cos0, sin0, dw, w, lr, l2);
  });
}

}  // namespace mck
