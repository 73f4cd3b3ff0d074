// K3 -- fused Fastfood expansion (replaces fastfood.py:179-226:
// apply_zhat_batch + feature_map_batch).
//
// Per row and block e:
//   x*B  : sign-bit XOR from a per-thread mask word          (fastfood.py:190)
//   H    : register butterflies + shared-memory exchanges     (:191)
//   Pi,G : one scatter into shared memory and one gather; slots are edge-
//          coloured so scatter and gather are bank-conflict free, and the
//          product z1[perm[p]] * g[p] is the same fp32 product the reference
//          forms after its gather (:192-193)
//   H    : middle rounds first, ending in the 16-byte store layout (:194)
//   C*s  : one multiply when 1/(sigma*sqrt n) is a power of two (exactly the
//          reference's two roundings), else two               (:195-196)
//   cos/sin epilogue (MUFU), [cos | sin] halves, optional float32(1/sqrt(D))
//          (:220-225); 16-byte stores.
// HBM traffic is one read of x and one write of the features.
//
// k_fastfood_pair (n = 1024, c0/c2/c3): two rows per warp, packed f32x2,
//   block-major work units, TMA-staged tables and x rows.
// k_fastfood (other n): one row per thread group; x kept in registers for all
//   E blocks for n <= 8192; n = 16384 (c4) runs 512-thread rows over
//   balanced (row, block) item ranges and reads its tables through L1/L2.
// The `parity` variant restates the reference arithmetic exactly (sequential
// base-256 sums, (a+b)-2b combine, separate roundings) for bit-exact z checks.
#include "mck_common.cuh"
#include "fwht_core.cuh"
#include "tables.cuh"
#include "async_copy.cuh"
#include "perm_color.cuh"

#include <cstring>
#include <vector>

namespace mck {

#ifndef MCK_ST_OUT
#define MCK_ST_OUT 2  // features are written once and never re-read here: no L1 allocation (c2 batch 110.2 -> 109.1 us; .cs 109.5, .wt 110.4)
#endif
__device__ __forceinline__ void st_out(float4* p, float4 v) {
#if MCK_ST_OUT == 1
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
#elif MCK_ST_OUT == 2
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
#elif MCK_ST_OUT == 3
  asm volatile("st.global.wt.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
#else
  *p = v;
#endif
}

template <class C>
constexpr int ff_rows_per_cta() { return C::T >= 256 ? 1 : 256 / C::T; }

// Per-block factor tables, staged into shared memory by TMA bulk copies:
// scat [R][T] uint2 | cs [N] f32 | bmask [bm_stride] u32 | gcol [R/4][T] u32.
// n >= 1024 (whole warps per row) use the edge-coloured permutation
// (perm_color.cu): scatter and gather are both bank-conflict free; smaller n
// scatter to the padded layout and gather with the structured layout read.
template <class C>
constexpr bool ff_colored() { return C::T >= 32; }
// n = 1024 runs the two-rows-per-thread kernel (k_fastfood_pair)
template <class C>
constexpr bool ff_pair() { return C::LOGN == 10 && C::LOGR == 5; }
template <class C>
constexpr int bm_stride() { return ((((C::R + 31) / 32) * C::T) + 3) & ~3; }
template <class C>
constexpr int tab_bytes() {
  return C::N * 8 + C::N * 4 + bm_stride<C>() * 4 + (ff_colored<C>() ? C::N : 0);
}
template <class C>
constexpr int tab_slot() { return (tab_bytes<C>() + 127) & ~127; }
template <class C>
constexpr size_t ff_rows_bytes() { return (size_t)ff_rows_per_cta<C>() * C::SMEM_FLOATS * 4; }
// Tables are staged when both buffers fit next to the row buffers (n <= 4096);
// larger n (c4: 197 KB of tables per block) reads them through L2.
template <class C>
constexpr bool ff_staged() { return 128 + 2 * (size_t)tab_slot<C>() + ff_rows_bytes<C>() <= 200 * 1024; }
template <class C>
constexpr size_t ff_smem_bytes() {
  return ff_staged<C>() ? 128 + 2 * (size_t)tab_slot<C>() + ff_rows_bytes<C>() : ff_rows_bytes<C>();
}


// ---------------------------------------------------------------- derived tables
__global__ void k_perminv(const int32_t* perm, int64_t n, int32_t E, int32_t* perminv,
                          int32_t* flag) {
  const int64_t total = n * E;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / n, i = t % n;
    const int32_t j = perm[t];
    if (j < 0 || j >= n) {
      atomicExch(flag, 1);
      continue;
    }
    perminv[e * n + j] = (int32_t)i;
  }
}

__global__ void k_perm_check(const int32_t* perm, const int32_t* perminv, int64_t n, int32_t E,
                             int32_t* flag) {
  const int64_t total = n * E;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / n, j = t % n;
    const int32_t i = perminv[t];
    if (i < 0 || i >= n || perm[e * n + i] != (int32_t)j) atomicExch(flag, 1);
  }
}

__global__ void k_cscale(const float* c, int64_t total, float scale, int fold, float* cs) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    cs[t] = fold ? c[t] * scale : c[t];
}

// Sign masks (layout L) and scatter entries (layout of H1's last round).
template <class C>
__global__ void k_prepare(const float* b, const float* g, const int32_t* perminv, int32_t E,
                          uint32_t* bmask, uint2* scat) {
  constexpr int R = C::R, T = C::T, W = (R + 31) / 32;
  constexpr uint32_t PM = last_mid_regs<C>();
  const int64_t total = (int64_t)E * R * T;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / (R * T);
    const int k = (int)((t / T) % R);
    const uint32_t tid = (uint32_t)(t % T);
    const int64_t off = e * (int64_t)C::N;
    const uint32_t j = lay_index<PM>(thread_part<C::FULL, PM>(tid), k);
    const int32_t pinv = perminv[off + j];
    // byte offset into the row's shared buffer: STS [offset + uniform base]
    scat[t] = make_uint2(4u * pad_addr((uint32_t)pinv), __float_as_uint(g[off + pinv]));
    if (k < W) {
      uint32_t bits = 0;
      for (int q = 0; q < 32 && 32 * k + q < R; ++q) {
        const uint32_t i = lay_index<C::PL>(thread_part<C::FULL, C::PL>(tid), 32 * k + q);
        if (b[off + i] < 0.0f) bits |= 1u << q;
      }
      bmask[e * bm_stride<C>() + k * T + tid] = bits;
    }
  }
}

// ---------------------------------------------------------------- sincos
// MUFU sin/cos work in turns on the fractional part of z/(2 pi); the only
// error beyond the unit's ~2^-21 is the rounding of z/(2 pi), i.e. about
// |z| * 2^-24 -- below the fp32 error of z itself, so no explicit range
// reduction is needed.
__device__ __forceinline__ void sincos_fast(float z, float& s, float& c) { __sincosf(z, &s, &c); }

struct FFParams {
  const float* x;
  int64_t m;
  int64_t ldx;
  int32_t d;
  const int32_t* rows;
  const uint32_t* bmask;
  const uint2* scat;
  const float* cs;
  const uint32_t* gcol;
  const uint16_t* soff;
  const float* ggath;
  float scale;
  float norm;
  float* out;
  int64_t ldo;
  int32_t E;   // blocks computed: e0 .. e0+E-1, written at columns (e-e0)*n
  int64_t D;
  int32_t e0;
  int32_t tile8;    // z written in the tiled layout (zt_offset, ldo = tile columns), fused path
};

// Persistent: each CTA walks row groups g = blockIdx.x, +gridDim.x, ...; the
// tables of iteration it+1 (next block, or block 0 of the next group) are in
// flight while iteration it computes.
template <class C>
constexpr int ff_min_blocks() {
  return C::R >= 64 ? 2 : (C::T * ff_rows_per_cta<C>() <= 256 ? 3 : 2);
}
// x kept in registers across the E blocks: small rows only (n = 16384 runs
// 512-thread rows at two CTAs per SM and re-reads x per block)
template <class C>
constexpr bool ff_xreg() { return C::R <= 32 && C::LOGN < 14; }

template <class C, bool FEAT, bool FOLD, bool VEC, bool XREG = ff_xreg<C>()>
__global__ void __launch_bounds__(C::T * ff_rows_per_cta<C>(), ff_min_blocks<C>())
k_fastfood(FFParams p) {
  constexpr int R = C::R, T = C::T, N = C::N, W = (R + 31) / 32;
  constexpr int ROWS = ff_rows_per_cta<C>();
  constexpr int SLOT = tab_slot<C>();
  constexpr bool STAGED = ff_staged<C>();
  extern __shared__ __align__(128) unsigned char ff_smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(ff_smem);
  unsigned char* tabs = ff_smem + 128;
  const int gid = threadIdx.x / T;
  const uint32_t tid = threadIdx.x % T;
  float* s = reinterpret_cast<float*>(ff_smem + (STAGED ? 128 + 2 * SLOT : 0)) + gid * C::SMEM_FLOATS;
  constexpr uint32_t P0 = C::mid_regs(0);

  const int64_t groups = (p.m + ROWS - 1) / ROWS;
  // XREG: groups strided over the CTAs, all E blocks per group (x read once).
  // Otherwise (n = 16384): (group, block) items, item = group * E + block,
  // strided over the CTAs (each CTA 55 or 56 items at config 4, so a launch
  // over several blocks fills every wave).  At any time the CTAs work on one
  // contiguous run of items, i.e. neighbouring rows of the same block: the
  // z tile lines of neighbouring rows are written close together.
  static_assert(XREG || !STAGED, "item loop assumes per-item table reads");
  const int64_t items = groups * p.E;
  const int64_t my_groups = XREG ? (groups > blockIdx.x ? (groups - 1 - blockIdx.x) / gridDim.x + 1 : 0)
                                 : (items > blockIdx.x ? (items - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  const int64_t total_it = my_groups * p.E;

  auto issue = [&](int64_t it) {  // thread 0 only
    const int e = p.e0 + (int)(it % p.E);
    unsigned char* dst = tabs + (it & 1) * SLOT;
    uint64_t* b = bar + (it & 1);
    mbar_expect_tx(b, tab_bytes<C>());
    bulk_g2s(dst, p.scat + (int64_t)e * N, N * 8, b);
    bulk_g2s(dst + N * 8, p.cs + (int64_t)e * N, N * 4, b);
    bulk_g2s(dst + N * 12, p.bmask + (int64_t)e * bm_stride<C>(), bm_stride<C>() * 4, b);
    if constexpr (ff_colored<C>())
      bulk_g2s(dst + N * 12 + bm_stride<C>() * 4, p.gcol + (int64_t)e * (N / 4), N, b);
  };
  pdl_wait();
  pdl_trigger();
  if (STAGED) {
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      mbar_init(bar + 1, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && total_it > 0) issue(0);
  }

  for (int64_t gi = 0; gi < my_groups; ++gi) {
    const int64_t slot = blockIdx.x + gi * gridDim.x;  // group (XREG) or item
    const int64_t grp = XREG ? slot : slot / p.E;
    const int64_t row = grp * ROWS + gid;
    const bool valid = row < p.m;
    const int e_lo = XREG ? 0 : (int)(slot % p.E);
    const int e_hi = XREG ? p.E : e_lo + 1;
    // ---- input row, layout L, zero padded (kept in registers for all E blocks)
    const float* xp = p.x + (valid ? (p.rows ? (int64_t)p.rows[row] : row) : 0) * p.ldx;
    auto load_x = [&](float (&dst)[R]) {
#pragma unroll
      for (int j = 0; j < R / 4; ++j) {
        const int i0 = 4 * (int)tid + j * 4 * T;
        if constexpr (VEC) {
          float4 t4 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (valid && i0 < p.d) t4 = __ldg(reinterpret_cast<const float4*>(xp + i0));
          dst[4 * j] = t4.x; dst[4 * j + 1] = t4.y; dst[4 * j + 2] = t4.z; dst[4 * j + 3] = t4.w;
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) dst[4 * j + c] = (valid && i0 + c < p.d) ? __ldg(xp + i0 + c) : 0.f;
        }
      }
    };
    // x stays in registers across the E blocks (XREG) or is re-read per
    // block (large R, or single-block launches of the fused path)
    float xr[XREG ? R : 1];
    if constexpr (XREG) load_x(xr);
    float* orow = p.out + (valid ? row : 0) * p.ldo;

    for (int e = e_lo; e < e_hi; ++e) {
      const int64_t it = gi * p.E + e;
      const uint2* t_scat;
      const float* t_cs;
      const uint32_t* t_bm;
      const uint32_t* t_gc;
      if constexpr (STAGED) {
        __syncthreads();  // buffer (it+1)&1 (read at it-1) is free
        if (threadIdx.x == 0 && it + 1 < total_it) issue(it + 1);
        mbar_wait(bar + (it & 1), (uint32_t)((it >> 1) & 1));
        const unsigned char* tb = tabs + (it & 1) * SLOT;
        t_scat = reinterpret_cast<const uint2*>(tb);
        t_cs = reinterpret_cast<const float*>(tb + N * 8);
        t_bm = reinterpret_cast<const uint32_t*>(tb + N * 12);
        t_gc = reinterpret_cast<const uint32_t*>(tb + N * 12 + bm_stride<C>() * 4);
      } else {
        t_scat = p.scat + (int64_t)(p.e0 + e) * N;
        t_cs = p.cs + (int64_t)(p.e0 + e) * N;
        t_bm = p.bmask + (int64_t)(p.e0 + e) * bm_stride<C>();
        t_gc = p.gcol + (int64_t)(p.e0 + e) * (N / 4);
      }

      float v[R];
      if constexpr (!XREG) load_x(v);
      // ---- x * B (sign XOR, exact)
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const uint32_t bits = t_bm[w * T + tid];
#pragma unroll
        for (int q = 0; q < 32 && 32 * w + q < R; ++q) {
          const float xv = XREG ? xr[(32 * w + q) % (XREG ? R : 1)] : v[32 * w + q];
          v[32 * w + q] = __uint_as_float(__float_as_uint(xv) ^ (((bits >> q) & 1u) << 31));
        }
      }
      // ---- H (first)
      butterflies<R, C::PL, C::PL>(v);
      middle_rounds<C, 0, C::PL>(s, tid, gid, v);
      // ---- Pi and G.  Tables read through L1/L2 (n = 16384): 16-bit slot
      // offsets (eight per 16-byte load), then G from a gather-layout table
      // after the gather (y[p] = z1[perm[p]] * g[p]).  Staged tables: one
      // scatter of z1[j] * g[perm^-1[j]] (the same fp32 product), table loads
      // batched ahead of the stores (the compiler cannot hoist a shared load
      // above a shared store to an unknown address by itself).
      constexpr bool COMPACT = !STAGED && ff_colored<C>();
      if constexpr (COMPACT) {
        const uint4* t_so = reinterpret_cast<const uint4*>(p.soff + (int64_t)(p.e0 + e) * N);
#pragma unroll
        for (int k0 = 0; k0 < R; k0 += 8) {
          const uint4 o = __ldg(t_so + (k0 / 8) * T + tid);
          const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float*>(reinterpret_cast<char*>(s) + ((ow[q / 2] >> (16 * (q % 2))) & 0xffffu)) =
                v[k0 + q];
        }
      } else {
#pragma unroll
        for (int k0 = 0; k0 < R; k0 += 8) {
          uint2 a[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) a[q] = t_scat[(k0 + q) * T + tid];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float*>(reinterpret_cast<char*>(s) + a[q].x) =
                v[k0 + q] * __uint_as_float(a[q].y);
        }
      }
      group_sync<T>(gid);
      if constexpr (ff_colored<C>()) {
        // gather group (warp w, register k) occupies words 32*(w*R + k) + colour
        const char* gb = reinterpret_cast<const char*>(s) + (tid / 32) * (R * 128);
        const float4* t_g4 = reinterpret_cast<const float4*>(p.ggath + (int64_t)(p.e0 + e) * N);
#pragma unroll
        for (int k4 = 0; k4 < R / 4; ++k4) {
          const uint32_t cw = t_gc[k4 * T + tid];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            v[4 * k4 + q] = *reinterpret_cast<const float*>(gb + (4 * k4 + q) * 128 + ((cw >> (8 * q)) & 0xffu));
          if constexpr (COMPACT) {
            const float4 g4 = __ldg(t_g4 + k4 * T + tid);
            mul_pk(v[4 * k4], v[4 * k4 + 1], g4.x, g4.y);
            mul_pk(v[4 * k4 + 2], v[4 * k4 + 3], g4.z, g4.w);
          }
        }
      } else {
        lds_layout<R, P0>(s, thread_part<C::FULL, P0>(tid), v);
      }
      group_sync<T>(gid);
      // ---- H (second), ending in layout L
      middle_rounds_then_L<C, 0, R>(s, tid, gid, v);
      butterflies<R, C::PL, C::PL>(v);
      // ---- C * scale, feature epilogue.  Output pointers are formed once per
      // block (per-j offsets are compile-time), the math runs unconditionally
      // and only the stores are predicated on the row being valid.
      float* const ob = orow + (int64_t)e * N + 4 * (int)tid;
      float* const obs = ob + p.D;
      const float* const csb = t_cs + 4 * (int)tid;
#pragma unroll
      for (int j = 0; j < R / 4; ++j) {
        const float4 c4 = *reinterpret_cast<const float4*>(csb + j * 4 * T);
        float z[4] = {v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]};
        const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
        mul_pk(z[0], z[1], cc[0], cc[1]);
        mul_pk(z[2], z[3], cc[2], cc[3]);
        if constexpr (!FOLD) {
          mul_pk(z[0], z[1], p.scale, p.scale);
          mul_pk(z[2], z[3], p.scale, p.scale);
        }
        if constexpr (FEAT) {
          float sn[4], cn[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) sincos_fast(z[c], sn[c], cn[c]);
          mul_pk(sn[0], sn[1], p.norm, p.norm);
          mul_pk(sn[2], sn[3], p.norm, p.norm);
          mul_pk(cn[0], cn[1], p.norm, p.norm);
          mul_pk(cn[2], cn[3], p.norm, p.norm);
          if (valid) {
            *reinterpret_cast<float4*>(ob + j * 4 * T) = make_float4(cn[0], cn[1], cn[2], cn[3]);
            *reinterpret_cast<float4*>(obs + j * 4 * T) = make_float4(sn[0], sn[1], sn[2], sn[3]);
          }
        } else if (valid) {
          const float4 z4 = make_float4(z[0], z[1], z[2], z[3]);
          if (p.tile8)
            st_out(reinterpret_cast<float4*>(p.out + zt_offset(p.ldo, row, (ob + j * 4 * T) - orow)), z4);
          else st_out(reinterpret_cast<float4*>(ob + j * 4 * T), z4);
        }
      }
    }
  }
}

// x ^ (t & 0x80000000) in one LOP3.
__device__ __forceinline__ uint32_t xor_sign(uint32_t x, uint32_t t) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(r) : "r"(x), "r"(t), "n"(0x80000000u));
  return r;
}


// ---------------------------------------------------------------- two rows per thread
// n = 1024.  Each warp owns TWO rows; register k holds the pair (row0[i],
// row1[i]) of one index i, so every butterfly stage is a packed f32x2 add/sub
// (including the stage on the lowest register bit that the one-row kernel
// leaves scalar), every exchange moves both rows with one 8-byte access, and
// each table entry (16-bit scatter offset, g in the gather layout, gather
// colour, C*scale, sign mask) is loaded once for two rows.  x is re-read per
// block (TMA-staged, L2-resident) instead of being held in registers.
// Exchanges use the 8-byte padding pad2 (conflict free per 16-lane phase for
// layouts L and P0); Pi uses 16-colour slots.
__host__ __device__ constexpr uint32_t pad2(uint32_t i) { return i + (i >> 4) + 4 * (i >> 7); }
constexpr int kPairRowFloat2 = 1116;  // pad2(1023) + 1, rounded to 16 bytes
#ifndef MCK_PAIR_WARPS
#define MCK_PAIR_WARPS 8
#endif
#ifndef MCK_PAIR_MINB
#define MCK_PAIR_MINB 2
#endif
constexpr int kPairWarps = MCK_PAIR_WARPS;
constexpr int kPairHdr = ((2 + kPairWarps) * 8 + 127) / 128 * 128;  // mbarriers, 128-byte aligned

template <int R, uint32_t P, uint32_t ACTIVE>
__device__ __forceinline__ void butterflies2(float2 (&v)[R]) {
#pragma unroll
  for (int a = 0; (1 << a) < R; ++a) {
    if (ACTIVE & deposit_bits(1u << a, P)) {
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (!(k & (1 << a))) bfly_pk(v[k].x, v[k].y, v[k | (1 << a)].x, v[k | (1 << a)].y);
    }
  }
}

template <int R, uint32_t P>
__device__ __forceinline__ void sts2(float2* s, uint32_t tpart, const float2 (&v)[R]) {
  float2* base = s + pad2(tpart);
#pragma unroll
  for (int k = 0; k < R; ++k) base[pad2(deposit_bits((uint32_t)k, P))] = v[k];
}

template <int R, uint32_t P>
__device__ __forceinline__ void lds2(const float2* s, uint32_t tpart, float2 (&v)[R]) {
  const float2* base = s + pad2(tpart);
#pragma unroll
  for (int k = 0; k < R; ++k) v[k] = base[pad2(deposit_bits((uint32_t)k, P))];
}

// two-row kernel table slot: soff u16[N] | ggath f32[N] | cs f32[N] | bmask | gcol u8[N]
template <class C>
constexpr int pair_tab_bytes() { return C::N * 11 + bm_stride<C>() * 4; }
template <class C>
constexpr int pair_tab_slot() { return (pair_tab_bytes<C>() + 127) & ~127; }
template <class C>
constexpr size_t ff_pair_smem_bytes() {
  return kPairHdr + 2 * (size_t)pair_tab_slot<C>() + (size_t)kPairWarps * kPairRowFloat2 * 8;
}

template <bool FEAT, bool FOLD, bool VEC>
__global__ void __launch_bounds__(kPairWarps * 32, MCK_PAIR_MINB) k_fastfood_pair(FFParams p) {
  using C = RowCfg<10, 5>;
  constexpr int R = C::R, T = C::T, N = C::N;
  constexpr int ROWS = 2 * kPairWarps;
  constexpr int SLOT = pair_tab_slot<C>();
  constexpr uint32_t PL = C::PL, P0 = C::mid_regs(0);
  static_assert(C::NMID == 1 && T == 32, "pair kernel layout");
  static_assert(2 * N * 4 <= kPairRowFloat2 * 8, "x staging fits the exchange buffer");
  extern __shared__ __align__(128) unsigned char ff_smem[];
  // header: table barriers [0,1], per-warp x barriers [2 .. 2+kPairWarps)
  uint64_t* bar = reinterpret_cast<uint64_t*>(ff_smem);
  unsigned char* tabs = ff_smem + kPairHdr;
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  uint64_t* xbar = bar + 2 + warp;
  float2* s = reinterpret_cast<float2*>(ff_smem + kPairHdr + 2 * SLOT) + warp * kPairRowFloat2;
  float* const xs = reinterpret_cast<float*>(s);  // x staging: row0 [0,N), row1 [N,2N)
  const uint32_t tp_l = thread_part<C::FULL, PL>(lane), tp_0 = thread_part<C::FULL, P0>(lane);

  // Work units (block e, row group of 16), block-major: u = e * groups + g.
  // Each CTA takes a contiguous, balanced range, so its factor tables change
  // at most a few times (x of a batch is L2-resident and re-read per block).
  const int64_t groups = (p.m + ROWS - 1) / ROWS;
  const int64_t units = groups * p.E;
  const int64_t u_lo = units * blockIdx.x / gridDim.x, u_hi = units * (blockIdx.x + 1) / gridDim.x;
  if (u_lo >= u_hi) {
    pdl_wait();
    pdl_trigger();
    return;
  }
  const int e_first = (int)(u_lo / groups), e_last = (int)((u_hi - 1) / groups);
  auto issue_tab = [&](int e, int slot) {  // thread 0 only
    const int eg = p.e0 + e;
    unsigned char* dst = tabs + slot * SLOT;
    uint64_t* b = bar + slot;
    // slot: soff u16[N] | ggath f32[N] | cs f32[N] | bmask | gcol u8[N]
    mbar_expect_tx(b, pair_tab_bytes<C>());
    bulk_g2s(dst, p.soff + (int64_t)eg * N, N * 2, b);
    bulk_g2s(dst + N * 2, p.ggath + (int64_t)eg * N, N * 4, b);
    bulk_g2s(dst + N * 6, p.cs + (int64_t)eg * N, N * 4, b);
    bulk_g2s(dst + N * 10, p.bmask + (int64_t)eg * bm_stride<C>(), bm_stride<C>() * 4, b);
    bulk_g2s(dst + N * 10 + bm_stride<C>() * 4, p.gcol + (int64_t)eg * (N / 4), N, b);
  };
  auto src_row = [&](int64_t r) -> const float* {
    return p.x + (p.rows ? (int64_t)p.rows[r] : r) * p.ldx;
  };
  // x rows of unit u -> this warp's staging area (lane 0 only; VEC: 16-byte rows)
  auto issue_x = [&](int64_t gx) {  // gx: row group of the unit
    const int64_t r0 = gx * ROWS + 2 * warp;
    const uint32_t rb = (uint32_t)p.d * 4u;
    const uint32_t bytes = (r0 < p.m ? rb : 0u) + (r0 + 1 < p.m ? rb : 0u);
    mbar_expect_tx(xbar, bytes);
    if (r0 < p.m) bulk_g2s(xs, src_row(r0), rb, xbar);
    if (r0 + 1 < p.m) bulk_g2s(xs + N, src_row(r0 + 1), rb, xbar);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 + kPairWarps; ++i) mbar_init(bar + i, 1);
    fence_mbar_init();
  }
  __syncthreads();
  // the factor tables are constant for the launch: their copies overlap the
  // predecessor's tail; x and the output wait for it (pdl_wait)
  if (threadIdx.x == 0) {
    issue_tab(e_first, 0);
    if (e_last > e_first) issue_tab(e_first + 1, 1);
  }
  pdl_wait();
  pdl_trigger();
  if constexpr (VEC) {
    if (lane == 0) issue_x(u_lo % groups);
  }

  int ti = -1, e_cur = -1;
  uint32_t xph = 0, bits = 0;
  const uint4* t_soff = nullptr;
  const float4* t_gg = nullptr;
  const float* t_cs = nullptr;
  const uint32_t* t_gc = nullptr;
  int e = e_first;
  int64_t g = u_lo - (int64_t)e_first * groups;  // unit u = e * groups + g, advanced incrementally
  for (int64_t u = u_lo; u < u_hi; ++u, ++g) {
    if (g == groups) {
      g = 0;
      ++e;
    }
    const int64_t row0 = g * ROWS + 2 * warp;
    const bool v0 = row0 < p.m, v1 = row0 + 1 < p.m;
    if (e != e_cur) {  // uniform across the CTA
      if (ti >= 0) {
        __syncthreads();  // every warp is done with slot ti&1 ... and slot (ti+1)&1 is free
        if (threadIdx.x == 0 && e + 1 <= e_last) issue_tab(e + 1, ti & 1);
      }
      ++ti;
      e_cur = e;
      mbar_wait(bar + (ti & 1), (uint32_t)((ti >> 1) & 1));
      const unsigned char* tb = tabs + (ti & 1) * SLOT;
      t_soff = reinterpret_cast<const uint4*>(tb);
      t_gg = reinterpret_cast<const float4*>(tb + N * 2);
      t_cs = reinterpret_cast<const float*>(tb + N * 6);
      bits = reinterpret_cast<const uint32_t*>(tb + N * 10)[lane];
      t_gc = reinterpret_cast<const uint32_t*>(tb + N * 10 + bm_stride<C>() * 4);
    }
    float* const orow0 = p.out + (v0 ? row0 : 0) * p.ldo;
    float* const orow1 = p.out + (v1 ? row0 + 1 : 0) * p.ldo;
    {
      // ---- x (layout L, both rows) * B as a sign XOR
      float2 v[R];
      if constexpr (VEC) {
        mbar_wait(xbar, xph);
        xph ^= 1u;
      }
#pragma unroll
      for (int j = 0; j < R / 4; ++j) {
        const int i0 = 4 * (int)lane + j * 4 * T;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        if constexpr (VEC) {
          if (v0 && i0 < p.d) a = *reinterpret_cast<const float4*>(xs + i0);
          if (v1 && i0 < p.d) b = *reinterpret_cast<const float4*>(xs + N + i0);
        } else {
          const float* xp0 = src_row(v0 ? row0 : 0);
          const float* xp1 = src_row(v1 ? row0 + 1 : 0);
          a.x = (v0 && i0 < p.d) ? __ldg(xp0 + i0) : 0.f;
          a.y = (v0 && i0 + 1 < p.d) ? __ldg(xp0 + i0 + 1) : 0.f;
          a.z = (v0 && i0 + 2 < p.d) ? __ldg(xp0 + i0 + 2) : 0.f;
          a.w = (v0 && i0 + 3 < p.d) ? __ldg(xp0 + i0 + 3) : 0.f;
          b.x = (v1 && i0 < p.d) ? __ldg(xp1 + i0) : 0.f;
          b.y = (v1 && i0 + 1 < p.d) ? __ldg(xp1 + i0 + 1) : 0.f;
          b.z = (v1 && i0 + 2 < p.d) ? __ldg(xp1 + i0 + 2) : 0.f;
          b.w = (v1 && i0 + 3 < p.d) ? __ldg(xp1 + i0 + 3) : 0.f;
        }
        const float xa[4] = {a.x, a.y, a.z, a.w}, xb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          // bit (4j+c) of the mask moved to bit 31, XORed into both rows
          const uint32_t t = bits << (31 - (4 * j + c));
          v[4 * j + c] = make_float2(__uint_as_float(xor_sign(__float_as_uint(xa[c]), t)),
                                     __uint_as_float(xor_sign(__float_as_uint(xb[c]), t)));
        }
      }
      if constexpr (VEC) __syncwarp();  // staging reads done before the exchange writes

      // ---- H (first): layout L rounds, exchange, round P0
      butterflies2<R, PL, PL>(v);
      sts2<R, PL>(s, tp_l, v);
      __syncwarp();
      lds2<R, P0>(s, tp_0, v);
      __syncwarp();
      butterflies2<R, P0, P0>(v);
      // ---- Pi and G: scatter (coloured 8-byte slots, 16-bit byte offsets),
      // gather, then y[p] = z1[perm[p]] * g[p] (the reference's fp32 product)
#pragma unroll
      for (int k0 = 0; k0 < R; k0 += 8) {
        const uint4 o = t_soff[(k0 / 8) * T + lane];
        const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float2*>(reinterpret_cast<char*>(s) + ((ow[q / 2] >> (16 * (q % 2))) & 0xffffu)) =
              v[k0 + q];
      }
      __syncwarp();
      {
        // gather group (register k, half-warp h) occupies 8-byte slots 16*(2k+h) + colour
        const char* gb = reinterpret_cast<const char*>(s) + 128 * (lane >> 4);
#pragma unroll
        for (int k4 = 0; k4 < R / 4; ++k4) {
          const uint32_t cw = t_gc[k4 * T + lane];
          const float4 g4 = t_gg[k4 * T + lane];
          const float gg[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float2 w = *reinterpret_cast<const float2*>(gb + (4 * k4 + q) * 256 + ((cw >> (8 * q)) & 0xffu));
            mul_pk(w.x, w.y, gg[q], gg[q]);
            v[4 * k4 + q] = w;
          }
        }
      }
      __syncwarp();
      // ---- H (second): round P0, exchange, layout L rounds
      butterflies2<R, P0, P0>(v);
      sts2<R, P0>(s, tp_0, v);
      __syncwarp();
      lds2<R, PL>(s, tp_l, v);
      if constexpr (VEC) fence_proxy_async_smem();  // exchange reads before the next x copy
      __syncwarp();
      if constexpr (VEC) {
        // next unit's x streams into the (now free) exchange buffer during the epilogue
        if (lane == 0 && u + 1 < u_hi) issue_x(g + 1 == groups ? 0 : g + 1);
      }
      butterflies2<R, PL, PL>(v);
      // ---- C * scale and the feature epilogue, both rows
      float* const ob0 = orow0 + (int64_t)e * N + 4 * (int)lane;
      float* const ob1 = orow1 + (int64_t)e * N + 4 * (int)lane;
      const float* const csb = t_cs + 4 * (int)lane;
#pragma unroll
      for (int j = 0; j < R / 4; ++j) {
        const float4 c4 = *reinterpret_cast<const float4*>(csb + j * 4 * T);
        const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
        float2 z[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          z[c] = v[4 * j + c];
          mul_pk(z[c].x, z[c].y, cc[c], cc[c]);
          if constexpr (!FOLD) mul_pk(z[c].x, z[c].y, p.scale, p.scale);
        }
        if constexpr (FEAT) {
          // sin/cos per value, then the 1/sqrt(D) multiplies paired in store
          // order so the products land in the 16-byte store registers
          float c0[4], s0[4], c1[4], s1[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            sincos_fast(z[c].x, s0[c], c0[c]);
            sincos_fast(z[c].y, s1[c], c1[c]);
          }
#pragma unroll
          for (int c = 0; c < 4; c += 2) {
            mul_pk(c0[c], c0[c + 1], p.norm, p.norm);
            mul_pk(s0[c], s0[c + 1], p.norm, p.norm);
            mul_pk(c1[c], c1[c + 1], p.norm, p.norm);
            mul_pk(s1[c], s1[c + 1], p.norm, p.norm);
          }
          if (v0) {
            st_out(reinterpret_cast<float4*>(ob0 + j * 4 * T), make_float4(c0[0], c0[1], c0[2], c0[3]));
            st_out(reinterpret_cast<float4*>(ob0 + p.D + j * 4 * T), make_float4(s0[0], s0[1], s0[2], s0[3]));
          }
          if (v1) {
            st_out(reinterpret_cast<float4*>(ob1 + j * 4 * T), make_float4(c1[0], c1[1], c1[2], c1[3]));
            st_out(reinterpret_cast<float4*>(ob1 + p.D + j * 4 * T), make_float4(s1[0], s1[1], s1[2], s1[3]));
          }
        } else {
          const float4 a = make_float4(z[0].x, z[1].x, z[2].x, z[3].x);
          const float4 b = make_float4(z[0].y, z[1].y, z[2].y, z[3].y);
          if (p.tile8) {
            const int64_t col = (ob0 + j * 4 * T) - orow0;
            if (v0) *reinterpret_cast<float4*>(p.out + zt_offset(p.ldo, row0, col)) = a;
            if (v1) *reinterpret_cast<float4*>(p.out + zt_offset(p.ldo, row0 + 1, col)) = b;
          } else {
            if (v0) *reinterpret_cast<float4*>(ob0 + j * 4 * T) = a;
            if (v1) *reinterpret_cast<float4*>(ob1 + j * 4 * T) = b;
          }
        }
      }
    }
  }
}

template <bool FEAT, bool FOLD, bool VEC>
int launch_ff_pair(const FFParams& p, cudaStream_t st) {
  using C = RowCfg<10, 5>;
  constexpr int ROWS = 2 * kPairWarps;
  const size_t smem = ff_pair_smem_bytes<C>();
  auto kern = k_fastfood_pair<FEAT, FOLD, VEC>;
  static PerDevice pd;
  const DeviceSlot* ds = nullptr;
  MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot& s) {
    MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem), "fastfood pair smem"));
    MCK_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s.occ, kern, kPairWarps * 32, smem),
                       "occupancy"));
    if (s.occ < 1) s.occ = 1;
    return MCK_OK;
  }));
  const int64_t items = (p.m + ROWS - 1) / ROWS * p.E;
  int64_t grid = (int64_t)ds->sms * ds->occ;
  if (grid > items) grid = items;
  {
    // small batches (<= 3 rounds, e.g. c0's 504 items on 296 CTAs): the fewest
    // CTAs that finish in the same number of rounds -- equal work per CTA, and
    // the slots left over go to the next independent launch (c0 steady state
    // 13.95 -> 13.67 us per batch; at c2's 14 rounds the full grid is faster)
    const int64_t rounds = (items + grid - 1) / grid;
    if (rounds <= 3) grid = (items + rounds - 1) / rounds;
  }
  return launch_pdl(kern, dim3((unsigned)grid), dim3(kPairWarps * 32), smem, st, "k_fastfood_pair", p);
}

// ---------------------------------------------------------------- parity variant
// One CTA per (row, block); follows fastfood.py:189-197 operation by operation.
__device__ void parity_wht_smem(float* a, float* tmp, int n) {
  const int base = n < 256 ? n : 256;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int c0 = j - (j % base), jj = j % base;
    float acc = 0.0f;
    for (int k = 0; k < base; ++k) {
      const float xk = a[c0 + k];
      acc = (__popc((unsigned)(k & jj)) & 1) ? acc - xk : acc + xk;
    }
    tmp[j] = acc;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) a[j] = tmp[j];
  __syncthreads();
  for (int h = base; h < n; h <<= 1) {
    for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
      const int grp = t / h, off = t % h;
      float* pa = a + grp * 2 * h + off;
      float* pb = pa + h;
      const float sum = *pa + *pb;
      *pa = sum;
      *pb = sum - 2.0f * *pb;
    }
    __syncthreads();
  }
}

__global__ void k_fastfood_parity(const float* x, int64_t ldx, int32_t d, const int32_t* rows,
                                  int64_t n, const float* b, const int32_t* perm, const float* g,
                                  const float* c, float scale, int feat, float norm, float* out,
                                  int64_t ldo, int64_t D) {
  extern __shared__ float pz[];
  float* a = pz;
  float* tmp = pz + n;
  const int64_t row = blockIdx.x;
  const int e = blockIdx.y;
  const int64_t src = rows ? (int64_t)rows[row] : row;
  const float* xp = x + src * ldx;
  const int64_t off = (int64_t)e * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = (i < d ? xp[i] : 0.0f) * b[off + i];
  __syncthreads();
  parity_wht_smem(a, tmp, (int)n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) tmp[i] = a[perm[off + i]];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = tmp[i] * g[off + i];
  __syncthreads();
  parity_wht_smem(a, tmp, (int)n);
  float* o = out + row * ldo + off;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float z = (a[i] * c[off + i]) * scale;
    if (feat) {
      o[i] = cosf(z) * norm;
      o[i + D] = sinf(z) * norm;
    } else {
      o[i] = z;
    }
  }
}

// ---------------------------------------------------------------- coloured Pi
// Host side (one-time setup): slots of the edge-coloured permutation.  H1
// leaves y[j] in (thread t, register k) of layout PM -> scatter group
// S = (t/32)*R + k; position p = perm^-1[j] is read by (t', k') of layout P0
// -> gather group G = (t'/32)*R + k'.  Slot = 32*G + colour(j).
template <class C, bool PAIR>
int color_tables(const TablesView& tv, cudaStream_t st) {
  // PAIR: two rows per thread, 8-byte elements, conflicts per 16-lane phase
  constexpr int R = C::R, T = C::T, N = C::N;
  constexpr int GW = PAIR ? 16 : 32, ES = PAIR ? 8 : 4, LEVELS = PAIR ? 4 : 5, M = N / GW;
  constexpr uint32_t PM = last_mid_regs<C>(), P0 = C::mid_regs(0);
  auto group = [](int t, int k) { return PAIR ? k * (T / GW) + t / GW : (t / 32) * R + k; };
  const int E = tv.E;
  std::vector<int32_t> pinv((size_t)E * N);
  std::vector<uint32_t> gbits((size_t)E * N);
  MCK_TRY(check_cuda(cudaMemcpyAsync(pinv.data(), tv.perminv, pinv.size() * 4,
                                     cudaMemcpyDeviceToHost, st), "perminv D2H"));
  MCK_TRY(check_cuda(cudaMemcpyAsync(gbits.data(), tv.g, gbits.size() * 4,
                                     cudaMemcpyDeviceToHost, st), "g D2H"));
  MCK_TRY(check_cuda(cudaStreamSynchronize(st), "colour tables sync"));
  std::vector<int32_t> sgrp(N), spos(N), ggrp(N), gpos(N);
  for (int t = 0; t < T; ++t)
    for (int k = 0; k < R; ++k) {
      const uint32_t j = deposit_bits((uint32_t)t, C::FULL & ~PM) | deposit_bits((uint32_t)k, PM);
      sgrp[j] = group(t, k);
      spos[j] = k * T + t;
      const uint32_t p = deposit_bits((uint32_t)t, C::FULL & ~P0) | deposit_bits((uint32_t)k, P0);
      ggrp[p] = group(t, k);
      gpos[p] = k * T + t;
    }
  std::vector<uint2> scat((size_t)E * N);
  std::vector<uint32_t> gcol((size_t)E * N / 4, 0u);
  static_assert(R % 8 == 0, "coloured layouts hold 32 registers");
  std::vector<uint16_t> soff((size_t)E * N);
  std::vector<float> ggath((size_t)E * N);
  std::vector<int32_t> left(N), right(N);
  std::vector<uint8_t> col(N);
  for (int e = 0; e < E; ++e) {
    const int32_t* pi = pinv.data() + (size_t)e * N;
    for (int j = 0; j < N; ++j) {
      left[j] = sgrp[j];
      right[j] = ggrp[pi[j]];
    }
    if (!edge_color_pow2(M, LEVELS, N, left.data(), right.data(), col.data()))
      return fail_value("internal: permutation edge colouring failed (block %d)", e);
    for (int j = 0; j < N; ++j) {
      const int32_t p = pi[j];
      scat[(size_t)e * N + spos[j]] =
          make_uint2((uint32_t)ES * ((uint32_t)GW * (uint32_t)ggrp[p] + col[j]), gbits[(size_t)e * N + p]);
      const int k = gpos[p] / T, t = gpos[p] % T;
      gcol[(size_t)e * (N / 4) + (k / 4) * T + t] |= ((uint32_t)ES * col[j]) << (8 * (k % 4));
      {
        const uint32_t off = (uint32_t)ES * ((uint32_t)GW * (uint32_t)ggrp[p] + col[j]);
        if (off > 0xffffu) return fail_value("internal: scatter offset exceeds 16 bits");
        const int sk = spos[j] / T, st_ = spos[j] % T;
        soff[(size_t)e * N + ((size_t)(sk / 8) * T + st_) * 8 + sk % 8] = (uint16_t)off;
        uint32_t gb = gbits[(size_t)e * N + p];
        float gf;
        memcpy(&gf, &gb, 4);
        ggath[(size_t)e * N + ((size_t)(k / 4) * T + t) * 4 + k % 4] = gf;
      }
    }
  }
  MCK_TRY(check_cuda(cudaMemcpyAsync(tv.soff, soff.data(), soff.size() * 2,
                                     cudaMemcpyHostToDevice, st), "soff H2D"));
  MCK_TRY(check_cuda(cudaMemcpyAsync(tv.ggath, ggath.data(), ggath.size() * 4,
                                     cudaMemcpyHostToDevice, st), "ggath H2D"));
  MCK_TRY(check_cuda(cudaMemcpyAsync(tv.scat, scat.data(), scat.size() * 8,
                                     cudaMemcpyHostToDevice, st), "scat H2D"));
  MCK_TRY(check_cuda(cudaMemcpyAsync(tv.gcol, gcol.data(), gcol.size() * 4,
                                     cudaMemcpyHostToDevice, st), "gcol H2D"));
  return check_cuda(cudaStreamSynchronize(st), "colour tables upload");
}

// ---------------------------------------------------------------- dispatch
template <class C>
int prepare_cfg(const TablesView& tv, cudaStream_t st) {
  const int64_t total = (int64_t)tv.E * C::R * C::T;
  unsigned grid = (unsigned)((total + 255) / 256);
  if (grid > 148 * 32) grid = 148 * 32;
  k_prepare<C><<<grid, 256, 0, st>>>(tv.b, tv.g, tv.perminv, tv.E, tv.bmask, tv.scat);
  MCK_TRY(check_launch("k_prepare"));
  if constexpr (ff_colored<C>()) return color_tables<C, ff_pair<C>()>(tv, st);
  return MCK_OK;
}

int prepare_tables(const TablesView& tv, float scale, int fold, cudaStream_t st, bool validate) {
  const int64_t total = tv.n * tv.E;
  unsigned grid = (unsigned)((total + 255) / 256);
  if (grid > 148 * 32) grid = 148 * 32;
  MCK_TRY(check_cuda(cudaMemsetAsync(tv.flag, 0, 4, st), "flag reset"));
  k_perminv<<<grid, 256, 0, st>>>(tv.perm, tv.n, tv.E, tv.perminv, tv.flag);
  MCK_TRY(check_launch("k_perminv"));
  if (validate) {
    k_perm_check<<<grid, 256, 0, st>>>(tv.perm, tv.perminv, tv.n, tv.E, tv.flag);
    MCK_TRY(check_launch("k_perm_check"));
    int32_t h = 0;
    MCK_TRY(check_cuda(cudaMemcpyAsync(&h, tv.flag, 4, cudaMemcpyDeviceToHost, st), "flag copy"));
    MCK_TRY(check_cuda(cudaStreamSynchronize(st), "flag sync"));
    if (h) return fail_value("permutation is not a bijection on {0..n-1}");
  }
  k_cscale<<<grid, 256, 0, st>>>(tv.c, total, scale, fold, tv.cs);
  MCK_TRY(check_launch("k_cscale"));
  int logn = 0;
  while ((int64_t(1) << logn) < tv.n) ++logn;
  switch (logn) {
    case 3: return prepare_cfg<RowCfg<3, 2>>(tv, st);
    case 4: return prepare_cfg<RowCfg<4, 3>>(tv, st);
    case 5: return prepare_cfg<RowCfg<5, 4>>(tv, st);
    case 6: return prepare_cfg<RowCfg<6, 4>>(tv, st);
    case 7: return prepare_cfg<RowCfg<7, 5>>(tv, st);
    case 8: return prepare_cfg<RowCfg<8, 5>>(tv, st);
    case 9: return prepare_cfg<RowCfg<9, 5>>(tv, st);
    case 10: return prepare_cfg<RowCfg<10, 5>>(tv, st);
    case 11: return prepare_cfg<RowCfg<11, 5>>(tv, st);
    case 12: return prepare_cfg<RowCfg<12, 5>>(tv, st);
    case 13: return prepare_cfg<RowCfg<13, 5>>(tv, st);
    case 14: return prepare_cfg<RowCfg<14, 5>>(tv, st);
    default: return MCK_OK;  // fused kernel not available; parity path only
  }
}

template <class C, bool FEAT, bool FOLD, bool VEC>
int launch_ff(const FFParams& p, cudaStream_t st) {
  constexpr int ROWS = ff_rows_per_cta<C>();
  const size_t smem = ff_smem_bytes<C>();
  auto kern = k_fastfood<C, FEAT, FOLD, VEC>;
  static PerDevice pd;  // per instantiation, per device
  const DeviceSlot* ds = nullptr;
  MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot& s) {
    MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem), "fastfood smem"));
    MCK_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s.occ, kern, C::T * ROWS, smem),
                       "occupancy"));
    if (s.occ < 1) s.occ = 1;
    return MCK_OK;
  }));
  const int64_t groups = (p.m + ROWS - 1) / ROWS;
  const int64_t work = ff_xreg<C>() ? groups : groups * p.E;
  int64_t grid = (int64_t)ds->sms * ds->occ;
  if (grid > work) grid = work;
  return launch_pdl(kern, dim3((unsigned)grid), dim3(C::T * ROWS), smem, st, "k_fastfood", p);
}

template <class C>
int launch_ff_cfg(const FFParams& p, bool feat, bool fold, bool vec, cudaStream_t st) {
  if constexpr (ff_pair<C>()) {
    if (feat) {
      if (fold) return vec ? launch_ff_pair<true, true, true>(p, st) : launch_ff_pair<true, true, false>(p, st);
      return vec ? launch_ff_pair<true, false, true>(p, st) : launch_ff_pair<true, false, false>(p, st);
    }
    if (fold) return vec ? launch_ff_pair<false, true, true>(p, st) : launch_ff_pair<false, true, false>(p, st);
    return vec ? launch_ff_pair<false, false, true>(p, st) : launch_ff_pair<false, false, false>(p, st);
  } else {
  if (feat) {
    if (fold) return vec ? launch_ff<C, true, true, true>(p, st) : launch_ff<C, true, true, false>(p, st);
    return vec ? launch_ff<C, true, false, true>(p, st) : launch_ff<C, true, false, false>(p, st);
  }
  if (fold) return vec ? launch_ff<C, false, true, true>(p, st) : launch_ff<C, false, true, false>(p, st);
  return vec ? launch_ff<C, false, false, true>(p, st) : launch_ff<C, false, false, false>(p, st);
  }
}

int launch_by_logn(const FFParams& p, int logn, bool feat, bool fold, cudaStream_t st);
template <class V> int fwht_fast(V*, int64_t, int64_t, cudaStream_t);
int fwht_parity(float*, int64_t, int64_t, cudaStream_t);

// ---------------------------------------------------------------- n > 16384
// padded_dim 2^15 .. 2^20: the row no longer fits one SM's registers and
// shared memory next to its tables, so each block runs as the reference
// writes it (fastfood.py:189-197), one pass per step over a chunk of rows in
// scratch (stream-ordered allocation, <= 256 MiB per buffer):
//   k_lg_load   v = pad(x) * B                  (exact sign flip)
//   H           the batched FWHT (cluster / two-phase kernels, K1)
//   k_lg_gather u = v[:, perm] * G
//   H
//   k_lg_epi    z = (u * C) * scale; z or [cos z | sin z] * norm into out
// Same per-element fp32 operations as the fused kernels; the parity variant
// uses the reference-order FWHT (bit-exact z).
__global__ void k_lg_load(const float* __restrict__ x, int64_t ldx, int32_t d,
                          const int32_t* __restrict__ rows, int64_t r0, int64_t nr, int64_t n,
                          const float* __restrict__ b, float* __restrict__ v) {
  const int64_t total = nr * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / n, i = t - r * n;
    const int64_t row = rows ? (int64_t)rows[r0 + r] : r0 + r;
    v[t] = i < d ? x[row * ldx + i] * b[i] : 0.f;
  }
}

__global__ void k_lg_gather(const float* __restrict__ v, int64_t nr, int64_t n,
                            const int32_t* __restrict__ perm, const float* __restrict__ g,
                            float* __restrict__ u) {
  const int64_t total = nr * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / n, i = t - r * n;
    u[t] = v[r * n + perm[i]] * g[i];
  }
}

__global__ void k_lg_epi(const float* __restrict__ u, int64_t nr, int64_t n, const float* __restrict__ c,
                         float scale, int feat, float norm, float* __restrict__ out, int64_t ldo,
                         int64_t col, int64_t D) {
  const int64_t total = nr * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / n, i = t - r * n;
    const float z = (u[t] * c[i]) * scale;
    float* o = out + r * ldo + col + i;
    if (feat) {
      float sn, cs;
      sincos_fast(z, sn, cs);
      o[0] = cs * norm;
      o[D] = sn * norm;
    } else {
      o[0] = z;
    }
  }
}

static int fastfood_large(const TablesView& tv, int32_t d, const float* x, int64_t m, int64_t ldx,
                          const int32_t* rows, bool feat, float scale, float norm, float* out,
                          int64_t ldo, int variant, cudaStream_t st) {
  const int64_t n = tv.n, D = n * tv.E;
  const int64_t chunk = (int64_t(1) << 26) / n < m ? (int64_t(1) << 26) / n : m;  // rows per pass
  float* v = nullptr;
  MCK_TRY(check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&v), (size_t)2 * chunk * n * 4, st),
                     "large-n scratch"));
  float* u = v + chunk * n;
  int rc = MCK_OK;
  const unsigned grid = 148 * 8;
  for (int64_t r0 = 0; r0 < m && rc == MCK_OK; r0 += chunk) {
    const int64_t nr = m - r0 < chunk ? m - r0 : chunk;
    for (int32_t e = 0; e < tv.E && rc == MCK_OK; ++e) {
      const int64_t eo = (int64_t)e * n;
      k_lg_load<<<grid, 256, 0, st>>>(x, ldx, d, rows, r0, nr, n, tv.b + eo, v);
      if ((rc = check_launch("k_lg_load")) != MCK_OK) break;
      rc = variant == MCK_WHT_PARITY ? fwht_parity(v, nr, n, st) : fwht_fast<float>(v, nr, n, st);
      if (rc != MCK_OK) break;
      k_lg_gather<<<grid, 256, 0, st>>>(v, nr, n, tv.perm + eo, tv.g + eo, u);
      if ((rc = check_launch("k_lg_gather")) != MCK_OK) break;
      rc = variant == MCK_WHT_PARITY ? fwht_parity(u, nr, n, st) : fwht_fast<float>(u, nr, n, st);
      if (rc != MCK_OK) break;
      k_lg_epi<<<grid, 256, 0, st>>>(u, nr, n, tv.c + eo, scale, feat ? 1 : 0, norm, out + r0 * ldo, ldo,
                                     eo, D);
      rc = check_launch("k_lg_epi");
    }
  }
  const int rf = check_cuda(cudaFreeAsync(v, st), "large-n scratch free");
  return rc != MCK_OK ? rc : rf;
}

int fastfood_run(const TablesView& tv, int32_t d, double sigma, const float* x, int64_t m,
                 int64_t ldx, const int32_t* rows, bool feat, bool normalize, float* out,
                 int64_t ldo, int variant, cudaStream_t st) {
  if (m == 0) return MCK_OK;
  const int64_t n = tv.n;
  const int64_t D = n * tv.E;
  // fastfood.py:186 scale = float32(1/(sigma*sqrt(n))); :225 float32(1/sqrt(D))
  const double scale_d = 1.0 / (sigma * sqrt((double)n));
  const float scale = (float)scale_d;
  const float norm = normalize ? (float)(1.0 / sqrt((double)D)) : 1.0f;
  int ex = 0;
  const bool fold = frexpf(scale, &ex) == 0.5f;  // power of two
  int logn = 0;
  while ((int64_t(1) << logn) < n) ++logn;
  if (logn > 14)
    return fastfood_large(tv, d, x, m, ldx, rows, feat, scale, norm, out, ldo, variant, st);
  if (variant == MCK_WHT_PARITY || logn < 3) {
    const size_t smem = (size_t)2 * n * sizeof(float);
    if (smem > 200 * 1024) return fail_value("parity expansion supports padded_dim <= 16384");
    if (smem > 48 * 1024)
      MCK_TRY(check_cuda(cudaFuncSetAttribute(k_fastfood_parity,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem), "parity smem"));
    if (variant != MCK_WHT_PARITY && logn > 14)
      return fail_value("padded_dim %lld exceeds the fused kernel's maximum 16384", (long long)n);
    for (int64_t r0 = 0; r0 < m; r0 += 65535) {
      const int64_t nr = m - r0 < 65535 ? m - r0 : 65535;
      dim3 grid((unsigned)nr, (unsigned)tv.E);
      k_fastfood_parity<<<grid, n < 256 ? (unsigned)((n + 31) / 32 * 32) : 256u, smem, st>>>(
          rows ? x : x + r0 * ldx, ldx, d, rows ? rows + r0 : nullptr, n, tv.b, tv.perm, tv.g,
          tv.c, scale, feat ? 1 : 0, norm, out + r0 * ldo, ldo, D);
      MCK_TRY(check_launch("k_fastfood_parity"));
    }
    return MCK_OK;
  }
  FFParams p{};
  p.x = x; p.m = m; p.ldx = ldx; p.d = d; p.rows = rows;
  p.bmask = tv.bmask; p.scat = tv.scat; p.cs = tv.cs; p.gcol = tv.gcol;
  p.soff = tv.soff; p.ggath = tv.ggath;
  p.scale = scale; p.norm = norm; p.out = out; p.ldo = ldo; p.E = tv.E; p.D = D;
  return launch_by_logn(p, logn, feat, fold, st);
}

// z of blocks e0 .. e0+ecount-1 only (columns 0 .. ecount*n of z): the
// producer half of the fused config-4 path (fused_head.cu).
int fastfood_z_blocks(const TablesView& tv, int32_t d, double sigma, const float* x, int64_t m,
                      int64_t ldx, const int32_t* rows, int32_t e0, int32_t ecount, float* z,
                      int64_t ldz, bool tile8, cudaStream_t st) {
  if (m == 0) return MCK_OK;
  const int64_t n = tv.n;
  const float scale = (float)(1.0 / (sigma * sqrt((double)n)));
  int ex = 0;
  const bool fold = frexpf(scale, &ex) == 0.5f;
  int logn = 0;
  while ((int64_t(1) << logn) < n) ++logn;
  if (logn < 3 || logn > 14) return fail_value("fused path supports padded_dim 8..16384");
  if (e0 < 0 || ecount < 1 || e0 + ecount > tv.E) return fail_value("block range out of bounds");
  FFParams p{};
  p.x = x; p.m = m; p.ldx = ldx; p.d = d; p.rows = rows;
  p.bmask = tv.bmask; p.scat = tv.scat; p.cs = tv.cs; p.gcol = tv.gcol;
  p.soff = tv.soff; p.ggath = tv.ggath;
  p.scale = scale; p.norm = 1.0f; p.out = z; p.ldo = ldz; p.E = ecount; p.D = n * ecount;
  p.e0 = e0;
  p.tile8 = tile8 ? 1 : 0;
  return launch_by_logn(p, logn, false, fold, st);
}

int launch_by_logn(const FFParams& p, int logn, bool feat, bool fold, cudaStream_t st) {
  const bool vec = (p.d % 4 == 0) && (p.ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(p.x) & 15) == 0);
  if ((p.ldo % 4) || (reinterpret_cast<uintptr_t>(p.out) & 15))
    return fail_value("output rows must be 16-byte aligned");
  switch (logn) {
    case 3: return launch_ff_cfg<RowCfg<3, 2>>(p, feat, fold, vec, st);
    case 4: return launch_ff_cfg<RowCfg<4, 3>>(p, feat, fold, vec, st);
    case 5: return launch_ff_cfg<RowCfg<5, 4>>(p, feat, fold, vec, st);
    case 6: return launch_ff_cfg<RowCfg<6, 4>>(p, feat, fold, vec, st);
    case 7: return launch_ff_cfg<RowCfg<7, 5>>(p, feat, fold, vec, st);
    case 8: return launch_ff_cfg<RowCfg<8, 5>>(p, feat, fold, vec, st);
    case 9: return launch_ff_cfg<RowCfg<9, 5>>(p, feat, fold, vec, st);
    case 10: return launch_ff_cfg<RowCfg<10, 5>>(p, feat, fold, vec, st);
    case 11: return launch_ff_cfg<RowCfg<11, 5>>(p, feat, fold, vec, st);
    case 12: return launch_ff_cfg<RowCfg<12, 5>>(p, feat, fold, vec, st);
    case 13: return launch_ff_cfg<RowCfg<13, 5>>(p, feat, fold, vec, st);
    case 14: return launch_ff_cfg<RowCfg<14, 5>>(p, feat, fold, vec, st);
    default: return fail_value("unsupported padded_dim 2^%d", logn);
  }
}

}  // namespace mck
