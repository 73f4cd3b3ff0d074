// K1 -- batched in-place Walsh-Hadamard transform (replaces wht.py:142-162).
//
// fast variant
//   n <= 2^14 : one thread group per row (fwht_core.cuh), rows stay in
//               registers; 16-byte coalesced global loads/stores.  Large
//               batches of 2^14 rows: one persistent CTA per SM with the next
//               row prefetched (fwht_persistent14_kernel).
//   2^15, 2^16: the whole row on one SM (fwht_tmem_first_kernel): H_2 / H_4
//               across the 2^14 segments first, piece by piece at load time,
//               pieces parked in tensor memory; then each segment is read
//               back, transformed in registers / shared memory and stored;
//               one HBM pass.
//   2^17:       two "virtual rows" x0 + x1 and x0 - x1, formed at load time,
//               one per SM of a 2-CTA cluster on the one-SM pipeline
//               (fwht_tmem_virtual_kernel); one HBM pass, no DSMEM.
//   2^18:       a cluster of 4 such SMs per row, H_4 across the chunks by
//               st.async pushes through DSMEM (fwht_tmem_cluster_kernel); one
//               HBM pass.
//   2^19, 2^20: the row is viewed as [N1][2^14].  Phase A transforms the
//               N1-long columns (registers; stores tagged L2 evict_last);
//               phase B runs the register kernel on the N1 segments.  Chunks
//               of <= 24 MiB keep phase A's output in the 126 MB L2 for
//               phase B, which overlaps the next chunk's phase A on a side
//               stream.
// parity variant (verification only; bit-exact to the reference on
//   OpenBLAS SkylakeX): every aligned base chunk (256) becomes the sequential
//   fp32 sum over k of H[k][j]*x_k, then combine stages (a+b, (a+b)-2b).
#include "mck_common.cuh"
#include "fwht_core.cuh"
#include "umma.cuh"



namespace mck {

template <class V> struct Vec4;
template <> struct Vec4<float> {
  __device__ static void load(const float* p, float (&o)[4]) {
    float4 t = *reinterpret_cast<const float4*>(p);
    o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
  }
  __device__ static void store(float* p, const float (&o)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
  }
};
template <> struct Vec4<double> {
  __device__ static void load(const double* p, double (&o)[4]) {
    double2 a = reinterpret_cast<const double2*>(p)[0];
    double2 b = reinterpret_cast<const double2*>(p)[1];
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
  }
  __device__ static void store(double* p, const double (&o)[4]) {
    reinterpret_cast<double2*>(p)[0] = make_double2(o[0], o[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(o[2], o[3]);
  }
};

// Load/store a whole row in layout L (register k: index bits {0,1} from k&3,
// top bits from k>>2; thread id on bits 2..).
template <class C, class V>
__device__ __forceinline__ void load_row_L(const V* row, uint32_t tid, V (&v)[C::R]) {
#pragma unroll
  for (int j = 0; j < C::R / 4; ++j) {
    V t[4];
    Vec4<V>::load(row + 4 * tid + (size_t)j * (4 * C::T), t);
#pragma unroll
    for (int c = 0; c < 4; ++c) v[4 * j + c] = t[c];
  }
}
// Same through L2 only (ld.global.cg): for kernels whose shared memory leaves
// little L1 (the in-flight lines of a prefetched segment otherwise need L1 room).
template <class C>
__device__ __forceinline__ void load_row_L_cg(const float* row, uint32_t tid, float (&v)[C::R]) {
#pragma unroll
  for (int j = 0; j < C::R / 4; ++j) {
    const float4 t = __ldcg(reinterpret_cast<const float4*>(row + 4 * tid + (size_t)j * (4 * C::T)));
    v[4 * j] = t.x; v[4 * j + 1] = t.y; v[4 * j + 2] = t.z; v[4 * j + 3] = t.w;
  }
}
template <class C, class V>
__device__ __forceinline__ void store_row_L(V* row, uint32_t tid, const V (&v)[C::R]) {
#pragma unroll
  for (int j = 0; j < C::R / 4; ++j) {
    V t[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) t[c] = v[4 * j + c];
    Vec4<V>::store(row + 4 * tid + (size_t)j * (4 * C::T), t);
  }
}

template <class C>
constexpr int rows_per_cta() { return C::T >= 256 ? 1 : 256 / C::T; }
template <class C, class V>
__global__ void __launch_bounds__(C::T * rows_per_cta<C>())
fwht_rows_kernel(V* __restrict__ data, int64_t rows) {
  constexpr int ROWS = rows_per_cta<C>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* smem = reinterpret_cast<V*>(smem_raw);
  const int gid = threadIdx.x / C::T;
  const uint32_t tid = threadIdx.x % C::T;
  V* s = smem + gid * C::SMEM_FLOATS;
  const int64_t row = (int64_t)blockIdx.x * ROWS + gid;
  if (row >= rows) return;  // whole groups exit together
  V* p = data + row * (int64_t)C::N;
  V v[C::R];
  load_row_L<C>(p, tid, v);
  butterflies<C::R, C::PL, C::PL>(v);
  middle_rounds<C, 0, C::PL>(s, tid, gid, v);
  constexpr uint32_t PM = last_mid_regs<C>();
  if constexpr (sizeof(V) == 4 && (C::LOGN == 11 || C::LOGN == 12) && (PM & 31u) == 0) {
    // the last butterfly layout has its lanes on index bits 0..4: a warp
    // instruction stores 128 contiguous bytes, no exchange back to layout L
    // (measured: 2^11 1.01 -> 1.05, 2^12 0.99 -> 1.05 of the copy bandwidth;
    // 2^13 and 2^14 lose, 0.97 -> 0.86 and 0.92 -> 0.83: four times the store
    // instructions cost more than the exchange there)
    V* pt = p + thread_part<C::FULL, PM>(tid);
#pragma unroll
    for (int k = 0; k < C::R; ++k) pt[deposit_bits((uint32_t)k, PM)] = v[k];
  } else {
    sts_layout<C::R, PM>(s, thread_part<C::FULL, PM>(tid), v);
    group_sync<C::T>(gid);
    lds_layout<C::R, C::PL>(s, thread_part<C::FULL, C::PL>(tid), v);
    store_row_L<C>(p, tid, v);
  }
}

template <class C, class V>
int launch_rows(V* data, int64_t rows, cudaStream_t st) {
  constexpr int ROWS = rows_per_cta<C>();
  const size_t smem = (size_t)ROWS * C::SMEM_FLOATS * sizeof(V);
  auto kern = fwht_rows_kernel<C, V>;
  if (smem > 48 * 1024) {
    MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem), "fwht smem attribute"));
  }
  const int64_t blocks = (rows + ROWS - 1) / ROWS;
  for (int64_t b0 = 0; b0 < blocks; b0 += (1ll << 30)) {
    const int64_t nb = blocks - b0 < (1ll << 30) ? blocks - b0 : (1ll << 30);
    kern<<<(unsigned)nb, C::T * ROWS, smem, st>>>(data + b0 * ROWS * (int64_t)C::N,
                                                  rows - b0 * ROWS);
  }
  return check_launch("fwht_rows_kernel");
}

// Phase A of the large-n path: H_{N1} along the column index of the
// [N1][N2] view.  A thread owns VW adjacent columns (one 16/8/4-byte vector
// per row of the view) with all N1 vectors in registers, and strides over the
// chunk's columns (grid sized to the machine, not to the data).
template <class V, int VW> struct VecT;
template <> struct VecT<float, 4> { using T = float4; };
template <> struct VecT<float, 2> { using T = float2; };
template <> struct VecT<float, 1> { using T = float; };
template <> struct VecT<double, 2> { using T = double2; };
template <> struct VecT<double, 1> { using T = double; };

__device__ __forceinline__ void vadd(float& a, float& b) { const float x = a; a = x + b; b = x - b; }
__device__ __forceinline__ void vadd(double& a, double& b) { const double x = a; a = x + b; b = x - b; }
__device__ __forceinline__ void vadd(float2& a, float2& b) { vadd(a.x, b.x); vadd(a.y, b.y); }
__device__ __forceinline__ void vadd(double2& a, double2& b) { vadd(a.x, b.x); vadd(a.y, b.y); }
__device__ __forceinline__ void vadd(float4& a, float4& b) {
  vadd(a.x, b.x); vadd(a.y, b.y); vadd(a.z, b.z); vadd(a.w, b.w);
}

template <int LOGN1, int VW, class V>
__global__ void __launch_bounds__(256) fwht_cols_kernel(V* __restrict__ data, int64_t rows,
                                                        int n2) {
  using VT = typename VecT<V, VW>::T;
  constexpr int N1 = 1 << LOGN1;
  const int64_t vcols = n2 / VW;
  const int64_t total = rows * vcols;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / vcols;
    VT* p = reinterpret_cast<VT*>(data + row * (int64_t)N1 * n2) + (t % vcols);
    VT v[N1];
#pragma unroll
    for (int i = 0; i < N1; ++i) v[i] = p[(int64_t)i * vcols];
#pragma unroll
    for (int h = 1; h < N1; h <<= 1) {
#pragma unroll
      for (int i = 0; i < N1; ++i)
        if (!(i & h)) vadd(v[i], v[i | h]);
    }
    // keep phase A's output resident in L2 for phase B
    const uint64_t pol = l2_policy_evict_last();
#pragma unroll
    for (int i = 0; i < N1; ++i) st_hint(&p[(int64_t)i * vcols], v[i], pol);
  }
}

template <class V>
int launch_rows_by_logn(V* data, int64_t rows, int logn, cudaStream_t st) {
  switch (logn) {
    case 3: return launch_rows<RowCfg<3, 2>, V>(data, rows, st);
    case 4: return launch_rows<RowCfg<4, 3>, V>(data, rows, st);
    case 5: return launch_rows<RowCfg<5, 4>, V>(data, rows, st);
    case 6: return launch_rows<RowCfg<6, 4>, V>(data, rows, st);
    case 7: return launch_rows<RowCfg<7, 5>, V>(data, rows, st);
    case 8: return launch_rows<RowCfg<8, 5>, V>(data, rows, st);
    case 9: return launch_rows<RowCfg<9, 5>, V>(data, rows, st);
    case 10: return launch_rows<RowCfg<10, 5>, V>(data, rows, st);
    case 11: return launch_rows<RowCfg<11, 5>, V>(data, rows, st);
    case 12: return launch_rows<RowCfg<12, 5>, V>(data, rows, st);
    case 13: return launch_rows<RowCfg<13, 5>, V>(data, rows, st);
    case 14: return launch_rows<RowCfg<14, 5>, V>(data, rows, st);
    case 15:
      if (sizeof(V) == 4) return launch_rows<RowCfg<15, 5>, V>(data, rows, st);
      return fail_value("internal: fp64 rows kernel limited to 2^14");
    default: return fail_value("internal: no row kernel for 2^%d", logn);
  }
}

template <int LOGN1, int VW, class V>
int launch_cols_t(V* data, int64_t rows, int n2, cudaStream_t st) {
  const int64_t total = rows * (n2 / VW);
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 8) grid = 148 * 8;
  fwht_cols_kernel<LOGN1, VW, V><<<(unsigned)grid, 256, 0, st>>>(data, rows, n2);
  return check_launch("fwht_cols_kernel");
}

template <class V>
int launch_cols(V* data, int64_t rows, int logn1, int n2, cudaStream_t st) {
  constexpr bool F = sizeof(V) == 4;
  switch (logn1) {
    case 1: return launch_cols_t<1, F ? 4 : 2, V>(data, rows, n2, st);
    case 2: return launch_cols_t<2, F ? 4 : 2, V>(data, rows, n2, st);
    case 3: return launch_cols_t<3, F ? 4 : 2, V>(data, rows, n2, st);
    case 4: return launch_cols_t<4, F ? 4 : 2, V>(data, rows, n2, st);
    case 5: return launch_cols_t<5, F ? 2 : 1, V>(data, rows, n2, st);
    case 6: return launch_cols_t<6, 1, V>(data, rows, n2, st);
    default: return fail_value("internal: no column kernel for 2^%d", logn1);
  }
}

// ---- tensor-memory kernels (2^15 .. 2^18, fp32).  A persistent 512-thread
// CTA owns its SM's tensor memory (256 KB) and uses it as a thread-private
// register extension: thread t of warp w reads / writes TMEM lane
// 32*(w%4)+t, columns (w/4)*32*NSEG + ... (tcgen05.st / tcgen05.ld, 32 columns
// per thread and 2^14 segment).  Every thread holds the same positions of
// every segment, so H across the segments needs no exchange at all.
#ifndef MCK_FWHT_TMEM
#define MCK_FWHT_TMEM 1
#endif
#ifndef MCK_FWHT_VIRTUAL
#define MCK_FWHT_VIRTUAL 2  // largest row / 2^16 on the virtual-row kernel (2^17: 0.71 -> 0.82; 4 = 2^18 too: 0.45 vs 0.55 with DSMEM)
#endif
#ifndef MCK_FWHT_TMEM_CLUSTER_MAX
#define MCK_FWHT_TMEM_CLUSTER_MAX 18  // largest log2 n on the TMEM cluster kernel (2^19, 2^20: two-phase path is faster)
#endif
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32], int o) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[o + 0])), "r"(__float_as_uint(v[o + 1])), "r"(__float_as_uint(v[o + 2])),
      "r"(__float_as_uint(v[o + 3])), "r"(__float_as_uint(v[o + 4])), "r"(__float_as_uint(v[o + 5])),
      "r"(__float_as_uint(v[o + 6])), "r"(__float_as_uint(v[o + 7])), "r"(__float_as_uint(v[o + 8])),
      "r"(__float_as_uint(v[o + 9])), "r"(__float_as_uint(v[o + 10])), "r"(__float_as_uint(v[o + 11])),
      "r"(__float_as_uint(v[o + 12])), "r"(__float_as_uint(v[o + 13])), "r"(__float_as_uint(v[o + 14])),
      "r"(__float_as_uint(v[o + 15]))
      : "memory");
}
__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// Phase 1 of the TMEM kernels: transform the NSEG segments of the chunk at
// `chunk` (segment 0 already in w) and park them; the loads of the following
// segment -- or of segment 0 of `next` (may be null) -- fly meanwhile.
constexpr int TMEM_S_FLOATS = (RowCfg<14, 5>::SMEM_FLOATS + 3) / 4 * 4;

// Eight parked registers (8j .. 8j+7) of every segment, H_NSEG applied.
template <int NSEG>
__device__ __forceinline__ void tmem_piece(uint32_t tbase, int j, float (&a)[NSEG][8]) {
#pragma unroll
  for (int sg = 0; sg < NSEG; ++sg) tmem_ld8_nowait(tbase + 32u * sg + 8u * j, a[sg]);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int h = 1; h < NSEG; h <<= 1)
#pragma unroll
    for (int sg = 0; sg < NSEG; ++sg)
      if (!(sg & h)) {
#pragma unroll
        for (int i = 0; i < 8; i += 2) bfly_pk(a[sg][i], a[sg][i + 1], a[sg | h][i], a[sg | h][i + 1]);
      }
}

// n = NSEG * 2^14, NSEG = 2 or 4: the whole row on ONE SM, one HBM pass, no
// cluster, with H_NSEG FIRST (the stages commute): the
// row arrives in NSEG pieces -- registers j*32/NSEG .. of layout L of every
// segment, prefetched one piece per segment step -- and each piece gets H_NSEG
// across the segments before it is parked.  A segment step then reads one
// H_NSEG-finished segment back from TMEM, runs the register / shared-memory
// transform and stores it straight from its last butterfly layout.  Loads (one
// piece) and stores (one segment) are spread evenly over the steps: there is
// no store burst at the end of the row any more.  TMEM stays exactly full: the
// 32 columns a step's segment frees take the next row's piece, which makes the
// parked layout alternate between segment-major (segment q register k at
// column 32 q + k) and piece-major (segment q register P j + i at column
// 32 j + P q + i, P = 32 / NSEG) from one row to the next.
template <int N, int LEN>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const float (&v)[LEN], int o) {
  static_assert(N == 8 || N == 16, "columns");
  if constexpr (N == 16) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(__float_as_uint(v[o + 0])), "r"(__float_as_uint(v[o + 1])), "r"(__float_as_uint(v[o + 2])),
        "r"(__float_as_uint(v[o + 3])), "r"(__float_as_uint(v[o + 4])), "r"(__float_as_uint(v[o + 5])),
        "r"(__float_as_uint(v[o + 6])), "r"(__float_as_uint(v[o + 7])), "r"(__float_as_uint(v[o + 8])),
        "r"(__float_as_uint(v[o + 9])), "r"(__float_as_uint(v[o + 10])), "r"(__float_as_uint(v[o + 11])),
        "r"(__float_as_uint(v[o + 12])), "r"(__float_as_uint(v[o + 13])), "r"(__float_as_uint(v[o + 14])),
        "r"(__float_as_uint(v[o + 15]))
        : "memory");
  } else {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(__float_as_uint(v[o + 0])), "r"(__float_as_uint(v[o + 1])),
                 "r"(__float_as_uint(v[o + 2])), "r"(__float_as_uint(v[o + 3])),
                 "r"(__float_as_uint(v[o + 4])), "r"(__float_as_uint(v[o + 5])),
                 "r"(__float_as_uint(v[o + 6])), "r"(__float_as_uint(v[o + 7]))
                 : "memory");
  }
}
template <int N, int LEN>
__device__ __forceinline__ void tmem_ld_cols_nowait(uint32_t taddr, float (&v)[LEN], int o) {
  static_assert(N == 8 || N == 16, "columns");
  uint32_t r[N];
  if constexpr (N == 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
  }
#pragma unroll
  for (int i = 0; i < N; ++i) v[o + i] = __uint_as_float(r[i]);
}

template <int NSEG>
struct TmemFirst {
  using C = RowCfg<14, 5>;
  static constexpr int P = 32 / NSEG;  // registers per piece and segment
  // piece j of the row at prow into w[q * P + i] (segment q, register j * P + i of layout L)
  __device__ static void load_piece(const float* prow, int j, uint32_t tid, float (&w)[32]) {
#pragma unroll
    for (int q = 0; q < NSEG; ++q)
#pragma unroll
      for (int t = 0; t < P / 4; ++t) {
        float x[4];
        Vec4<float>::load(prow + (int64_t)q * C::N + 4 * tid + (size_t)(j * (P / 4) + t) * (4 * C::T), x);
#pragma unroll
        for (int e = 0; e < 4; ++e) w[q * P + 4 * t + e] = x[e];
      }
  }
  __device__ static void across_segments(float (&w)[32]) {
#pragma unroll
    for (int h = 1; h < NSEG; h <<= 1)
#pragma unroll
      for (int q = 0; q < NSEG; ++q)
        if (!(q & h)) {
#pragma unroll
          for (int i = 0; i < P; i += 2)
            bfly_pk(w[q * P + i], w[q * P + i + 1], w[(q | h) * P + i], w[(q | h) * P + i + 1]);
        }
  }
  // column of (segment q, register j * P + i): segment-major (MAJ = 0) or piece-major
  template <int MAJ>
  __device__ static constexpr uint32_t col(int q, int j) { return MAJ == 0 ? 32 * q + P * j : 32 * j + P * q; }
  // park piece j (already H_NSEG'ed) of a row whose layout is MAJ
  template <int MAJ>
  __device__ static void park_piece(uint32_t tbase, int j, const float (&w)[32]) {
#pragma unroll
    for (int q = 0; q < NSEG; ++q) tmem_st_cols<P>(tbase + col<MAJ>(q, j), w, q * P);
  }
  // read segment q of a row whose layout is MAJ into v (layout L registers)
  template <int MAJ>
  __device__ static void fetch_segment(uint32_t tbase, int q, float (&v)[32]) {
#pragma unroll
    for (int j = 0; j < NSEG; ++j) tmem_ld_cols_nowait<P>(tbase + col<MAJ>(q, j), v, j * P);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  }
};

// One row whose parked layout is MAJ: NSEG segment steps; `next` (may be null)
// is the row whose pieces are parked meanwhile (piece 0 already in w) in the
// other layout, `after` (may be null) the row after that (its piece 0 is left
// in w).
template <int NSEG, int MAJ>
__device__ __forceinline__ void tmem_first_row(float* s, float* s2, uint32_t tid, uint32_t tbase, float* prow,
                                               const float* next, const float* after, float (&w)[32]) {
  using C = RowCfg<14, 5>;
  using TF = TmemFirst<NSEG>;
  constexpr uint32_t PM = last_mid_regs<C>();
  float* pt = prow + thread_part<C::FULL, PM>(tid);
#pragma unroll
  for (int sg = 0; sg < NSEG; ++sg) {
    float v[C::R];
    TF::template fetch_segment<MAJ>(tbase, sg, v);  // frees the segment's 32 columns ...
    if (next) {
      TF::across_segments(w);
      TF::template park_piece<1 - MAJ>(tbase, sg, w);  // ... which take the next row's piece sg
      if (sg + 1 < NSEG) TF::load_piece(next, sg + 1, tid, w);
      else if (after) TF::load_piece(after, 0, tid, w);
    }
    butterflies<C::R, C::PL, C::PL>(v);
    middle_rounds_2buf<C, 0, C::PL>(s, s2, tid, 0, v);
#pragma unroll
    for (int k = 0; k < C::R; ++k) pt[(int64_t)sg * C::N + deposit_bits((uint32_t)k, PM)] = v[k];
    umma::tmem_wait_st();
    __syncthreads();  // re-align the warps: the next piece's loads go out as one burst
  }
}

template <int NSEG>
__global__ void __launch_bounds__(RowCfg<14, 5>::T, 1)
fwht_tmem_first_kernel(float* __restrict__ data, int64_t rows) {
  using C = RowCfg<14, 5>;
  using TF = TmemFirst<NSEG>;
  constexpr int64_t ROW = (int64_t)NSEG * C::N;
  constexpr uint32_t COLS = 32 * NSEG * (C::T / 128);
  static_assert(COLS <= 512 && (COLS & (COLS - 1)) == 0, "TMEM columns");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* s = reinterpret_cast<float*>(smem_raw);
  float* s2 = s + TMEM_S_FLOATS;
  __shared__ uint32_t tmem_slot;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) umma::tmem_alloc<COLS>(&tmem_slot);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tbase = tmem_slot + ((32u * (warp & 3u)) << 16) + (warp >> 2) * (32u * NSEG);

  const int64_t step = gridDim.x;
  int64_t row = blockIdx.x;
  float w[32];
  if (row < rows) {
    // first row: all pieces, H_NSEG, parked segment-major
#pragma unroll
    for (int j = 0; j < NSEG; ++j) {
      TF::load_piece(data + row * ROW, j, tid, w);
      TF::across_segments(w);
      TF::template park_piece<0>(tbase, j, w);
    }
    umma::tmem_wait_st();
    if (row + step < rows) TF::load_piece(data + (row + step) * ROW, 0, tid, w);
  }
  auto at = [&](int64_t r) -> float* { return r < rows ? data + r * ROW : nullptr; };
  for (; row < rows; row += 2 * step) {
    tmem_first_row<NSEG, 0>(s, s2, tid, tbase, data + row * ROW, at(row + step), at(row + 2 * step), w);
    if (row + step < rows)
      tmem_first_row<NSEG, 1>(s, s2, tid, tbase, data + (row + step) * ROW, at(row + 2 * step), at(row + 3 * step), w);
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<COLS>(tmem_slot);
}

// n = 2^14 the same way, without tensor memory: a persistent 512-thread CTA
// per SM, the next row's loads in a second register set under the current
// transform, two alternating exchange buffers, the row stored from its last
// butterfly layout.
__global__ void __launch_bounds__(RowCfg<14, 5>::T, 1)
fwht_persistent14_kernel(float* __restrict__ data, int64_t rows) {
  using C = RowCfg<14, 5>;
  constexpr uint32_t PM = last_mid_regs<C>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* s = reinterpret_cast<float*>(smem_raw);
  float* s2 = s + TMEM_S_FLOATS;
  const uint32_t tid = threadIdx.x;
  const uint32_t tpart = thread_part<C::FULL, PM>(tid);
  float w[C::R];
  int64_t row = blockIdx.x;
  if (row < rows) load_row_L<C>(data + row * C::N, tid, w);
  for (; row < rows; row += gridDim.x) {
    float v[C::R];
#pragma unroll
    for (int k = 0; k < C::R; ++k) v[k] = w[k];
    if (row + gridDim.x < rows) load_row_L<C>(data + (row + gridDim.x) * C::N, tid, w);
    butterflies<C::R, C::PL, C::PL>(v);
    middle_rounds_2buf<C, 0, C::PL>(s, s2, tid, 0, v);
    float* pt = data + row * C::N + tpart;
#pragma unroll
    for (int k = 0; k < C::R; ++k) pt[deposit_bits((uint32_t)k, PM)] = v[k];
    __syncthreads();  // re-align the warps: the next row's loads go out as one burst
  }
}

int launch_persistent14(float* data, int64_t rows, cudaStream_t st) {
  const size_t smem = 2 * (size_t)TMEM_S_FLOATS * sizeof(float);
  auto kern = fwht_persistent14_kernel;
  static PerDevice pd;
  const DeviceSlot* ds = nullptr;
  MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot&) {
    MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem), "fwht persistent smem"));
    return MCK_OK;
  }));
  int64_t grid = ds->sms;
  if (grid > rows) grid = rows;
  kern<<<(unsigned)grid, RowCfg<14, 5>::T, smem, st>>>(data, rows);
  return check_launch("fwht_persistent14_kernel");
}

template <int NSEG>
int launch_tmem_t(float* data, int64_t rows, cudaStream_t st) {
  using C = RowCfg<14, 5>;
  // two exchange buffers, more than half of the SM's shared memory: one CTA
  // per SM, which owns the TMEM
  const size_t smem = 2 * (size_t)TMEM_S_FLOATS * sizeof(float);
  static_assert(2 * (size_t)TMEM_S_FLOATS * sizeof(float) > 116 * 1024, "one CTA per SM");
  auto kern = fwht_tmem_first_kernel<NSEG>;
  static PerDevice pd;
  const DeviceSlot* ds = nullptr;
  MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot&) {
    MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem), "fwht tmem smem"));
    return MCK_OK;
  }));
  int64_t grid = ds->sms;
  if (grid > rows) grid = rows;
  kern<<<(unsigned)grid, C::T, smem, st>>>(data, rows);
  return check_launch("fwht_tmem_first_kernel");
}

// n = K * 2^16, K = 2..16 (fp32): one cluster of K CTAs per row, one HBM
// pass.  CTA c owns the contiguous 2^16 chunk c (four 2^14 segments).  After
// a segment's register/shared-memory transform, H_K across the chunks runs at
// equal chunk offsets and every thread keeps its element positions: of its 32
// registers, the 32/K that peer k owns are pushed straight from the registers
// into peer k's receive buffer (st.async through DSMEM, completing on the
// peer's mbarrier).  One segment later -- the pushes have flown under the
// next segment's transform -- the thread collects its own 32/K positions of
// all K chunks, applies H_K and parks the 32 values in tensor memory.  After
// four segments the row closes like the one-SM kernel: H_4 across the parked
// segments and 128-byte warp stores, now into all K chunks.  Two receive
// buffers; the pushes of segment g+2 wait for every CTA to have read segment
// g (split cluster barrier, arrived a whole segment earlier).
__device__ __forceinline__ uint32_t map_to_cta(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async4(uint32_t addr, uint32_t bar, float a, float b, float c, float d) {
  asm volatile(
      "st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(addr),
      "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d)),
      "r"(bar)
      : "memory");
}
__device__ __forceinline__ void st_async2(uint32_t addr, uint32_t bar, float a, float b) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1,%2}, [%3];" ::"r"(addr),
               "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int kNoClusterFits = -0x4e4f;  // internal: launch_tmem_cluster could not place a cluster

template <int K>
struct TmemCluster {
  using C = RowCfg<14, 5>;
  static constexpr int V = 32 / K;             // values per thread, piece and owner
  static constexpr int VW = V >= 4 ? 4 : 2;    // vector width of a push
  static constexpr int NV = V / VW;            // pushes per owner
  static constexpr uint32_t PIECE_BYTES = 32u * C::T * 4u;  // 64 KB: K sources x V values x T threads
  static constexpr uint32_t SRC_BYTES = PIECE_BYTES / K;    // one source's share
  static constexpr uint32_t REMOTE_BYTES = SRC_BYTES * (K - 1);
  static constexpr size_t S_BYTES = ((size_t)C::SMEM_FLOATS * 4 + 15) / 16 * 16;
  // one buffer for the CTA's own share (written after the previous segment's
  // collect has read it) and two for the peers' shares (in flight under the
  // next transform).  K = 2: 162 KB, which fits the 164 KB carve-out and
  // leaves 92 KB of L1 for the prefetch loads (DESIGN: carve-out vs loads)
  static constexpr size_t SMEM = S_BYTES + SRC_BYTES + 2 * (size_t)REMOTE_BYTES + 16;
  // vector q of thread tid inside one source's share
  __device__ static uint32_t slot(int q, uint32_t tid) { return (q * C::T + tid) * (VW * 4u); }
  // index of source `src` among the K - 1 remote shares of CTA `dst`
  __device__ static uint32_t remote_index(uint32_t src, uint32_t dst) { return src < dst ? src : src - 1; }
};

template <int K>
__global__ void __launch_bounds__(RowCfg<14, 5>::T, 1)
fwht_tmem_cluster_kernel(float* __restrict__ data, int64_t rows) {
  using C = RowCfg<14, 5>;
  using TC = TmemCluster<K>;
  constexpr int SEG = C::N, V = TC::V, VW = TC::VW, NV = TC::NV;
  constexpr int64_t CHUNK = 4 * SEG;
  constexpr uint32_t PM = last_mid_regs<C>();
  constexpr uint32_t PUSH_BYTES = TC::PIECE_BYTES / K * (K - 1);  // a CTA's own share stays local
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* s = reinterpret_cast<float*>(smem_raw);
  unsigned char* own = smem_raw + TC::S_BYTES;  // this CTA's own share
  unsigned char* rb = own + TC::SRC_BYTES;      // two buffers of the peers' shares
  uint64_t* full = reinterpret_cast<uint64_t*>(rb + 2 * TC::REMOTE_BYTES);
  __shared__ uint32_t tmem_slot;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  uint32_t c;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(c));
  if (warp == 0) umma::tmem_alloc<512>(&tmem_slot);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
    mbar_expect_tx(&full[0], PUSH_BYTES);
    mbar_expect_tx(&full[1], PUSH_BYTES);
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  // barriers initialised cluster-wide before any push; leaves one arrival
  // outstanding (paired with the wait in front of the first push)
  cluster_arrive();
  cluster_wait();
  cluster_arrive();
  const uint32_t tbase = tmem_slot + ((32u * (warp & 3u)) << 16) + (warp >> 2) * 128u;
  const uint32_t rb_u32 = smem_u32(rb), full_u32 = smem_u32(full);
  // this CTA owns registers c*V .. c*V+V-1 of every thread's 32 (layout PM)
  const uint32_t own_dep = deposit_bits(c * V, PM);
  const uint32_t tpart = thread_part<C::FULL, PM>(tid);

  const int64_t nclusters = gridDim.x / K, cid = blockIdx.x / K;
  const int64_t mine = cid < rows ? (rows - cid + nclusters - 1) / nclusters : 0;
  float w[C::R];
  if (mine > 0) load_row_L_cg<C>(data + cid * (K * CHUNK) + c * CHUNK, tid, w);

  // collect segment sg (buffer sg & 1): own positions of all K chunks, H_K, park
  auto consume = [&](int sg) {
    const uint32_t buf = (uint32_t)(sg & 1) * TC::REMOTE_BYTES;
    mbar_wait(&full[sg & 1], (uint32_t)(sg >> 1) & 1u);
    float x[32];  // x[k * V + i]: chunk k, owned register i
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const unsigned char* at = (uint32_t)k == c
                                      ? own + TC::slot(q, tid)
                                      : rb + buf + TC::remote_index(k, c) * TC::SRC_BYTES + TC::slot(q, tid);
        if constexpr (VW == 4) {
          const float4 t = *reinterpret_cast<const float4*>(at);
          x[k * V + 4 * q] = t.x; x[k * V + 4 * q + 1] = t.y; x[k * V + 4 * q + 2] = t.z; x[k * V + 4 * q + 3] = t.w;
        } else {
          const float2 t = *reinterpret_cast<const float2*>(at);
          x[k * V + 2 * q] = t.x; x[k * V + 2 * q + 1] = t.y;
        }
      }
    if (tid == 0) mbar_expect_tx(&full[sg & 1], PUSH_BYTES);  // re-arm for the buffer's next use
#pragma unroll
    for (int h = 1; h < K; h <<= 1)
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (!(k & h)) {
#pragma unroll
          for (int i = 0; i < V; i += 2)
            bfly_pk(x[k * V + i], x[k * V + i + 1], x[(k | h) * V + i], x[(k | h) * V + i + 1]);
        }
    // the buffer's values have been consumed: release it to the peers.  The
    // barrier only orders these reads against later pushes (the pushed data
    // itself is published by the mbarrier), so no release fence is needed --
    // a fence here would wait for every global store in flight.
    cluster_arrive_relaxed();
    tmem_st32(tbase + 32u * sg, x, 0);
    tmem_st32(tbase + 32u * sg + 16u, x, 16);
  };

  for (int64_t it = 0; it <= mine; ++it) {
    const bool have = it < mine;
    const int64_t row = cid + it * nclusters;
    const float* chunk = data + row * (K * CHUNK) + c * CHUNK;
#pragma unroll
    for (int sg = 0; sg < 4; ++sg) {
      float keep[V];
      if (have) {
        float v[C::R];
#pragma unroll
        for (int k = 0; k < C::R; ++k) v[k] = w[k];
        if (sg + 1 < 4) {
          load_row_L_cg<C>(chunk + (int64_t)(sg + 1) * SEG, tid, w);
        } else if (it + 1 < mine) {
          load_row_L_cg<C>(chunk + nclusters * (K * CHUNK), tid, w);
        }
        butterflies<C::R, C::PL, C::PL>(v);
        middle_rounds<C, 0, C::PL>(s, tid, 0, v);
        cluster_wait();  // every CTA has read what buffer sg & 1 held
        const uint32_t buf = (uint32_t)(sg & 1) * TC::REMOTE_BYTES;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if ((uint32_t)k == c) continue;
          const uint32_t dst = map_to_cta(rb_u32 + buf + TC::remote_index(c, k) * TC::SRC_BYTES, k);
          const uint32_t bar = map_to_cta(full_u32 + 8u * (sg & 1), k);
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const int f = k * V + q * VW;
            const uint32_t at = dst + TC::slot(q, tid);
            if constexpr (VW == 4)
              st_async4(at, bar, v[f], v[f + 1], v[f + 2], v[f + 3]);
            else
              st_async2(at, bar, v[f], v[f + 1]);
          }
        }
        // the own share, kept until the previous segment's has been read
#pragma unroll
        for (int k = 0; k < K; ++k)
          if ((uint32_t)k == c) {
#pragma unroll
            for (int i = 0; i < V; ++i) keep[i] = v[k * V + i];
          }
        if (it == 0 && sg == 0) cluster_arrive_relaxed();  // nothing to collect yet
      }
      const bool pending = sg > 0 ? have : it > 0;
      if (pending) {
        if (!have) cluster_wait();  // closing round: no push waited for the previous arrival
        consume((sg + 3) & 3);
      }
      if (have) {
        // own share of this segment (its buffer's previous content is consumed);
        // read back by this thread only
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          unsigned char* at = own + TC::slot(q, tid);
          if constexpr (VW == 4)
            *reinterpret_cast<float4*>(at) = make_float4(keep[4 * q], keep[4 * q + 1], keep[4 * q + 2], keep[4 * q + 3]);
          else
            *reinterpret_cast<float2*>(at) = make_float2(keep[2 * q], keep[2 * q + 1]);
        }
      }
      if (sg == 0 && it > 0) {
        umma::tmem_wait_st();
        // close the previous row: H_4 across its parked segments, stores
        float* pt = data + (row - nclusters) * (K * CHUNK) + tpart + own_dep;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float a[4][8];
          tmem_piece<4>(tbase, j, a);
#pragma unroll
          for (int sgo = 0; sgo < 4; ++sgo)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int m = 8 * j + i;  // parked column: chunk m / V, owned register m % V
              pt[(int64_t)(m / V) * CHUNK + sgo * SEG + deposit_bits((uint32_t)(m % V), PM)] = a[sgo][i];
            }
        }
      }
    }
  }
  cluster_wait();
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<512>(tmem_slot);
}

template <int K>
int launch_tmem_cluster_t(float* data, int64_t rows, cudaStream_t st) {
  using C = RowCfg<14, 5>;
  using TC = TmemCluster<K>;
  auto kern = fwht_tmem_cluster_kernel<K>;
  static PerDevice pd;
  const DeviceSlot* ds = nullptr;
  MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot& slot) {
    MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)TC::SMEM), "fwht tmem cluster smem"));
    if (K > 8)
      MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                         "fwht cluster size"));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(K * 148);
    cfg.blockDim = dim3(C::T);
    cfg.dynamicSmemBytes = TC::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    MCK_TRY(check_cuda(cudaOccupancyMaxActiveClusters(&n, kern, &cfg), "fwht cluster occupancy"));
    slot.occ = n;  // co-resident clusters on the device (0: none fits, e.g. a partitioned GPU)
    return MCK_OK;
  }));
  if (ds->occ < 1) return kNoClusterFits;
  int64_t nc = ds->occ;
  if (nc > rows) nc = rows;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(nc * K));
  cfg.blockDim = dim3(C::T);
  cfg.dynamicSmemBytes = TC::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = K;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  MCK_TRY(check_cuda(cudaLaunchKernelEx(&cfg, kern, data, rows), "fwht_tmem_cluster_kernel launch"));
  return check_launch("fwht_tmem_cluster_kernel");
}

// n = VR * 2^16, VR = 2 or 4 (fp32): "virtual rows".  H_n = H_VR (x) H_{2^16}
// and the stages commute, so output chunk vr of a row is the 2^16 transform
// of sum_c (-1)^popc(vr & c) x_c over the row's VR input chunks.  CTA vr of a
// VR-CTA cluster computes exactly that: it runs the one-SM pipeline above on
// its virtual row, whose pieces are formed at load time from the same
// positions of ALL VR chunks (each input is read VR times, once from HBM and
// VR - 1 times from L2: the CTAs of a cluster walk the row together).  No
// data crosses between the SMs -- no DSMEM, no receive buffers; the cluster
// exists for its barrier: the transform is in place, so a CTA may only store
// its output chunk once every CTA has loaded the whole row (arrive after the
// row's last piece is parked, wait before its first store).  A piece (8
// registers per segment) arrives as VR sub-pieces so that 32 registers of
// loads are in flight at a time; they are consumed at VR points spread over
// the segment step.
template <int N, int LEN>
__device__ __forceinline__ void tmem_st_small(uint32_t taddr, const float (&v)[LEN], int o) {
  static_assert(N == 2 || N == 4, "columns");
  if constexpr (N == 4)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
                 "r"(__float_as_uint(v[o + 0])), "r"(__float_as_uint(v[o + 1])),
                 "r"(__float_as_uint(v[o + 2])), "r"(__float_as_uint(v[o + 3]))
                 : "memory");
  else
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr),
                 "r"(__float_as_uint(v[o + 0])), "r"(__float_as_uint(v[o + 1]))
                 : "memory");
}

template <int VR>
struct TmemVirtual {
  using C = RowCfg<14, 5>;
  using TF = TmemFirst<4>;
  static constexpr int PV = 8 / VR;  // registers per segment and chunk in one sub-piece
  static constexpr int64_t CHUNK = 4 * (int64_t)C::N;
  // sub-piece u (piece j = u / VR, part h = u % VR) of the row at `row`:
  // w[(c * 4 + q) * PV + e] = chunk c, segment q, register 8 j + PV h + e of layout L
  __device__ static void load_sub(const float* row, int u, uint32_t tid, float (&w)[32]) {
    const int k0 = 8 * (u / VR) + PV * (u % VR);
    const size_t off = (size_t)(k0 & 3) + 4 * tid + (size_t)(k0 >> 2) * (4 * C::T);
#pragma unroll
    for (int c = 0; c < VR; ++c)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float* p = row + c * CHUNK + (int64_t)q * C::N + off;
        if constexpr (PV == 4) {
          const float4 t = *reinterpret_cast<const float4*>(p);
          w[(c * 4 + q) * 4] = t.x; w[(c * 4 + q) * 4 + 1] = t.y; w[(c * 4 + q) * 4 + 2] = t.z; w[(c * 4 + q) * 4 + 3] = t.w;
        } else {
          const float2 t = *reinterpret_cast<const float2*>(p);
          w[(c * 4 + q) * 2] = t.x; w[(c * 4 + q) * 2 + 1] = t.y;
        }
      }
  }
  // this CTA's virtual row from the raw sub-piece, then H_4 across the segments
  __device__ static void form(const float (&w)[32], uint32_t vr, float (&d)[4 * PV]) {
#pragma unroll
    for (int i = 0; i < 4 * PV; ++i) d[i] = w[i];
#pragma unroll
    for (int c = 1; c < VR; ++c) {
      const bool neg = __popc(vr & (uint32_t)c) & 1;
#pragma unroll
      for (int i = 0; i < 4 * PV; ++i) d[i] = neg ? d[i] - w[c * 4 * PV + i] : d[i] + w[c * 4 * PV + i];
    }
#pragma unroll
    for (int h = 1; h < 4; h <<= 1)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (!(q & h)) {
#pragma unroll
          for (int i = 0; i < PV; i += 2) bfly_pk(d[q * PV + i], d[q * PV + i + 1], d[(q | h) * PV + i], d[(q | h) * PV + i + 1]);
        }
  }
  template <int MAJ>
  __device__ static void park_sub(uint32_t tbase, int j, int h, const float (&d)[4 * PV]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) tmem_st_small<PV>(tbase + TF::template col<MAJ>(q, j) + PV * h, d, q * PV);
  }
};

// One virtual row parked in layout MAJ.  out: this CTA's output chunk of the
// row; next / after: the following rows (may be null), w holds next's
// sub-piece 0 on entry and after's on exit.
template <int VR, int MAJ>
__device__ __forceinline__ void tmem_virtual_row(float* s, float* s2, uint32_t tid, uint32_t vr, uint32_t tbase,
                                                 float* out, const float* next, const float* after,
                                                 float (&w)[32]) {
  using C = RowCfg<14, 5>;
  using TF = TmemFirst<4>;
  using TV = TmemVirtual<VR>;
  constexpr uint32_t P0 = C::mid_regs(0), PM = last_mid_regs<C>();
  static_assert(C::NMID == 2, "two exchanges");
  float* pt = out + thread_part<C::FULL, PM>(tid);
#pragma unroll
  for (int sg = 0; sg < 4; ++sg) {
    float v[C::R];
    TF::template fetch_segment<MAJ>(tbase, sg, v);  // frees the columns the next row's piece sg takes
    auto service = [&](int h) {  // part h of the next row's piece sg; then the following loads
      if (!next) return;
      float d[4 * TV::PV];
      TV::form(w, vr, d);
      TV::template park_sub<1 - MAJ>(tbase, sg, h, d);
      const int u = sg * VR + h + 1;
      if (u < 4 * VR) TV::load_sub(next, u, tid, w);
      else if (after) TV::load_sub(after, 0, tid, w);
    };
    service(0);
    butterflies<C::R, C::PL, C::PL>(v);
    sts_layout<C::R, C::PL>(s, thread_part<C::FULL, C::PL>(tid), v);
    __syncthreads();
    lds_layout<C::R, P0>(s, thread_part<C::FULL, P0>(tid), v);
    if (VR == 4) service(1);
    butterflies<C::R, P0, C::mid_active(0)>(v);
    sts_layout<C::R, P0>(s2, thread_part<C::FULL, P0>(tid), v);
    __syncthreads();
    lds_layout<C::R, PM>(s2, thread_part<C::FULL, PM>(tid), v);
    service(VR == 4 ? 2 : 1);
    butterflies<C::R, PM, C::mid_active(1)>(v);
    if (VR == 4) service(3);
    if (sg == 3 && next) cluster_arrive_relaxed();  // this CTA has loaded the whole next row
    if (sg == 0) cluster_wait();                    // every CTA has loaded this row: its chunks may be overwritten
#pragma unroll
    for (int k = 0; k < C::R; ++k) pt[(int64_t)sg * C::N + deposit_bits((uint32_t)k, PM)] = v[k];
    umma::tmem_wait_st();
    __syncthreads();  // re-align the warps: the next loads go out as one burst
  }
}

template <int VR>
__global__ void __launch_bounds__(RowCfg<14, 5>::T, 1)
fwht_tmem_virtual_kernel(float* __restrict__ data, int64_t rows) {
  using C = RowCfg<14, 5>;
  using TV = TmemVirtual<VR>;
  constexpr int64_t ROW = VR * TV::CHUNK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* s = reinterpret_cast<float*>(smem_raw);
  float* s2 = s + TMEM_S_FLOATS;
  __shared__ uint32_t tmem_slot;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  uint32_t vr;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(vr));
  if (warp == 0) umma::tmem_alloc<512>(&tmem_slot);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tbase = tmem_slot + ((32u * (warp & 3u)) << 16) + (warp >> 2) * 128u;

  const int64_t nclusters = gridDim.x / VR, cid = blockIdx.x / VR;
  const int64_t mine = cid < rows ? (rows - cid + nclusters - 1) / nclusters : 0;
  const int64_t step = nclusters * ROW;
  float* const row0 = data + cid * ROW;
  float w[32];
  if (mine > 0) {
    // first row: every sub-piece, formed and parked segment-major
#pragma unroll
    for (int u = 0; u < 4 * VR; ++u) {
      TV::load_sub(row0, u, tid, w);
      float d[4 * TV::PV];
      TV::form(w, vr, d);
      TV::template park_sub<0>(tbase, u / VR, u % VR, d);
    }
    umma::tmem_wait_st();
    cluster_arrive_relaxed();  // first row loaded
    if (mine > 1) TV::load_sub(row0 + step, 0, tid, w);
  }
  auto at = [&](int64_t it) -> float* { return it < mine ? row0 + it * step : nullptr; };
  for (int64_t it = 0; it < mine; it += 2) {
    tmem_virtual_row<VR, 0>(s, s2, tid, vr, tbase, at(it) + vr * TV::CHUNK, at(it + 1), at(it + 2), w);
    if (it + 1 < mine)
      tmem_virtual_row<VR, 1>(s, s2, tid, vr, tbase, at(it + 1) + vr * TV::CHUNK, at(it + 2), at(it + 3), w);
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<512>(tmem_slot);
}

template <int VR>
int launch_tmem_virtual_t(float* data, int64_t rows, cudaStream_t st) {
  using C = RowCfg<14, 5>;
  const size_t smem = 2 * (size_t)TMEM_S_FLOATS * sizeof(float);
  auto kern = fwht_tmem_virtual_kernel<VR>;
  static PerDevice pd;
  const DeviceSlot* ds = nullptr;
  auto config = [&](unsigned grid, cudaLaunchAttribute* at) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(C::T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = VR;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cfg;
  };
  MCK_TRY(per_device(pd, &ds, [&](int, DeviceSlot& slot) {
    MCK_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                       "fwht virtual smem"));
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = config(VR * 148, at);
    cfg.stream = nullptr;
    int n = 0;
    MCK_TRY(check_cuda(cudaOccupancyMaxActiveClusters(&n, kern, &cfg), "fwht virtual occupancy"));
    slot.occ = n;
    return MCK_OK;
  }));
  if (ds->occ < 1) return kNoClusterFits;
  int64_t nc = ds->occ;
  if (nc > rows) nc = rows;
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = config((unsigned)(nc * VR), at);
  MCK_TRY(check_cuda(cudaLaunchKernelEx(&cfg, kern, data, rows), "fwht_tmem_virtual_kernel launch"));
  return check_launch("fwht_tmem_virtual_kernel");
}

int launch_tmem_cluster(float* data, int64_t rows, int logn, cudaStream_t st) {
  switch (logn) {
    case 17: return MCK_FWHT_VIRTUAL >= 2 ? launch_tmem_virtual_t<2>(data, rows, st) : launch_tmem_cluster_t<2>(data, rows, st);
    case 18: return MCK_FWHT_VIRTUAL >= 4 ? launch_tmem_virtual_t<4>(data, rows, st) : launch_tmem_cluster_t<4>(data, rows, st);
    case 19: return launch_tmem_cluster_t<8>(data, rows, st);
    case 20: return launch_tmem_cluster_t<16>(data, rows, st);
    default: return fail_value("internal: no TMEM cluster kernel for 2^%d", logn);
  }
}

// Second stream used to overlap phase B of chunk k with phase A of chunk k+1.
struct SideStreams {
  cudaStream_t s[16] = {};
};
static SideStreams g_side;

static int side_stream(cudaStream_t* out) {
  int dev = 0;
  MCK_TRY(check_cuda(cudaGetDevice(&dev), "device"));
  if (dev >= 16) return fail_value("device index out of range");
  if (!g_side.s[dev])
    MCK_TRY(check_cuda(cudaStreamCreateWithFlags(&g_side.s[dev], cudaStreamNonBlocking), "stream"));
  *out = g_side.s[dev];
  return MCK_OK;
}

// tiny rows: one thread per row, serial butterflies (n <= 4)
template <class V>
__global__ void fwht_tiny_kernel(V* data, int64_t rows, int n) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  V* p = data + r * n;
  for (int h = 1; h < n; h <<= 1)
    for (int i = 0; i < n; ++i)
      if (!(i & h)) { V a = p[i], b = p[i | h]; p[i] = a + b; p[i | h] = a - b; }
}


template <class V>
int fwht_fast(V* data, int64_t rows, int64_t n, cudaStream_t st) {
  int logn = 0;
  while ((int64_t(1) << logn) < n) ++logn;
  if (rows == 0 || n == 1) return MCK_OK;
  const int max_row_logn = sizeof(V) == 4 ? 15 : 14;
  if (logn <= 2) {
    fwht_tiny_kernel<V><<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(data, rows, (int)n);
    return check_launch("fwht_tiny_kernel");
  }
  if constexpr (sizeof(V) == 4) {
#if MCK_FWHT_TMEM
    // enough rows for two per SM: the persistent kernel (0.93 -> 0.96 of HBM at 1 GiB)
    if (logn == 14 && rows >= 2 * 148) return launch_persistent14(data, rows, st);
    if (logn == 16) return launch_tmem_t<4>(data, rows, st);
    if (logn == 15) return launch_tmem_t<2>(data, rows, st);
    if (logn >= 17 && logn <= MCK_FWHT_TMEM_CLUSTER_MAX) {
      // where no such cluster can be resident the two-phase path below takes over
      const int rc = launch_tmem_cluster(data, rows, logn, st);
      if (rc != kNoClusterFits) return rc;
    }
#endif
  }
  if (logn <= max_row_logn) return launch_rows_by_logn<V>(data, rows, logn, st);
  const int logn2 = 14, logn1 = logn - logn2;
  if (logn1 > 6) return fail_value("length %lld exceeds the supported maximum 2^20", (long long)n);
  const int n2 = 1 << logn2;
  // Chunks of <= 24 MiB: phase B of a chunk finds phase A's output in L2.
  // Phase A of chunk k+1 (main stream) overlaps phase B of chunk k (side
  // stream); the caller's stream waits for the last phase B.
  int64_t chunk = (24ll << 20) / (n * (int64_t)sizeof(V));
  if (chunk < 1) chunk = 1;
  cudaStream_t side;
  MCK_TRY(side_stream(&side));
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  MCK_TRY(check_cuda(cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming), "event"));
  MCK_TRY(check_cuda(cudaEventRecord(ev_b, st), "event"));
  MCK_TRY(check_cuda(cudaStreamWaitEvent(side, ev_b, 0), "wait"));  // side starts after prior work
  int rc = MCK_OK;
  for (int64_t r0 = 0; r0 < rows && rc == MCK_OK; r0 += chunk) {
    const int64_t nr = rows - r0 < chunk ? rows - r0 : chunk;
    V* p = data + r0 * n;
    rc = launch_cols<V>(p, nr, logn1, n2, st);
    if (rc != MCK_OK) break;
    if (!ev_a) rc = check_cuda(cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming), "event");
    if (rc == MCK_OK) rc = check_cuda(cudaEventRecord(ev_a, st), "event");
    if (rc == MCK_OK) rc = check_cuda(cudaStreamWaitEvent(side, ev_a, 0), "wait");
    // phase B: the persistent 2^14 kernel when the chunk has two segments per
    // SM (2^19 0.49 -> 0.54, 2^20 0.50 -> 0.52), else one CTA per segment
    if constexpr (sizeof(V) == 4) {
      if (rc == MCK_OK && (nr << logn1) >= 2 * 148) {
        rc = launch_persistent14(p, nr << logn1, side);
        continue;
      }
    }
    if (rc == MCK_OK) rc = launch_rows_by_logn<V>(p, nr << logn1, logn2, side);
  }
  if (rc == MCK_OK) rc = check_cuda(cudaEventRecord(ev_b, side), "event");
  if (rc == MCK_OK) rc = check_cuda(cudaStreamWaitEvent(st, ev_b, 0), "wait");
  if (ev_a) cudaEventDestroy(ev_a);
  cudaEventDestroy(ev_b);
  return rc;
}

// ---------------------------------------------------------------- parity
// Base chunks: y_j = sum_{k=0..B-1} H[k][j] x_k accumulated sequentially in
// fp32 (products by +-1 exact), one thread per output element.
__global__ void parity_base_kernel(float* __restrict__ data, int64_t chunks, int base) {
  extern __shared__ float sx[];
  const int64_t c = blockIdx.x;
  if (c >= chunks) return;
  float* p = data + c * base;
  for (int i = threadIdx.x; i < base; i += blockDim.x) sx[i] = p[i];
  __syncthreads();
  for (int j = threadIdx.x; j < base; j += blockDim.x) {
    float acc = 0.0f;
    for (int k = 0; k < base; ++k) {
      const float xk = sx[k];
      acc = (__popc((unsigned)(k & j)) & 1) ? acc - xk : acc + xk;
    }
    p[j] = acc;
  }
}

// One combine stage at span h: a' = a + b ; b' = a' - 2b  (wht.py:115-126).
__global__ void parity_combine_kernel(float* __restrict__ data, int64_t total_pairs, int64_t h) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total_pairs) return;
  const int64_t grp = t / h, off = t % h;
  float* a = data + grp * 2 * h + off;
  float* b = a + h;
  const float s = *a + *b;
  *a = s;
  *b = s - 2.0f * *b;
}

int fwht_parity(float* data, int64_t rows, int64_t n, cudaStream_t st) {
  if (rows == 0) return MCK_OK;
  const int base = n < 256 ? (int)n : 256;
  const int64_t chunks = rows * (n / base);
  // first element of the base: y_j starts at 0 + (+-x_0); adding to 0.0f is
  // exact, so this equals the BLAS accumulation order.
  parity_base_kernel<<<(unsigned)chunks, base < 256 ? base : 256, base * sizeof(float), st>>>(
      data, chunks, base);
  MCK_TRY(check_launch("parity_base_kernel"));
  const int64_t pairs = rows * n / 2;
  for (int64_t h = base; h < n; h <<= 1) {
    parity_combine_kernel<<<(unsigned)((pairs + 255) / 256), 256, 0, st>>>(data, pairs, h);
    MCK_TRY(check_launch("parity_combine_kernel"));
  }
  return MCK_OK;
}

template int fwht_fast<float>(float*, int64_t, int64_t, cudaStream_t);
template int fwht_fast<double>(double*, int64_t, int64_t, cudaStream_t);

}  // namespace mck
