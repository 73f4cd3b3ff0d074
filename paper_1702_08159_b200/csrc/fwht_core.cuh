// Register-resident Walsh-Hadamard core for one row of N = 2^LOGN elements
// held by a group of T = N / R threads (R = 2^LOGR elements per thread).
//
// The unnormalised transform is the tensor product of independent 2-point
// butterflies on every index bit, so stages commute: a thread butterflies
// whichever LOGR index bits it currently holds in registers ("a round"),
// then the group exchanges elements through shared memory so that other bits
// become register-resident.  A row therefore costs one coalesced global read
// and one global write plus ceil(log2(T)/LOGR) shared-memory exchanges.
//
// Layouts (register bit set P; thread-id bits fill the remaining bits in
// ascending order):
//   L  : P = {0,1} U top (LOGR-2) bits  -> 16-byte vector global access,
//        lanes on bits 2..6 (coalesced 512 B per warp instruction)
//   M_j: P = middle bits 2+j*LOGR ... (plus unused "filler" high bits when
//        fewer than LOGR middle bits remain)
// Shared memory uses one pad word per 32 (addr = i + i/32), which makes every
// layout above bank-conflict free for scalar LDS/STS.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mck {

__host__ __device__ constexpr uint32_t deposit_bits(uint32_t v, uint32_t mask) {
  uint32_t out = 0;
  int src = 0;
  for (int b = 0; b < 32; ++b) {
    if (mask & (1u << b)) {
      if (v & (1u << src)) out |= 1u << b;
      ++src;
    }
  }
  return out;
}

__host__ __device__ constexpr int popcount_c(uint32_t m) {
  int c = 0;
  for (int b = 0; b < 32; ++b) c += (m >> b) & 1u;
  return c;
}

// Padded shared-memory address: one word per 32 plus four per 1024.  Checked
// by exhaustive simulation to make every layout of RowCfg<10..15, 5> and
// RowCfg<12..14, 6> bank-conflict free for scalar LDS/STS.
__host__ __device__ __forceinline__ constexpr uint32_t pad_addr(uint32_t i) {
  return i + (i >> 5) + 4 * (i >> 10);
}

template <int LOGN_, int LOGR_>
struct RowCfg {
  static constexpr int LOGN = LOGN_;
  static constexpr int LOGR = LOGR_;
  static constexpr int N = 1 << LOGN;
  static constexpr int R = 1 << LOGR;
  static constexpr int LOGT = LOGN - LOGR;
  static constexpr int T = 1 << LOGT;
  static constexpr uint32_t FULL = (uint32_t)N - 1u;
  static_assert(LOGR >= 2 && LOGN >= LOGR + 1, "row config");
  // layout L
  static constexpr uint32_t PL =
      3u | ((((1u << (LOGR - 2)) - 1u)) << (LOGN - LOGR + 2));
  // middle bits 2 .. 2+LOGT-1
  static constexpr int NMID = (LOGT + LOGR - 1) / LOGR;
  static constexpr int SMEM_FLOATS = N + N / 32 + N / 256 + 4;  // padded row (pad_addr)

  // Active (butterflied) middle bits of round j.
  __host__ __device__ static constexpr uint32_t mid_active(int j) {
    int lo = 2 + j * LOGR;
    int hi = lo + LOGR;
    if (hi > 2 + LOGT) hi = 2 + LOGT;
    uint32_t m = 0;
    for (int b = lo; b < hi; ++b) m |= 1u << b;
    return m;
  }
  // Register bits of middle round j: active bits plus passenger ("filler")
  // bits -- the highest bits not butterflied in this round -- so that every
  // round holds R values and the lanes stay on the low index bits.
  __host__ __device__ static constexpr uint32_t mid_regs(int j) {
    uint32_t m = mid_active(j);
    int need = LOGR - popcount_c(m);
    for (int b = LOGN - 1; need > 0 && b >= 0; --b) {
      if (!(m & (1u << b))) {  // any bit not butterflied in this round
        m |= 1u << b;
        --need;
      }
    }
    return m;
  }
  __host__ __device__ static constexpr uint32_t mid_active_all() {
    uint32_t m = 0;
    for (int b = 2; b < 2 + LOGT; ++b) m |= 1u << b;
    return m;
  }
};

// Element index of register k in a layout with register mask P, for a thread
// whose thread-bit contribution is `tpart` (= deposit(tid, ~P)).
template <uint32_t P>
__device__ __forceinline__ uint32_t lay_index(uint32_t tpart, int k) {
  return tpart | deposit_bits((uint32_t)k, P);
}

template <uint32_t FULL, uint32_t P>
__device__ __forceinline__ uint32_t thread_part(uint32_t tid) {
  return deposit_bits(tid, FULL & ~P);
}

// Packed fp32 pair butterfly (a0,a1) <- (a0,a1)+(b0,b1), (b0,b1) <- (a0,a1)-(b0,b1):
// sm_100 FADD2 does two lanes' worth of adds per instruction.
__device__ __forceinline__ void bfly_pk(float& a0, float& a1, float& b0, float& b1) {
  unsigned long long A, B, S, D;
  asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(S) : "l"(A), "l"(B));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a0), "=f"(a1) : "l"(S));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(b0), "=f"(b1) : "l"(D));
}

// (a0,a1) *= (b0,b1) with one FMUL2.
__device__ __forceinline__ void mul_pk(float& a0, float& a1, float b0, float b1) {
  unsigned long long A, B, M;
  asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(M) : "l"(A), "l"(B));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a0), "=f"(a1) : "l"(M));
}

// Butterflies over the register-index bits whose deposited index bit is in
// ACTIVE (a subset of P).  For fp32, stages on register bits >= 1 combine
// register pairs (2m, 2m+1) with packed FADD2; the stage on register bit 0
// (inside a pair) stays scalar.
template <int R, uint32_t P, uint32_t ACTIVE, class V>
__device__ __forceinline__ void butterflies(V (&v)[R]) {
#pragma unroll
  for (int a = 0; (1 << a) < R; ++a) {
    if (ACTIVE & deposit_bits(1u << a, P)) {
      if constexpr (sizeof(V) == 4) {
        if (a >= 1) {
#pragma unroll
          for (int k = 0; k < R; k += 2)
            if (!(k & (1 << a))) bfly_pk(v[k], v[k + 1], v[k | (1 << a)], v[(k | (1 << a)) + 1]);
          continue;
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (!(k & (1 << a))) {
          V x = v[k], y = v[k | (1 << a)];
          v[k] = x + y;
          v[k | (1 << a)] = x - y;
        }
      }
    }
  }
}

// pad_addr is additive over disjoint bit sets (no carries between them), so
// the address splits into a per-thread base plus a compile-time offset per
// register: one base register, immediate offsets in every LDS/STS.
template <int R, uint32_t P, class V>
__device__ __forceinline__ void sts_layout(V* s, uint32_t tpart, const V (&v)[R]) {
  V* base = s + pad_addr(tpart);
#pragma unroll
  for (int k = 0; k < R; ++k) base[pad_addr(deposit_bits((uint32_t)k, P))] = v[k];
}

template <int R, uint32_t P, class V>
__device__ __forceinline__ void lds_layout(const V* s, uint32_t tpart, V (&v)[R]) {
  const V* base = s + pad_addr(tpart);
#pragma unroll
  for (int k = 0; k < R; ++k) v[k] = base[pad_addr(deposit_bits((uint32_t)k, P))];
}

// Group barrier for T threads that start at a multiple of T inside the CTA.
template <int T>
__device__ __forceinline__ void group_sync(int group_id) {
  if constexpr (T <= 32) {
    __syncwarp();
  } else {
    // named barrier per group (ids 1..15); T threads participate
    asm volatile("bar.sync %0, %1;" ::"r"(group_id + 1), "r"(T) : "memory");
  }
}

// Middle rounds, compile-time recursion over j: exchange from layout PREV
// into round j, butterfly its active bits.
template <class C, int J, uint32_t PREV, int R, class V>
__device__ __forceinline__ void middle_rounds(V* s, uint32_t tid, int gid, V (&v)[R]) {
  if constexpr (J < C::NMID) {
    constexpr uint32_t PJ = C::mid_regs(J);
    constexpr uint32_t AJ = C::mid_active(J);
    sts_layout<R, PREV>(s, thread_part<C::FULL, PREV>(tid), v);
    group_sync<C::T>(gid);
    lds_layout<R, PJ>(s, thread_part<C::FULL, PJ>(tid), v);
    group_sync<C::T>(gid);
    butterflies<R, PJ, AJ>(v);
    middle_rounds<C, J + 1, PJ, R>(s, tid, gid, v);
  }
}

// Middle rounds over two alternating exchange buffers: round j uses buffer
// j & 1, so the barrier of the following exchange also protects this one's
// buffer and each exchange needs a single barrier.  Fast warps then run their
// butterflies and next stores while slower warps are still loading.  Needs an
// even number of exchanges per pass (the caller repeats passes back to back).
template <class C, int J, uint32_t PREV, int R, class V>
__device__ __forceinline__ void middle_rounds_2buf(V* s0, V* s1, uint32_t tid, int gid, V (&v)[R]) {
  static_assert(C::NMID % 2 == 0, "alternating buffers need an even number of exchanges");
  if constexpr (J < C::NMID) {
    constexpr uint32_t PJ = C::mid_regs(J);
    constexpr uint32_t AJ = C::mid_active(J);
    V* s = (J & 1) ? s1 : s0;
    sts_layout<R, PREV>(s, thread_part<C::FULL, PREV>(tid), v);
    group_sync<C::T>(gid);
    lds_layout<R, PJ>(s, thread_part<C::FULL, PJ>(tid), v);
    butterflies<R, PJ, AJ>(v);
    middle_rounds_2buf<C, J + 1, PJ, R>(s0, s1, tid, gid, v);
  }
}

// Register mask of the last middle round (the layout the row is in after
// middle_rounds<C, 0, ...>).
template <class C>
__host__ __device__ constexpr uint32_t last_mid_regs() {
  return C::mid_regs(C::NMID - 1);
}

// Reverse order for the second transform of the Fastfood block: middle
// rounds first (starting from data already laid out in round 0's registers),
// finishing with an exchange back to layout L.
template <class C, int J, int R, class V>
__device__ __forceinline__ void middle_rounds_then_L(V* s, uint32_t tid, int gid, V (&v)[R]) {
  constexpr uint32_t PJ = C::mid_regs(J);
  butterflies<R, PJ, C::mid_active(J)>(v);
  if constexpr (J + 1 < C::NMID) {
    constexpr uint32_t PN = C::mid_regs(J + 1);
    sts_layout<R, PJ>(s, thread_part<C::FULL, PJ>(tid), v);
    group_sync<C::T>(gid);
    lds_layout<R, PN>(s, thread_part<C::FULL, PN>(tid), v);
    group_sync<C::T>(gid);
    middle_rounds_then_L<C, J + 1, R>(s, tid, gid, v);
  } else {
    sts_layout<R, PJ>(s, thread_part<C::FULL, PJ>(tid), v);
    group_sync<C::T>(gid);
    lds_layout<R, C::PL>(s, thread_part<C::FULL, C::PL>(tid), v);
    group_sync<C::T>(gid);
  }
}

}  // namespace mck
