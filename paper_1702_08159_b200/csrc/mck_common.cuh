// Common device/host helpers for the B200 Fastfood library.
//
// * fmix64 / stream keys: the reference's pinned mixer
//   (pkg/src/mckernel/detrand.py:60-93, pkg/README.md:78-108).
// * pairwise float64 summation in numpy's exact order (used wherever the
//   reference reduces with ndarray.sum over a contiguous axis:
//   fastfood.py:103,107,128, detrand.py:208).
// * error state for the C ABI (mck_last_error).
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>
#include <utility>
#include <cuda_runtime.h>

#include "../../include/mckernel_b200.h"

namespace mck {

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int fail_value(const char* fmt, ...);   // returns MCK_ERR_VALUE
int check_cuda(cudaError_t e, const char* what);  // MCK_OK or MCK_ERR_CUDA
int check_launch(const char* what);

#define MCK_TRY(expr)                                   \
  do {                                                  \
    int _rc = (expr);                                   \
    if (_rc != MCK_OK) return _rc;                      \
  } while (0)

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: kernels of the hot loops are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs may
// become resident while its predecessor in the stream drains.  Every such
// kernel calls pdl_wait() before it touches memory a predecessor may write
// or read (griddepcontrol.wait returns once the predecessor grid completed
// and its writes are visible), then pdl_trigger() so that its own successor
// can be scheduled; code before pdl_wait() touches only constant inputs and
// on-chip state.  Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <class... KArgs, class... Args>
int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
               const char* what, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  MCK_TRY(check_cuda(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), what));
  return check_launch(what);
}

// ---------------------------------------------------------------- per-device setup
// Kernel attributes (cudaFuncSetAttribute) and occupancy are per device, so a
// launcher's one-time setup is cached per device index, and the first call on
// each device runs it under a lock (launchers may be called from several host
// threads).  `init(dev, slot)` fills the slot and returns an MCK status.
constexpr int kMaxDevices = 64;

struct DeviceSlot {
  int occ = 0;   // resident CTAs per SM of the kernel
  int sms = 0;   // multiprocessor count of the device
};

struct PerDevice {
  std::atomic<bool> ready[kMaxDevices] = {};
  DeviceSlot slot[kMaxDevices];
  std::mutex mu;
};

template <class F>
int per_device(PerDevice& pd, const DeviceSlot** out, F&& init) {
  int dev = 0;
  MCK_TRY(check_cuda(cudaGetDevice(&dev), "device"));
  if (dev < 0 || dev >= kMaxDevices) return fail_value("device index %d out of range", dev);
  if (!pd.ready[dev].load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lk(pd.mu);
    if (!pd.ready[dev].load(std::memory_order_relaxed)) {
      DeviceSlot s;
      MCK_TRY(check_cuda(cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, dev), "sms"));
      MCK_TRY(init(dev, s));
      pd.slot[dev] = s;
      pd.ready[dev].store(true, std::memory_order_release);
    }
  }
  *out = &pd.slot[dev];
  return MCK_OK;
}

// ---------------------------------------------------------------- z tiles
// Tiled layout of a fused-path z group tile with `cols` columns (config 4):
// [row / 128][col / 2^L][row % 128][col % 2^L], L = MCK_ZT_LOG = 5: each
// row piece is one 128-byte line and 128 rows x 32 z form a contiguous 16 KB
// unit.  The z producer writes whole lines (8 threads per line), the
// backward contraction reads 8-row runs of whole lines and the forward reads
// [128 rows][8 z] slices of a unit.  Measured (c4 step): L = 3 2.91 ms,
// L = 4 2.77, L = 5 2.76; row-major tiles 3.1 ms.  The tile is allocated for
// m rounded up to 128 rows.
#ifndef MCK_ZT_LOG
#define MCK_ZT_LOG 5
#endif
__host__ __device__ __forceinline__ int64_t zt_offset(int64_t cols, int64_t row, int64_t col) {
  constexpr int L = MCK_ZT_LOG;
  return ((((row >> 7) * (cols >> L)) + (col >> L)) << (7 + L)) + ((row & 127) << L) +
         (col & ((1 << L) - 1));
}

// ---------------------------------------------------------------- hashing
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kFmixC1 = 0xFF51AFD7ED558CCDull;
constexpr uint64_t kFmixC2 = 0xC4CEB9FE1A85EC53ull;
constexpr uint64_t kFnvOffset = 0xCBF29CE484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001B3ull;
constexpr double kTwoM53 = 1.1102230246251565e-16;  // 2^-53

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 33;
  z *= kFmixC1;
  z ^= z >> 33;
  z *= kFmixC2;
  z ^= z >> 33;
  return z;
}

inline uint64_t fnv1a64(const char* s) {
  uint64_t h = kFnvOffset;
  for (; *s; ++s) h = (h ^ static_cast<unsigned char>(*s)) * kFnvPrime;
  return h;
}

// detrand.py:78-83
inline uint64_t stream_key(uint64_t seed, const char* label, uint64_t block) {
  uint64_t k = fmix64(seed);
  k = fmix64(k ^ fnv1a64(label));
  return fmix64(k ^ (block * kGamma));
}

// Draw at counter c of the stream with key `key` (detrand.py:126,131).
__host__ __device__ __forceinline__ uint64_t draw(uint64_t key, uint64_t c) {
  return fmix64(key + c * kGamma);
}

// detrand.py:142: top 53 bits scaled to [0, 1).
__host__ __device__ __forceinline__ double uniform01(uint64_t key, uint64_t c) {
  return static_cast<double>(draw(key, c) >> 11) * kTwoM53;
}

// detrand.py:174-183: one Box-Muller pair from uniforms at counters
// (2p, 2p+1) relative to `base`.  2*pi is rounded first, as numpy's
// `2.0 * np.pi * u2` is evaluated left to right.
__device__ __forceinline__ void box_muller(double u1, double u2, double& z0, double& z1) {
  if (u1 == 0.0) u1 = kTwoM53;
  const double r = sqrt(-2.0 * log(u1));
  const double ang = (2.0 * 3.141592653589793) * u2;
  double s, c;
  sincos(ang, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

__device__ __forceinline__ void gauss_pair(uint64_t key, uint64_t ucounter, double& z0, double& z1) {
  box_muller(uniform01(key, ucounter), uniform01(key, ucounter + 1), z0, z1);
}

// ---------------------------------------------------------------- pairwise sums
// numpy pairwise_sum (float64, contiguous): n < 8 sequential; n <= 128 eight
// strided accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the
// n%8 tail; otherwise split at n2 = (n/2) rounded down to a multiple of 8.
// Serial, any n.  Used for small n and as the building block of the warp
// version below.  `get(i)` returns element i.
template <class Get>
__device__ double pairwise_serial(Get get, int64_t lo, int64_t n) {
  // explicit stack instead of recursion
  struct Frame { int64_t lo, n; int state; double left; };
  Frame st[40];
  int sp = 0;
  st[0] = {lo, n, 0, 0.0};
  double ret = 0.0;
  while (true) {
    Frame& f = st[sp];
    if (f.state == 0) {
      if (f.n < 8) {
        double r = 0.0;  // numpy starts from 0. (sign of zero is irrelevant here)
        for (int64_t i = 0; i < f.n; ++i) r += get(f.lo + i);
        ret = r;
      } else if (f.n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = get(f.lo + j);
        int64_t m = f.n - (f.n % 8);
        for (int64_t i = 8; i < m; i += 8)
          for (int j = 0; j < 8; ++j) r[j] += get(f.lo + i + j);
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (int64_t i = m; i < f.n; ++i) res += get(f.lo + i);
        ret = res;
      } else {
        int64_t n2 = f.n / 2;
        n2 -= n2 % 8;
        f.state = 1;
        st[++sp] = {f.lo, n2, 0, 0.0};
        continue;
      }
    } else if (f.state == 1) {
      f.left = ret;
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      f.state = 2;
      st[++sp] = {f.lo + n2, f.n - n2, 0, 0.0};
      continue;
    } else {
      ret = f.left + ret;
    }
    if (sp == 0) return ret;
    --sp;
  }
}

// Warp-cooperative pairwise sum for a power-of-two n >= 1024 (so that the
// numpy tree is a balanced tree of n/128 leaves of 128 elements, each leaf
// eight 16-term strided accumulators).  Lane = 4*g + q: lane-group g (0..7)
// owns a contiguous run of n/1024 leaves, slot q (0..3) owns accumulators
// 2q and 2q+1 of each leaf.  `pair(p, a, b)` returns elements 2p and 2p+1.
// Result is returned in every lane.
template <class Pair>
__device__ double pairwise_warp_pow2(Pair pair, int64_t n, int lane) {
  const int g = lane >> 2, q = lane & 3;
  const int64_t leaves_per_group = n / 1024;
  const int64_t leaf0 = g * leaves_per_group;
  // binary-counter stack for the balanced combination of consecutive leaves
  double stack[24];
  int level[24];
  int sp = 0;
  for (int64_t lf = 0; lf < leaves_per_group; ++lf) {
    const int64_t base = (leaf0 + lf) * 128;  // element index of the leaf
    double r0 = 0.0, r1 = 0.0;
    for (int i = 0; i < 16; ++i) {
      double a, b;
      pair((base + 8 * i + 2 * q) >> 1, a, b);
      if (i == 0) { r0 = a; r1 = b; } else { r0 += a; r1 += b; }
    }
    double v = r0 + r1;                                   // r[2q] + r[2q+1]
    v = v + __shfl_xor_sync(0xffffffffu, v, 1);           // (r0+r1)+(r2+r3)
    v = v + __shfl_xor_sync(0xffffffffu, v, 2);           // ... + ((r4+r5)+(r6+r7))
    stack[sp] = v;
    level[sp] = 0;
    ++sp;
    while (sp >= 2 && level[sp - 1] == level[sp - 2]) {
      stack[sp - 2] = stack[sp - 2] + stack[sp - 1];
      level[sp - 2] += 1;
      --sp;
    }
  }
  double v = stack[0];
  v = v + __shfl_xor_sync(0xffffffffu, v, 4);
  v = v + __shfl_xor_sync(0xffffffffu, v, 8);
  v = v + __shfl_xor_sync(0xffffffffu, v, 16);
  return v;
}


// ---------------------------------------------------------------- L2 policy stores
// Stores tagged with an L2 eviction-priority policy (createpolicy): used to keep
// an intermediate (FWHT column pass, fused-path z tile) resident for its
// consumer kernel.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_hint(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(float2* p, float2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y),
               "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
               "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}


}  // namespace mck
