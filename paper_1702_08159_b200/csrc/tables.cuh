// Device layout of the factor tables (one caller-owned buffer; offsets are
// 256-byte aligned).  Public part = the reference's FastfoodBlock arrays
// (fastfood.py:82-93) stacked over E blocks; private part = tables derived
// for the fused kernel's register layouts.
#pragma once

#include <cstdint>

namespace mck {

struct TablesView {
  int64_t n;
  int32_t E;
  // public
  float* b;        // [E][n]  +-1
  int32_t* perm;   // [E][n]  gather: out[i] = in[perm[i]]
  float* g;        // [E][n]
  float* c;        // [E][n]
  // private
  int32_t* perminv;  // [E][n]
  double* g64;       // [E][n]  float64 G before the cast (for |g|)
  double* gnorm;     // [E]
  float* cs;         // [E][n]  C*scale (scale folded when it is a power of two)
  uint32_t* bmask;   // [E][words][T]  sign bits in layout-L register order
  uint2* scat;       // [E][R][T]      {smem byte offset of element j's slot, bits of g[perm^-1[j]]}
  uint32_t* gcol;    // [E][R/4][T]    gather slot colours (4 bytes per word; n >= 1024)
  uint16_t* soff;    // [E][R/8][T][8] scatter slot byte offsets (n = 1024 two-row kernel)
  float* ggath;      // [E][R/4][T][4] g in the gather layout (n = 1024 two-row kernel)
  int32_t* flag;     // validation flag
};

inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

inline int64_t tables_layout(int64_t n, int32_t E, char* base, TablesView* tv) {
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    char* p = base ? base + off : nullptr;
    off += align256(bytes);
    return p;
  };
  const int64_t en = n * (int64_t)E;
  TablesView v{};
  v.n = n;
  v.E = E;
  v.b = (float*)take(en * 4);
  v.perm = (int32_t*)take(en * 4);
  v.g = (float*)take(en * 4);
  v.c = (float*)take(en * 4);
  v.perminv = (int32_t*)take(en * 4);
  v.g64 = (double*)take(en * 8);
  v.gnorm = (double*)take((int64_t)E * 8);
  v.cs = (float*)take(en * 4);
  // sign masks: at most one 32-bit word per 32 elements, rounded up per thread
  v.bmask = (uint32_t*)take(((en + 31) / 32 + (int64_t)E * 64) * 4);
  v.scat = (uint2*)take(en * 8);
  v.gcol = (uint32_t*)take(en);
  v.soff = (uint16_t*)take(en * 2);
  v.ggath = (float*)take(en * 4);
  v.flag = (int32_t*)take(16);
  if (tv) *tv = v;
  return off;
}

}  // namespace mck
