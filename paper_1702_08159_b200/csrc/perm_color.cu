// Bank-conflict-free shared-memory permutation (setup-time host code).
//
// The fused kernel moves the H1 output through shared memory to apply Pi
// (fastfood.py:192).  A warp's scatter instruction writes the 32 elements of
// one "scatter group" (32 lanes x one register), a gather instruction reads
// the 32 elements of one "gather group".  Element i joins scatter group S(i)
// to gather group G(perm^-1 i): a 32-regular bipartite multigraph with n/32
// nodes per side.  A proper 32-edge-colouring (always exists, Koenig) gives
// every element a bank c(i) such that each scatter and each gather touches
// 32 distinct banks; the element's slot is 32*G + c(i).
//
// Colouring by repeated Euler splits: in a 2^k-regular bipartite multigraph,
// walking closed trails and sending left->right edges to one half and
// right->left edges to the other leaves two 2^(k-1)-regular halves; k
// levels give 2^k perfect matchings = colours.  O(n k) per block.  Degree 32
// serves one-row warps (4-byte slots), degree 16 the two-row kernel's
// half-warp phases (8-byte slots).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "perm_color.cuh"

namespace mck {

bool edge_color_pow2(int m, int levels, int64_t nedges, const int32_t* l, const int32_t* r,
                     uint8_t* col) {
  const int deg = 1 << levels;
  if (levels < 0 || levels > 7 || nedges != (int64_t)m * deg) return false;
  const int64_t n = nedges;
  std::vector<int32_t> cls(n, 0);
  std::vector<int32_t> start, fill, adj(2 * n);
  std::vector<uint8_t> used(n), side(n);
  for (int lev = 0; lev < levels; ++lev) {
    const int64_t keys = ((int64_t)1 << lev) * 2 * m;
    auto key_l = [&](int64_t e) { return (int64_t)cls[e] * 2 * m + l[e]; };
    auto key_r = [&](int64_t e) { return (int64_t)cls[e] * 2 * m + m + r[e]; };
    start.assign(keys + 1, 0);
    for (int64_t e = 0; e < n; ++e) {
      ++start[key_l(e) + 1];
      ++start[key_r(e) + 1];
    }
    for (int64_t k = 0; k < keys; ++k) start[k + 1] += start[k];
    fill.assign(start.begin(), start.end() - 1);
    for (int64_t e = 0; e < n; ++e) {
      adj[fill[key_l(e)]++] = (int32_t)e;
      adj[fill[key_r(e)]++] = (int32_t)e;
    }
    std::vector<int64_t> ptr(start.begin(), start.end() - 1);
    std::fill(used.begin(), used.end(), 0);
    for (int64_t e0 = 0; e0 < n; ++e0) {
      if (used[e0]) continue;
      int64_t u = key_l(e0);
      for (;;) {
        while (ptr[u] < start[u + 1] && used[adj[ptr[u]]]) ++ptr[u];
        if (ptr[u] == start[u + 1]) break;  // closed trail (even degrees)
        const int64_t e = adj[ptr[u]++];
        used[e] = 1;
        const bool left = (u % (2 * m)) < m;
        side[e] = left ? 0 : 1;
        u = left ? key_r(e) : key_l(e);
      }
    }
    for (int64_t e = 0; e < n; ++e) cls[e] = 2 * cls[e] + side[e];
  }
  // verify: every (node, colour) pair used exactly once on both sides
  std::vector<uint8_t> seen((size_t)m * deg * 2, 0);
  for (int64_t e = 0; e < n; ++e) {
    if (l[e] < 0 || l[e] >= m || r[e] < 0 || r[e] >= m) return false;
    uint8_t& a = seen[((size_t)l[e] * deg + cls[e]) * 2];
    uint8_t& b = seen[((size_t)r[e] * deg + cls[e]) * 2 + 1];
    if (a || b) return false;
    a = b = 1;
    col[e] = (uint8_t)cls[e];
  }
  return true;
}

}  // namespace mck

extern "C" int mck_diag_edge_color32(int32_t m, const int32_t* l, const int32_t* r, uint8_t* col) {
  return mck::edge_color_pow2(m, 5, (int64_t)m * 32, l, r, col) ? 0 : 1;
}
