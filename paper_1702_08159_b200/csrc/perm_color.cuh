// Edge colouring for the bank-conflict-free permutation (perm_color.cu).
#pragma once

#include <cstdint>

namespace mck {

// Proper 2^levels-edge-colouring of a 2^levels-regular bipartite multigraph
// with m nodes per side; edge e joins left l[e] to right r[e].  Returns false
// if the graph is not regular (the result is verified before returning true).
bool edge_color_pow2(int m, int levels, int64_t nedges, const int32_t* l, const int32_t* r,
                     uint8_t* col);

}  // namespace mck
