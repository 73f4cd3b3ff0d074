// Edge colouring for the bank-conflict-free permutation (perm_color.cu).
#pragma once

#include <cstdint>

namespace mck {

// Proper 32-edge-colouring of a 32-regular bipartite multigraph with m nodes
// per side; edge e joins left l[e] to right r[e].  Returns false if the graph
// is not 32-regular (the result is verified before returning true).
bool edge_color32(int m, int64_t nedges, const int32_t* l, const int32_t* r, uint8_t* col);

}  // namespace mck
