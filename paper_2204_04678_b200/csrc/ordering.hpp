// Native nested dissection (ordering.cpp): the reference's ordering.py
// algorithm restated in C++, plus the separator-aligned tile partition.
#pragma once
#include <cstdint>
#include <vector>

namespace pinla {

struct NDNode {  // ordering.py:99-115 TreeNode
  int64_t start = 0, end = 0, span_start = 0;
  int parent = -1;
  bool leaf = true;
  std::vector<int> children;
};

struct NDResult {
  std::vector<int64_t> perm;  // new -> old
  std::vector<NDNode> nodes;  // reference node order (emission order)
  int root = 0;
  int64_t n_dense = 0;        // peeled dense vertices (last, in the root separator)
};

NDResult nested_dissection(int64_t n, const int64_t* indptr, const int64_t* indices,
                           int64_t leaf_cutoff);
std::vector<int64_t> nd_tile_bounds(const NDResult& r, int64_t tile_max);
void scalar_pattern(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* perm,
                    std::vector<int64_t>& Lp, std::vector<int64_t>& Li);

}  // namespace pinla
