// Internal host-side types of the hmx library (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <vector>

namespace hmx {

struct TreeNode {
  int64_t start, stop, level;
  int64_t child[2];  // -1 for leaves
  double lo[3], hi[3];
};

struct ClusterTree {
  int64_t n = 0;
  std::vector<int64_t> perm;  // perm[k] = original index at tree slot k
  std::vector<TreeNode> nodes;  // preorder, root = 0
};

struct BlockLeaf {
  int64_t kind;  // 0 dense, 1 admissible
  int64_t r0, r1, c0, c1;  // point ranges in tree order
  int64_t rnode, cnode;
};

int build_cluster_tree(const double* pts, int64_t n, int64_t n_leaf, ClusterTree& out);
int build_block_leaves(const ClusterTree& rows, const ClusterTree& cols, double eta, std::vector<BlockLeaf>& out);
bool admissible(const TreeNode& a, const TreeNode& b, double eta);

}  // namespace hmx
