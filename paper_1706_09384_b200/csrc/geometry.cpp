// Native cluster tree + eta-admissible block partition (host C++), bit-exact
// with the reference geometry (/root/reference/pkg/src/hmatx/geometry.py).
//
// This is SURVEY.md 8(f) item 2: the reference builds the trees in Python
// (0.2-4 s per config); here it is a few ms.  Bit-exactness notes:
//  * cluster tree (geometry.py:182-220): tight box = exact min/max; split axis
//    = first argmax of (hi - lo); mid = 0.5 * (lo + hi); "coord <= mid" goes to
//    the lower child, stable partition of the range; if one side is empty,
//    stable argsort of the coordinates and the first half (by order) is lower,
//    still partitioned in position order (idx[lower], idx[~lower]).
//  * diam_box (geometry.py:94-96) is np.linalg.norm -> BLAS ddot, whose n=3
//    tail loop is the FMA chain fma(v2,v2, fma(v1,v1, v0*v0)) on OpenBLAS
//    0.3.30; dist_box (geometry.py:99-106) is
//    sqrt(((a0^2 + a1^2) + a2^2) + ((b0^2 + b1^2) + b2^2)) with x*x squares.
//    This file is compiled with -ffp-contract=off so only the explicit fma()
//    calls fuse.
//  * admissibility is strict: min(diam) < eta * dist (geometry.py:113).
//  * leaves() order (geometry.py:261-268) = stack DFS, children pushed in
//    row-major order, so the LAST child is visited first.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include "hmx_host.h"

namespace hmx {

static inline double diam_box(const double* lo, const double* hi) {
  const double v0 = hi[0] - lo[0], v1 = hi[1] - lo[1], v2 = hi[2] - lo[2];
  return std::sqrt(std::fma(v2, v2, std::fma(v1, v1, v0 * v0)));
}

static inline double dist_box(const double* alo, const double* ahi, const double* blo, const double* bhi) {
  double a[3], b[3];
  for (int k = 0; k < 3; ++k) {
    a[k] = std::max(alo[k] - bhi[k], 0.0);
    b[k] = std::max(blo[k] - ahi[k], 0.0);
  }
  const double sa = (a[0] * a[0] + a[1] * a[1]) + a[2] * a[2];
  const double sb = (b[0] * b[0] + b[1] * b[1]) + b[2] * b[2];
  return std::sqrt(sa + sb);
}

bool admissible(const TreeNode& a, const TreeNode& b, double eta) {
  const double da = diam_box(a.lo, a.hi), db = diam_box(b.lo, b.hi);
  return std::min(da, db) < eta * dist_box(a.lo, a.hi, b.lo, b.hi);
}

int build_cluster_tree(const double* pts, int64_t n, int64_t n_leaf, ClusterTree& out) {
  out.n = n;
  out.perm.resize(n);
  std::iota(out.perm.begin(), out.perm.end(), int64_t(0));
  out.nodes.clear();
  out.nodes.reserve(2 * n);
  struct Work {
    int64_t a, b, level, parent;
    int side;
  };
  std::vector<Work> stack{{0, n, 0, -1, 0}};
  std::vector<int64_t> lowbuf, highbuf;
  std::vector<char> low;
  std::vector<int64_t> order;
  while (!stack.empty()) {
    Work w = stack.back();
    stack.pop_back();
    TreeNode node;
    node.start = w.a;
    node.stop = w.b;
    node.level = w.level;
    node.child[0] = node.child[1] = -1;
    for (int k = 0; k < 3; ++k) {
      node.lo[k] = INFINITY;
      node.hi[k] = -INFINITY;
    }
    for (int64_t t = w.a; t < w.b; ++t) {
      const double* p = pts + 3 * out.perm[t];
      for (int k = 0; k < 3; ++k) {
        node.lo[k] = std::min(node.lo[k], p[k]);
        node.hi[k] = std::max(node.hi[k], p[k]);
      }
    }
    const int64_t v = (int64_t)out.nodes.size();
    out.nodes.push_back(node);
    if (w.parent >= 0) out.nodes[w.parent].child[w.side] = v;
    const int64_t cnt = w.b - w.a;
    if (cnt <= n_leaf) continue;
    int axis = 0;
    double ext = node.hi[0] - node.lo[0];
    for (int k = 1; k < 3; ++k) {
      const double e = node.hi[k] - node.lo[k];
      if (e > ext) {
        ext = e;
        axis = k;
      }
    }
    const double mid = 0.5 * (node.lo[axis] + node.hi[axis]);
    low.assign(cnt, 0);
    int64_t nlow = 0;
    for (int64_t t = 0; t < cnt; ++t) {
      low[t] = pts[3 * out.perm[w.a + t] + axis] <= mid;
      nlow += low[t];
    }
    if (nlow == 0 || nlow == cnt) {
      order.resize(cnt);
      std::iota(order.begin(), order.end(), int64_t(0));
      std::stable_sort(order.begin(), order.end(), [&](int64_t p, int64_t q) {
        return pts[3 * out.perm[w.a + p] + axis] < pts[3 * out.perm[w.a + q] + axis];
      });
      std::fill(low.begin(), low.end(), 0);
      for (int64_t t = 0; t < cnt / 2; ++t) low[order[t]] = 1;
      nlow = cnt / 2;
    }
    lowbuf.clear();
    highbuf.clear();
    for (int64_t t = 0; t < cnt; ++t) (low[t] ? lowbuf : highbuf).push_back(out.perm[w.a + t]);
    std::copy(lowbuf.begin(), lowbuf.end(), out.perm.begin() + w.a);
    std::copy(highbuf.begin(), highbuf.end(), out.perm.begin() + w.a + nlow);
    const int64_t cut = w.a + nlow;
    stack.push_back({cut, w.b, w.level + 1, v, 1});
    stack.push_back({w.a, cut, w.level + 1, v, 0});
  }
  return 0;
}

int build_block_leaves(const ClusterTree& rows, const ClusterTree& cols, double eta, std::vector<BlockLeaf>& out) {
  out.clear();
  std::vector<std::pair<int64_t, int64_t>> stack{{0, 0}};
  while (!stack.empty()) {
    auto [r, c] = stack.back();
    stack.pop_back();
    const TreeNode& R = rows.nodes[r];
    const TreeNode& C = cols.nodes[c];
    if (admissible(R, C, eta)) {
      out.push_back({1, R.start, R.stop, C.start, C.stop, r, c});
      continue;
    }
    const bool rl = R.child[0] < 0, cl = C.child[0] < 0;
    if (rl && cl) {
      out.push_back({0, R.start, R.stop, C.start, C.stop, r, c});
      continue;
    }
    int64_t rk[2] = {r, -1}, ck[2] = {c, -1};
    int nr = 1, nc = 1;
    if (!rl) {
      rk[0] = R.child[0];
      rk[1] = R.child[1];
      nr = 2;
    }
    if (!cl) {
      ck[0] = C.child[0];
      ck[1] = C.child[1];
      nc = 2;
    }
    for (int a = 0; a < nr; ++a)
      for (int b = 0; b < nc; ++b) stack.push_back({rk[a], ck[b]});
  }
  return 0;
}

}  // namespace hmx
