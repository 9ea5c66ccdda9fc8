"""Oracle: point clouds, cluster tree and block partition (CPU).  TEST INFRASTRUCTURE.

Restates ``/root/reference/pkg/src/hmatx/geometry.py`` with flat arrays
instead of node objects:

* ``sphere_cloud`` / ``plate_cloud`` -- ``make_geometry`` (``geometry.py:310-344``)
* ``diam_box`` / ``dist_box`` / ``is_admissible`` -- ``geometry.py:94-113``
  (the same numpy calls, so the same rounding: ``np.linalg.norm`` -> BLAS dot
  for the diameter, ``sqrt(sum(gap**2) + sum(gap**2))`` for the distance;
  strict ``<`` in the admissibility test, ``geometry.py:113``)
* ``cluster_tree`` -- ``build_cluster_tree`` (``geometry.py:182-220``): tight
  box, longest axis (first on ties), midpoint split with ``<= mid`` to the lower
  child, stable median fallback, preorder node numbering.
* ``block_leaves`` -- ``build_block_tree`` + ``BlockTree.leaves``
  (``geometry.py:261-295``): leaves in the reference's stack order (last child
  first).

Pinned bit-exact (permutation, node ranges, leaf list) against the reference
module and ``tests/golden/geometry_*.npz`` by ``tests/test_oracle_pins.py``.
"""

from dataclasses import dataclass

import numpy as np

DENSE, ADMISSIBLE = 0, 1


def sphere_cloud(n, radius=1.0):
    """Fibonacci-spiral sphere points and radial normals (``geometry.py:332-343``)."""
    if radius <= 0:
        raise ValueError("size must be positive")
    if n < 1:
        raise ValueError("count must be positive")
    rad = float(radius)
    if n == 1:
        pts = np.array([[0.0, 0.0, rad]])
    else:
        k = np.arange(n)
        z = 1.0 - 2.0 * (k + 0.5) / n
        phi = k * np.pi * (3.0 - np.sqrt(5.0))
        rho = np.sqrt(1.0 - z**2)
        pts = rad * np.column_stack([rho * np.cos(phi), rho * np.sin(phi), z])
    nrm = pts / np.linalg.norm(pts, axis=1)[:, None]
    return np.ascontiguousarray(pts), np.ascontiguousarray(nrm)


def plate_cloud(n, half_width=1.0):
    """Uniform n x n grid on [-a,a]^2 x {0}, normals (0,0,1) (``geometry.py:325-331``)."""
    if half_width <= 0:
        raise ValueError("size must be positive")
    if n < 1:
        raise ValueError("count must be positive")
    ax = np.linspace(-float(half_width), float(half_width), n)
    g1, g2 = np.meshgrid(ax, ax, indexing="ij")
    pts = np.column_stack([g1.ravel(), g2.ravel(), np.zeros(n * n)])
    return pts, np.tile([0.0, 0.0, 1.0], (n * n, 1))


def diam_box(lo, hi):
    """Box diagonal length (``geometry.py:94-96``)."""
    return float(np.linalg.norm(hi - lo))


def dist_box(alo, ahi, blo, bhi):
    """Closest-face box distance (``geometry.py:99-106``)."""
    g1 = np.maximum(alo - bhi, 0.0)
    g2 = np.maximum(blo - ahi, 0.0)
    return float(np.sqrt(np.sum(g1**2) + np.sum(g2**2)))


def is_admissible(alo, ahi, blo, bhi, eta):
    """min(diam) < eta * dist, strict (``geometry.py:109-113``)."""
    if eta <= 0:
        raise ValueError("eta must be positive")
    return min(diam_box(alo, ahi), diam_box(blo, bhi)) < eta * dist_box(alo, ahi, blo, bhi)


@dataclass
class OracleClusterTree:
    """Flat preorder cluster tree.  ``perm[k]`` = original index at tree slot k."""

    perm: np.ndarray      # (N,) int64
    start: np.ndarray     # (nodes,) int64
    stop: np.ndarray      # (nodes,) int64
    lo: np.ndarray        # (nodes, 3) f64 tight box minima
    hi: np.ndarray        # (nodes, 3) f64 tight box maxima
    level: np.ndarray     # (nodes,) int64
    child: np.ndarray     # (nodes, 2) int64, -1 for leaves
    points_tree: np.ndarray

    def is_leaf(self, v):
        return self.child[v, 0] < 0


def cluster_tree(points, n_leaf):
    """Midpoint-bisection cluster tree (``geometry.py:182-220``)."""
    if n_leaf < 1:
        raise ValueError("n_leaf must be >= 1")
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.shape[0] == 0:
        raise ValueError("empty input")
    n = pts.shape[0]
    perm = np.arange(n)
    start, stop, lo, hi, level, child = [], [], [], [], [], []

    def new_node(a, b, lev, blo, bhi):
        start.append(a); stop.append(b); level.append(lev)
        lo.append(blo); hi.append(bhi); child.append([-1, -1])
        return len(start) - 1

    # explicit preorder: (range, level, parent slot to patch)
    work = [(0, n, 0, -1, 0)]
    while work:
        a, b, lev, parent, side = work.pop()
        sel = perm[a:b]
        sub = pts[sel]
        blo, bhi = sub.min(axis=0), sub.max(axis=0)
        v = new_node(a, b, lev, blo, bhi)
        if parent >= 0:
            child[parent][side] = v
        if b - a <= n_leaf:
            continue
        axis = int(np.argmax(bhi - blo))
        coord = pts[sel, axis]
        mid = 0.5 * (blo[axis] + bhi[axis])
        low = coord <= mid
        if low.all() or not low.any():
            order = np.argsort(coord, kind="stable")
            low = np.zeros(b - a, dtype=bool)
            low[order[: (b - a) // 2]] = True
        perm[a:b] = np.concatenate([sel[low], sel[~low]])
        cut = a + int(low.sum())
        # right pushed first so the left subtree is numbered first (preorder)
        work.append((cut, b, lev + 1, v, 1))
        work.append((a, cut, lev + 1, v, 0))
    return OracleClusterTree(
        perm=perm.astype(np.int64),
        start=np.array(start, dtype=np.int64),
        stop=np.array(stop, dtype=np.int64),
        lo=np.array(lo), hi=np.array(hi),
        level=np.array(level, dtype=np.int64),
        child=np.array(child, dtype=np.int64),
        points_tree=pts[perm],
    )


def block_leaves(rows, cols, eta):
    """Leaves of the eta-admissible block tree in ``BlockTree.leaves()`` order.

    Returns an (nb, 3) int64 array of (kind, row_node, col_node) with kind
    DENSE=0 / ADMISSIBLE=1 (``geometry.py:261-268, 277-295``).
    """
    if eta <= 0:
        raise ValueError("eta must be positive")
    out = []
    stack = [(0, 0)]
    while stack:
        r, c = stack.pop()
        if is_admissible(rows.lo[r], rows.hi[r], cols.lo[c], cols.hi[c], eta):
            out.append((ADMISSIBLE, r, c))
            continue
        rl, cl = rows.is_leaf(r), cols.is_leaf(c)
        if rl and cl:
            out.append((DENSE, r, c))
            continue
        rk = (r,) if rl else tuple(rows.child[r])
        ck = (c,) if cl else tuple(cols.child[c])
        stack.extend((a, b) for a in rk for b in ck)
    return np.array(out, dtype=np.int64).reshape(-1, 3)


def leaf_table(rows, cols, leaves):
    """(nb, 5) int64 table (kind, r0, r1, c0, c1) -- the C-ABI block-list layout."""
    k, r, c = leaves[:, 0], leaves[:, 1], leaves[:, 2]
    return np.stack([k, rows.start[r], rows.stop[r], cols.start[c], cols.stop[c]], axis=1)
