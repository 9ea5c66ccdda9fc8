"""Pin the oracle to the reference: bit-exact against the live reference
modules (build container only) and against the committed golden fixtures
generated from the reference (tests/golden/make_golden.py)."""

import glob
import os

import numpy as np
import pytest

from oracle import geometry as OG
from oracle import kernels as OK

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _oracle_geometry(kind, n, leaf, eta):
    pts, _ = OG.sphere_cloud(n) if kind == "sphere" else OG.plate_cloud(n)
    ct = OG.cluster_tree(pts, leaf)
    lv = OG.block_leaves(ct, ct, eta)
    return ct, OG.leaf_table(ct, ct, lv)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "geometry_*.npz"))))
def test_oracle_geometry_matches_golden(path):
    g = np.load(path)
    ct, tab = _oracle_geometry(str(g["kind"]), int(g["n"]), int(g["n_leaf"]), float(g["eta"]))
    np.testing.assert_array_equal(ct.perm, g["perm"])
    np.testing.assert_array_equal(tab, g["table"])


def test_oracle_kernels_match_golden():
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    X, Y, NY = g["X"], g["Y"], g["NY"]
    cases = {
        "H": OK.scalar_block(11.3, X, Y, self_shift=4096.0),
        "H_lap": OK.scalar_block(0.0, X, Y, self_shift=4096.0),
        "U": OK.elasto_u_block(9.262, 16.042, 1 / 16.042**2, X, Y, self_shift=8192.0),
        "U_low": OK.elasto_u_block(2.0 / np.sqrt(3.0), 2.0, 0.25, X * 0.01, Y * 0.01, self_shift=1.0),
        "T": OK.elasto_t_block(26.197, 45.375, 1.0, 1.0, 1 / 45.375**2, X, Y, NY, self_shift=65536.0),
    }
    for k, v in cases.items():
        # bit-exact on the generating host; libm may differ by an ulp elsewhere
        np.testing.assert_allclose(v, g[k], rtol=1e-14, atol=0, err_msg=k)
    assert OK.scalar_block(11.3, X, Y) is None and bool(g["H_none_is_none"])


def test_oracle_bit_exact_vs_live_reference(reference_modules):
    G, R, _ = reference_modules
    rng = np.random.default_rng(5)
    X = rng.standard_normal((30, 3))
    Y = rng.standard_normal((33, 3))
    Y[2] = X[9]
    NY = rng.standard_normal((33, 3))
    NY /= np.linalg.norm(NY, axis=1)[:, None]
    pairs = [
        (R.scalar_block(7.0, X, Y, self_shift=5.0), OK.scalar_block(7.0, X, Y, self_shift=5.0)),
        (R.elasto_u_block(3.0, 5.0, 0.04, X, Y, self_shift=5.0), OK.elasto_u_block(3.0, 5.0, 0.04, X, Y, self_shift=5.0)),
        (R.elasto_t_block(3.0, 5.0, 1.3, 0.7, 0.04, X, Y, NY, self_shift=5.0),
         OK.elasto_t_block(3.0, 5.0, 1.3, 0.7, 0.04, X, Y, NY, self_shift=5.0)),
    ]
    for a, b in pairs:
        np.testing.assert_array_equal(a, b)
    for kind, n, leaf, eta in [("sphere", 2048, 32, 3.0), ("plate", 25, 4, 3.0), ("sphere", 700, 10, 0.5)]:
        cl = G.make_geometry(kind, n, 1.0)
        ct = G.build_cluster_tree(cl, leaf)
        bt = G.build_block_tree(ct, ct, eta)
        ref = np.array([(1 if isinstance(l, G.AdmissibleLeaf) else 0, l.row.start, l.row.stop, l.col.start,
                         l.col.stop) for l in bt.leaves()])
        oct_, tab = _oracle_geometry(kind, n, leaf, eta)
        np.testing.assert_array_equal(oct_.perm, ct.permutation)
        np.testing.assert_array_equal(tab, ref)


def test_spec_geometry_kats():
    # SPEC.md:70-72, 80-82, 90-92
    lo, hi = np.zeros(3), np.ones(3)
    assert OG.diam_box(lo, hi) == pytest.approx(np.sqrt(3))
    assert OG.diam_box(np.zeros(3), np.array([3.0, 4.0, 0.0])) == 5.0
    assert OG.diam_box(lo, lo) == 0.0
    assert OG.dist_box(lo, hi, lo + 3, hi + 3) == pytest.approx(2 * np.sqrt(3))
    assert OG.dist_box(lo, hi, lo, hi) == 0.0
    assert OG.dist_box(lo, hi, np.array([2.0, 0, 0]), np.array([3.0, 1, 1])) == 1.0
    assert OG.is_admissible(lo, hi, lo + 3, hi + 3, 3.0)
    assert not OG.is_admissible(lo, hi, lo, hi, 3.0)
    p = np.zeros(3)
    assert OG.is_admissible(p, p, p + np.array([1.0, 0, 0]), p + np.array([1.0, 0, 0]), 3.0)
    # 4 collinear points, n_leaf = 1 -> coordinate-order singletons
    pts = np.array([[3.0, 0, 0], [0.0, 0, 0], [2.0, 0, 0], [1.0, 0, 0]])
    ct = OG.cluster_tree(pts, 1)
    np.testing.assert_array_equal(ct.perm, [1, 3, 2, 0])
    # 50 points, n_leaf 100 -> single node
    assert len(OG.cluster_tree(np.random.default_rng(0).standard_normal((50, 3)), 100).start) == 1
