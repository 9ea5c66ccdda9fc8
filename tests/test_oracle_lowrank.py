"""SPEC known-answer tests for the oracle low-rank / H-matrix / GMRES
restatement.  CPU only."""

import numpy as np
import pytest

from oracle import hmatrix as OH
from oracle import kernels as OK
from oracle import lowrank as OL
from oracle import solve as OS
from tests._problems import Problem


class DenseGen:
    """BlockGenerator over an explicit matrix (d x d point blocks)."""

    def __init__(self, A, d):
        self.A, self.d = A, d
        self.m, self.n = A.shape[0] // d, A.shape[1] // d

    def row(self, i):
        return self.A[self.d * i : self.d * i + self.d, :]

    def col(self, j):
        return self.A[:, self.d * j : self.d * j + self.d]


def test_aca_rank_one_and_zero():
    rng = np.random.default_rng(0)
    u = rng.standard_normal(20) + 1j * rng.standard_normal(20)
    v = rng.standard_normal(15) + 1j * rng.standard_normal(15)
    r = OL.aca(DenseGen(np.outer(u, v), 1), 1e-6)
    assert r.steps == 1 and r.converged
    assert np.abs(r.U @ r.V.conj().T - np.outer(u, v)).max() < 1e-12
    z = OL.aca(DenseGen(np.zeros((9, 12), complex), 3), 1e-4)
    assert z.steps == 0 and z.converged and z.U.shape[1] == 0


def test_vector_aca_single_3x3_exact():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((3, 3)) + 1j * rng.standard_normal((3, 3))
    r = OL.aca(DenseGen(A, 3), 1e-4)
    assert r.steps == 1 and r.converged
    np.testing.assert_allclose(r.U @ r.V.conj().T, A, atol=1e-13)


def test_recompress_rank_and_idempotence():
    rng = np.random.default_rng(2)
    U = rng.standard_normal((40, 3)) + 1j * rng.standard_normal((40, 3))
    V = rng.standard_normal((30, 3)) + 1j * rng.standard_normal((30, 3))
    U2 = np.concatenate([U, U[:, :1]], axis=1)
    V2 = np.concatenate([V, V[:, :1]], axis=1)
    a, b = OL.recompress(U2, V2, 1e-10)
    assert a.shape[1] == 3  # duplicated column: rank strictly drops
    a2, b2 = OL.recompress(a, b, 1e-10)
    assert a2.shape[1] == a.shape[1]
    np.testing.assert_allclose(a2 @ b2.conj().T, a @ b.conj().T, atol=1e-12)


@pytest.mark.parametrize("tag,n", [("H4k", 1024), ("U8k", 512), ("T65k", 512)])
def test_aca_recompress_within_3eps_dense(tag, n):
    # SPEC.md:329 on dense-checkable blocks
    pb = Problem(tag, n)
    rng = np.random.default_rng(3)
    adm = np.flatnonzero(pb.table[:, 0] == 1)
    for b in rng.choice(adm, 12, replace=False):
        k, r0, r1, c0, c1 = pb.table[b]
        NY = None if pb.nrm is None else pb.nrm[c0:c1]
        gen = OL.BlockGen(pb.kind, pb.params, pb.pts[r0:r1], pb.pts[c0:c1], NY, float(pb.N))
        res = OL.aca(gen, pb.w.eps)
        U, V = OL.recompress(res.U, res.V, pb.w.eps)
        A = gen.dense()
        assert U.shape[1] <= res.U.shape[1]
        assert np.linalg.norm(A - U @ V.conj().T) <= 3 * pb.w.eps * np.linalg.norm(A)
        assert U.shape[1] >= OL.numerical_rank(A, pb.w.eps) - 1


def test_vector_aca_interpolation_zeros():
    # residual vanishes on selected pivot rows / columns
    pb = Problem("U8k", 512)
    b = int(np.flatnonzero(pb.table[:, 0] == 1)[5])
    k, r0, r1, c0, c1 = pb.table[b]
    gen = OL.BlockGen("U", pb.params, pb.pts[r0:r1], pb.pts[c0:c1], None, float(pb.N))
    res = OL.aca(gen, 1e-4)
    R = gen.dense() - res.U @ res.V.conj().T
    scale = np.abs(gen.dense()).max()
    for i, j in res.pivots:
        assert np.abs(R[3 * i : 3 * i + 3, :]).max() <= 1e-12 * scale
        assert np.abs(R[:, 3 * j : 3 * j + 3]).max() <= 1e-12 * scale


def test_reducibility_scalar_fails_vector_succeeds():
    # SPEC.md:601 / PAPER.md (FSplane): coplanar plate U block
    from oracle import geometry as OG

    pts, _ = OG.plate_cloud(24)
    ct = OG.cluster_tree(pts, 16)
    lv = OG.block_leaves(ct, ct, 3.0)
    tab = OG.leaf_table(ct, ct, lv)
    b = [i for i, t in enumerate(tab) if t[0] == 1 and (t[2] - t[1]) >= 32][0]
    k, r0, r1, c0, c1 = tab[b]
    X, Y = ct.points_tree[r0:r1], ct.points_tree[c0:c1]
    kp, ks = 5 * np.pi / 2, 5 * np.pi
    A = OK.elasto_u_block(kp, ks, 1 / ks**2, X, Y)
    vec = OL.aca(DenseGen(A, 3), 1e-4)
    assert np.linalg.norm(A - vec.U @ vec.V.conj().T) <= 3e-4 * np.linalg.norm(A)
    sca = OL.aca(DenseGen(A, 1), 1e-4)
    assert np.linalg.norm(A - sca.U @ sca.V.conj().T) > 1e-3 * np.linalg.norm(A)


def test_aca_full_and_numerical_rank():
    rng = np.random.default_rng(4)
    A = (rng.standard_normal((30, 2)) + 0j) @ (rng.standard_normal((2, 25)) + 0j)
    U, V, conv = OL.aca_full(A, 1e-10)
    assert conv and U.shape[1] == 2
    assert OL.numerical_rank(np.eye(5), 1e-4) == 5
    assert OL.numerical_rank(A, 1e-4) == 2


def test_randomized_svd():
    rng = np.random.default_rng(6)
    A = (rng.standard_normal((60, 5)) + 1j * rng.standard_normal((60, 5))) @ (
        rng.standard_normal((5, 40)) + 1j * rng.standard_normal((5, 40)))
    U, V, conv = OL.randomized_svd(A, 1e-8)
    assert conv and np.linalg.norm(A - U @ V.conj().T) <= 1e-8 * np.linalg.norm(A)
    Ur, Vr = OL.recompress(U, V, 1e-8)
    assert Ur.shape[1] == 5
    U0, V0, c0 = OL.randomized_svd(np.zeros((10, 8), complex), 1e-4)
    assert U0.shape[1] == 0 and c0


def test_oracle_matvec_and_gmres_small():
    pb = Problem("U8k", 256)
    oh = pb.oracle_h(workers=1)
    A = OH.dense_matrix(pb.kind, pb.params, pb.pts, pb.nrm, float(pb.N))
    x = pb.rhs(1)
    y = OH.matvec(oh, x)
    yd = OH.from_tree(oh, A @ OH.to_tree(oh, x))
    assert np.linalg.norm(y - yd) <= 3 * pb.w.eps * np.linalg.norm(yd)
    assert not np.any(OH.matvec(oh, np.zeros_like(x)))
    xs, it, hist, conv = OS.gmres(lambda v: OH.matvec(oh, v), x, 1e-8, 50, 500)
    assert conv and np.linalg.norm(OH.matvec(oh, xs) - x) <= 1.0001e-8 * np.linalg.norm(x)
    assert all(b <= a * (1 + 1e-12) for a, b in zip(hist, hist[1:]))
    x0, it0, h0, c0 = OS.gmres(lambda v: OH.matvec(oh, v), np.zeros_like(x), 1e-4)
    assert it0 == 0 and c0 and not np.any(x0)
    # restarted path + scipy cross-check of the iteration count (small shift -> many iterations)
    import scipy.sparse.linalg as sla

    rng = np.random.default_rng(0)
    M = np.eye(120) * 3 + (rng.standard_normal((120, 120)) + 1j * rng.standard_normal((120, 120))) / 11
    bb = rng.standard_normal(120) + 0j
    xs2, it2, hist2, conv2 = OS.gmres(lambda v: M @ v, bb, 1e-10, 7, 500)
    assert conv2 and np.linalg.norm(M @ xs2 - bb) <= 1e-9 * np.linalg.norm(bb)
    cnt = []
    sla.gmres(M, bb, rtol=1e-10, atol=0, restart=7, maxiter=500, callback=lambda r: cnt.append(r),
              callback_type="pr_norm")
    assert abs(len(cnt) - it2) <= 2
