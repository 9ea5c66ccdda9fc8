"""Oracle H-LU / formatted arithmetic (CPU) against SPEC.md's own examples
(SPEC.md:401-429, 487-505).  The reference module is absent (parity unpinned);
these pin the oracle to SPEC's exact / derived properties before it is used as
the checker of the device H-LU (tests/test_gpu_hlu.py)."""

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

import paper_1706_09384_b200 as hmx
from oracle import hlu as OL
from oracle import hmatrix as OH
from oracle import solve as OS
from tests._problems import Problem, oracle_params


@pytest.fixture(autouse=True)
def _one_blas_thread():
    with threadpool_limits(1):
        yield


class Plate:
    """Diagonally shifted plate ElastoU system (self-block rule zeta = N_c)."""

    def __init__(self, n_side=12, n_leaf=16, eta=3.0, eps=1e-6, ks=4.0, kind="U", self_shift=None):
        w = Problem("U8k", 8).w
        from dataclasses import replace

        self.w = replace(w, ks=ks, n_leaf=n_leaf, eta=eta, eps=eps, kind=kind,
                         kappa=ks if kind == "H" else 0.0)
        self.d = self.w.d
        self.cloud = hmx.make_geometry("plate", n_side, 1.0, d=self.d)
        self.N = self.cloud.points.shape[0]
        self.ct = hmx.build_cluster_tree(self.cloud, n_leaf)
        self.bt = hmx.build_block_tree(self.ct, self.ct, eta)
        self.params = oracle_params(self.w.spec())
        self.zeta = float(self.N) if self_shift is None else self_shift
        self.oh = OH.assemble(self.w.kind, self.params, self.ct.points_tree, None, self.ct.permutation,
                              self.bt.leaf_table, eps, self_shift=self.zeta)

    def tree(self):
        return OL.from_payload(self.bt, self.d, self.oh.payload)

    def dense(self):
        return OH.dense_matrix(self.w.kind, self.params, self.ct.points_tree, None, self.zeta)


@pytest.fixture(scope="module")
def plate():
    return Plate()


def _rand(n, seed, k=1):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k)))


def test_addmul_all_dense_exact():
    # all-Dense small case -> equals dense A + A'A'' exactly (one dense leaf)
    cl = hmx.make_geometry("sphere", 40, 1.0)
    ct = hmx.build_cluster_tree(cl, 64)
    bt = hmx.build_block_tree(ct, ct, 3.0)
    assert len(bt.table) == 1 and bt.table[0, 0] == 0
    A, B, C = (_rand(40, s, 40) for s in (1, 2, 3))
    t = OL.from_dense(bt, 1, C, 0.0)
    OL.formatted_addmul(t, OL.from_dense(bt, 1, A, 0.0), OL.from_dense(bt, 1, B, 0.0), 1e-4)
    assert np.array_equal(t.a, C + A @ B)


def test_addmul_lowrank_rank_bound():
    # LowRank(r1) + LowRank(r2) LowRank(r3) -> rank <= r1 + min(r2, r3) before recompression
    rng = np.random.default_rng(0)

    def lr(m, n, r):
        x = OL.Node(OL.LOWRANK, 0, m, 0, n)
        x.u = rng.standard_normal((m, r)) + 1j * rng.standard_normal((m, r))
        x.v = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
        return x

    for r1, r2, r3 in [(3, 5, 2), (4, 2, 6), (0, 3, 3)]:
        C, A, B = lr(30, 20, r1), lr(30, 25, r2), lr(25, 20, r3)
        ref = C.u @ C.v.conj().T + (A.u @ A.v.conj().T) @ (B.u @ B.v.conj().T)
        cx = OL.Ctx(0.0)
        OL.addmul(cx, C, A, B, 1.0)
        k = C.u.shape[1] + sum(p[0].shape[1] for p in C.pend)
        assert k <= r1 + min(r2, r3)
        OL.flush_all(cx, C)
        assert C.u.shape[1] <= r1 + min(r2, r3)
        assert np.linalg.norm(C.u @ C.v.conj().T - ref) <= 1e-12 * np.linalg.norm(ref)


def test_addmul_random_h_operands():
    # random H-formatted operands at N ~ 1000, eps_LU = 1e-6 ->
    # ||result - dense||_F <= 10 eps (||A||_F + ||A'||_F ||A''||_F)
    pb = Problem("H4k", 1000)
    pts = pb.ct.points_tree
    from oracle import kernels as OK

    mats = [OK.scalar_block(k, pts, pts, self_shift=s) for k, s in ((3.0, 50.0), (7.0, 10.0), (11.3, 1.0))]
    eps = 1e-6
    A, A1, A2 = (OL.from_dense(pb.bt, 1, M, eps) for M in mats)
    cx = OL.Ctx(0.0)
    Ad, A1d, A2d = (OL.dense(cx, t) for t in (A, A1, A2))
    OL.formatted_addmul(A, A1, A2, eps)
    err = np.linalg.norm(OL.dense(cx, A) - (Ad + A1d @ A2d))
    bound = 10 * eps * (np.linalg.norm(Ad) + np.linalg.norm(A1d) * np.linalg.norm(A2d))
    assert err <= bound, (err, bound)


def test_hlu_consistency_and_eps_scaling(plate):
    # ||L U x - A_H x|| / ||A_H x|| <= 10 eps_LU; 1e-4 vs 1e-6 -> ~two orders
    xt = _rand(plate.d * plate.N, 5)[:, 0]
    yh = OH.matvec_tree(plate.oh, xt)
    errs = {}
    for eps in (1e-4, 1e-6):
        root = plate.tree()
        OL.hlu(root, eps)
        errs[eps] = np.linalg.norm(OL.lu_apply_tree(root, xt) - yh) / np.linalg.norm(yh)
        assert errs[eps] <= 10 * eps
    assert errs[1e-6] < errs[1e-4] / 10


def test_hlu_weak_shift(plate):
    # same consistency with a shift far below zeta = N_c (the off-diagonal blocks matter)
    p = Plate(self_shift=2.0)
    xt = _rand(p.d * p.N, 6)[:, 0]
    yh = OH.matvec_tree(p.oh, xt)
    root = p.tree()
    OL.hlu(root, 1e-6)
    assert np.linalg.norm(OL.lu_apply_tree(root, xt) - yh) <= 1e-5 * np.linalg.norm(yh)


def test_hlu_single_leaf_is_dense_lu():
    # 1-leaf dense matrix -> dense LU, machine-precision residual
    cl = hmx.make_geometry("sphere", 50, 1.0)
    ct = hmx.build_cluster_tree(cl, 64)
    bt = hmx.build_block_tree(ct, ct, 3.0)
    A = _rand(50, 7, 50) + 50 * np.eye(50)
    root = OL.from_dense(bt, 1, A, 0.0)
    OL.hlu(root, 1e-4)
    b = _rand(50, 8)[:, 0]
    x = OL.solve_tree(root, b)
    assert np.linalg.norm(A @ x - b) <= 1e-13 * np.linalg.norm(b)


def test_triangular_solve_recovers_y(plate):
    # b = L_H U_H y -> y to 1e-10; SPEC.md:443 consistency 1e-10
    root = plate.tree()
    OL.hlu(root, 1e-4)
    y = _rand(plate.d * plate.N, 9)[:, 0]
    b = OL.lu_apply_tree(root, y)
    assert np.linalg.norm(OL.solve_tree(root, b) - y) <= 1e-10 * np.linalg.norm(y)


def test_identity_solve():
    # identity H-matrix -> x0 = b
    pb = Problem("H4k", 300)
    root = OL.from_dense(pb.bt, 1, np.eye(300, dtype=complex), 1e-8)
    OL.hlu(root, 1e-4)
    b = _rand(300, 10)[:, 0]
    assert np.allclose(OL.solve_tree(root, b), b, rtol=0, atol=1e-13)


def test_singular_leaf_raises():
    pb = Problem("H4k", 300)
    A = np.eye(300, dtype=complex)
    A[5, 5] = 0.0
    root = OL.from_dense(pb.bt, 1, A, 1e-8)
    with pytest.raises(ArithmeticError, match="block path"):
        OL.hlu(root, 1e-4)


def test_direct_vs_gmres(plate):
    # GMRES solution agrees with solve_direct to max(tol, 10 eps_LU)
    root = plate.tree()
    eps = 1e-6
    OL.hlu(root, eps)
    b = _rand(plate.d * plate.N, 11)[:, 0]
    x_d = OL.solve_tree(root, b)
    tol = 1e-8
    x_g, it, _, conv = OS.gmres(lambda v: OH.matvec_tree(plate.oh, v), b, tol, 50, 500)
    assert conv
    assert np.linalg.norm(x_g - x_d) <= max(tol, 10 * eps) * np.linalg.norm(x_d)
