"""Device H-LU / formatted arithmetic / triangular solves
against the oracle (oracle/hlu.py, pinned by tests/test_oracle_hlu.py) on the
same inputs: oracle-assembled factors loaded into the device H, and device
assemblies of the sphere U / T / Helmholtz configurations at reduced size."""

import numpy as np
import pytest
import torch
from threadpoolctl import threadpool_limits

import paper_1706_09384_b200 as hmx
from paper_1706_09384_b200 import hierarchical_lu as HL
from oracle import hlu as OL
from oracle import hmatrix as OH
from oracle import kernels as OK
from tests._problems import Problem
from tests.test_oracle_hlu import Plate

pytestmark = pytest.mark.gpu


def _rand(n, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def _device_h(p):
    h = hmx.HMatrix.from_factors(p.d, p.N, p.ct.permutation, p.bt.leaf_table, p.oh.payload)
    h.block_tree = p.bt
    return h


@pytest.mark.parametrize("shift,eps", [(None, 1e-4), (2.0, 1e-6)])
def test_hlu_matches_oracle_same_factors(shift, eps):
    """Same input H (oracle factors) -> device and oracle factorisations: identical
    truncated ranks per factor block, solutions agree to 1e-10 (the bitwise-level
    differences are cuSOLVER vs LAPACK rounding), both consistent to 10 eps_LU."""
    with threadpool_limits(1):
        p = Plate(self_shift=shift, eps=1e-6)
        o = p.tree()
        OL.hlu(o, eps)
    h = _device_h(p)
    f = HL.hlu(h, eps)
    rd = [x.rank for x in HL._walk(f.root) if isinstance(x, HL.LowRank)]
    ro = [x.u.shape[1] for x in OL.leaves(o) if x.kind == OL.LOWRANK]
    assert np.abs(np.array(rd) - np.array(ro)).max() <= 1
    b = _rand(p.d * p.N, 3)
    x = HL.triangular_solve(f, b)
    idx = OL.tree_index(p.ct.permutation, p.d)
    xo = np.empty_like(b)
    xo[idx] = OL.solve_tree(o, b[idx])
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
    y = hmx.matvec(h, b)
    assert np.linalg.norm(HL.lu_matvec(f, b) - y) <= 10 * eps * np.linalg.norm(y)


@pytest.mark.parametrize("tag,n", [("U8k", 1024), ("T65k", 768), ("H4k", 2048)])
def test_hlu_device_assembled(tag, n):
    """Device assembly -> device H-LU: 10 eps_LU consistency, b = L U y
    recovers y to 1e-10, solve_direct agrees with solve_gmres to
    max(tol, 10 eps_LU), eps 1e-4 -> 1e-6 drops the residual ~2 orders."""
    pb = Problem(tag, n)
    H, _ = pb.device_h()
    b = pb.rhs(4)
    y = hmx.matvec(H, b)
    res = {}
    for eps in (1e-4, 1e-6):
        f = HL.hlu(H, eps)
        res[eps] = np.linalg.norm(HL.lu_matvec(f, b) - y) / np.linalg.norm(y)
        assert res[eps] <= 10 * eps, (eps, res[eps])
    assert res[1e-6] < res[1e-4] / 10
    yy = HL.lu_matvec(f, b)
    assert np.linalg.norm(HL.triangular_solve(f, yy) - b) <= 1e-10 * np.linalg.norm(b)
    x_d, f2 = hmx.solve_direct(H, b, 1e-6)
    tol = 1e-8
    g = hmx.solve_gmres(H, b, hmx.GmresConfig(tol=tol, restart=50, max_iters=500))
    assert g.converged
    assert np.linalg.norm(g.x - x_d) <= max(tol, 1e-5) * np.linalg.norm(x_d)
    # factor reuse: a second right-hand side through the same factors
    b2 = pb.rhs(5)
    x2 = hmx.triangular_solve(f2, b2)
    assert np.linalg.norm(hmx.matvec(H, x2) - b2) <= 1e-4 * np.linalg.norm(b2)


def test_device_tensor_io():
    pb = Problem("U8k", 512)
    H, _ = pb.device_h()
    f = HL.hlu(H, 1e-6)
    b = pb.rhs(6)
    xb = HL.triangular_solve(f, b)
    xt = HL.triangular_solve(f, torch.as_tensor(b, device="cuda"))
    assert xt.is_cuda and np.array_equal(xt.cpu().numpy(), xb)


def test_formatted_addmul_vs_oracle():
    """SPEC.md:408 on the device: random H operands (N = 1000, eps 1e-6), error vs the
    dense product <= 10 eps (||A|| + ||A'|| ||A''||); the oracle on the same operands agrees."""
    pb = Problem("H4k", 1000)
    pts = pb.ct.points_tree
    mats = [OK.scalar_block(k, pts, pts, self_shift=s) for k, s in ((3.0, 50.0), (7.0, 10.0), (11.3, 1.0))]
    eps = 1e-6
    A, A1, A2 = (HL.from_dense(pb.bt, 1, M, eps) for M in mats)
    Ad, A1d, A2d = (HL.to_dense(t).cpu().numpy() for t in (A, A1, A2))
    HL.formatted_addmul(A, A1, A2, eps)
    R = HL.to_dense(A).cpu().numpy()
    err = np.linalg.norm(R - (Ad + A1d @ A2d))
    assert err <= 10 * eps * (np.linalg.norm(Ad) + np.linalg.norm(A1d) * np.linalg.norm(A2d))
    with threadpool_limits(1):
        o = [OL.from_dense(pb.bt, 1, M, eps) for M in mats]
        OL.formatted_addmul(o[0], o[1], o[2], eps)
        Ro = OL.dense(OL.Ctx(0.0), o[0])
    assert np.linalg.norm(R - Ro) <= 10 * eps * np.linalg.norm(Ro)


def test_addmul_all_dense_exact():
    cl = hmx.make_geometry("sphere", 40, 1.0)
    ct = hmx.build_cluster_tree(cl, 64)
    bt = hmx.build_block_tree(ct, ct, 3.0)
    rng = np.random.default_rng(1)
    A, B, C = (rng.standard_normal((40, 40)) + 1j * rng.standard_normal((40, 40)) for _ in range(3))
    t = HL.from_dense(bt, 1, C, 0.0)
    HL.formatted_addmul(t, HL.from_dense(bt, 1, A, 0.0), HL.from_dense(bt, 1, B, 0.0), 1e-4)
    ref = C + A @ B
    assert isinstance(t.nodes(), HL.Dense)
    assert np.linalg.norm(HL.to_dense(t).cpu().numpy() - ref) <= 1e-14 * np.linalg.norm(ref)


def test_identity_and_singular():
    pb = Problem("H4k", 300)
    I = np.eye(300, dtype=complex)
    root = HL.from_dense(pb.bt, 1, I, 1e-8)
    root.factor(1e-4)
    b = torch.as_tensor(_rand(300, 7), device="cuda")[:, None]
    x = root.apply(b, 0)
    assert torch.allclose(x, b, rtol=0, atol=1e-13)
    assert torch.allclose(root.apply(b, 1), b, rtol=0, atol=1e-13)
    I[5, 5] = 0.0
    root = HL.from_dense(pb.bt, 1, I, 1e-8)
    with pytest.raises(hmx.FactorizationError, match="block path"):
        root.factor(1e-4)


def test_source_h_unchanged():
    """The H-LU works on a copy: the assembled H (immutable) still gives the same matvec."""
    pb = Problem("U8k", 512)
    H, _ = pb.device_h()
    b = pb.rhs(8)
    y0 = hmx.matvec(H, b)
    HL.hlu(H, 1e-4)
    assert np.array_equal(hmx.matvec(H, b), y0)


def test_source_h_unchanged_one_point_leaves():
    """d = 1 with one-point leaves: 1 x n / m x 1 leaf views of the HBM streams are already contiguous,
    and the H-LU must still copy them (in-place Schur updates would otherwise write into H)."""
    cl = hmx.make_geometry("sphere", 96, 1.0, d=1)
    ct = hmx.build_cluster_tree(cl, 1)
    bt = hmx.build_block_tree(ct, ct, 3.0)
    H, _ = hmx.assemble(hmx.KernelSpec.helmholtz(2.0), cl, ct, bt, hmx.ACAConfig(eps_aca=1e-6))
    b = _rand(96, 21)
    y0 = hmx.matvec(H, b)
    f = HL.hlu(H, 1e-6)
    assert np.array_equal(hmx.matvec(H, b), y0)
    x = hmx.triangular_solve(f, b)
    assert np.linalg.norm(hmx.matvec(H, x) - b) <= 1e-4 * np.linalg.norm(b)


def test_single_leaf_is_dense_lu():
    """a 1-leaf H-matrix reduces to the pivoted dense LU (machine-precision residual)."""
    from dataclasses import replace

    pb = Problem("U8k", 40)
    w = replace(pb.w, n_leaf=64)
    cl = hmx.make_geometry("sphere", 40, 1.0, d=3)
    ct = hmx.build_cluster_tree(cl, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    assert len(bt.table) == 1
    H, _ = hmx.assemble(w.spec(), cl, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    b = _rand(120, 12)
    x, f = hmx.solve_direct(H, b, 1e-4)
    assert f.stats["n_getrf"] == 1
    assert np.linalg.norm(hmx.matvec(H, x) - b) <= 1e-13 * np.linalg.norm(b)


def test_lu_snapshot_round_trip(tmp_path):
    """LU factors saved and loaded hold bitwise the same leaves and solve a new
    right-hand side with the in-process residual; a flipped payload byte is a checksum error."""
    pb = Problem("T65k", 600)
    H, _ = pb.device_h()
    f = hmx.hlu(H, 1e-6)
    p = tmp_path / "lu.hmx"
    hmx.snapshot("save", str(p), f)
    g = hmx.snapshot("load", str(p))
    assert isinstance(g, HL.LUFactors)
    for x, y in zip(HL._walk(f.root), HL._walk(g.root)):
        assert type(x) is type(y) and (x.r0, x.r1, x.c0, x.c1) == (y.r0, y.r1, y.c0, y.c1)
        pairs = ([(x.u, y.u), (x.v, y.v)] if isinstance(x, HL.LowRank) else
                 [(x.L, y.L), (x.U, y.U), (x.pidx, y.pidx)] if x.factored else [(x.a, y.a)])
        for p_, q_ in pairs:
            assert torch.equal(p_, q_)
    b = pb.rhs(9)
    x0, x1 = hmx.triangular_solve(f, b), hmx.triangular_solve(g, b)
    assert np.linalg.norm(x1 - x0) <= 1e-13 * np.linalg.norm(x0)
    r0 = np.linalg.norm(hmx.matvec(H, x0) - b)
    r1 = np.linalg.norm(hmx.matvec(H, x1) - b)
    assert abs(r1 - r0) <= 1e-3 * r0
    raw = bytearray(p.read_bytes())
    raw[len(raw) // 2] ^= 0x40
    p.write_bytes(bytes(raw))
    with pytest.raises(hmx.SnapshotCorruptError):
        hmx.snapshot("load", str(p))
