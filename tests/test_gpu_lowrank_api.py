"""One-block low-rank operations of the reference API on the
device: BlockGenerator, aca_partial / aca_vector (same kernel as the batched
assembly), recompress, and the dense utilities numerical_rank / aca_full /
randomized_svd.  Checked against the oracle (oracle/lowrank.py restates the
SPEC algorithm) and the SPEC examples."""

import numpy as np
import pytest

import paper_1706_09384_b200 as hmx
from paper_1706_09384_b200.configs import WORKLOADS

from ._problems import Problem

pytestmark = pytest.mark.gpu


def _admissible_leaf(pb, min_size=0):
    t = pb.table
    adm = np.flatnonzero(t[:, 0] == 1)
    size = (t[adm, 2] - t[adm, 1]) * (t[adm, 4] - t[adm, 3])
    ok = adm[size >= min_size]
    return int(ok[np.argsort(-size[size >= min_size])[len(ok) // 3]])


@pytest.mark.parametrize("tag,n", [("H4k", 2048), ("U8k", 2048), ("T65k", 2048)])
def test_aca_block_matches_oracle(tag, n):
    from oracle import kernels as OK
    from oracle import lowrank as OL

    pb = Problem(tag, n)
    b = _admissible_leaf(pb, 400)
    _, r0, r1, c0, c1 = pb.table[b][:5]
    X, Y = pb.pts[r0:r1], pb.pts[c0:c1]
    NY = None if pb.nrm is None else pb.nrm[c0:c1]
    gen = hmx.BlockGenerator(pb.spec, X, Y, NY)
    cfg = hmx.ACAConfig(eps_aca=pb.w.eps)
    f = hmx.aca_partial(gen, cfg) if pb.d == 1 else hmx.aca_vector(gen, cfg)
    ref = OL.aca(OL.BlockGen(pb.kind, pb.params, X, Y, NY, None), pb.w.eps)
    assert abs(f.steps - ref.steps) <= 1 and abs(f.rank - ref.U.shape[1]) <= pb.d
    A = OK.block(pb.kind, pb.params, X, Y, NY)
    assert np.linalg.norm(A - f.dense()) <= 3 * pb.w.eps * np.linalg.norm(A)
    # strips agree with the entry access and the dense block
    np.testing.assert_allclose(gen.row(2), A[pb.d * 2:pb.d * 3], rtol=0, atol=1e-13 * np.abs(A).max())
    np.testing.assert_allclose(gen.col(1), A[:, pb.d:2 * pb.d], rtol=0, atol=1e-13 * np.abs(A).max())
    np.testing.assert_allclose(gen.block_entry(3, 4), A[3 * pb.d:4 * pb.d, 4 * pb.d:5 * pb.d], rtol=0,
                               atol=1e-13 * np.abs(A).max())
    # recompress: rank never grows, error stays at eps, idempotent rank
    g = hmx.recompress(f, pb.w.eps)
    assert g.rank <= f.rank
    assert np.linalg.norm(A - g.dense()) <= 3 * pb.w.eps * np.linalg.norm(A)
    assert abs(hmx.recompress(g, pb.w.eps).rank - g.rank) <= 1
    ro = OL.recompress(ref.U, ref.V, pb.w.eps)
    assert abs(g.rank - ro[0].shape[1]) <= 1


def test_single_3x3_block_is_exact_in_one_step():
    # a block that is one invertible 3x3 kernel value -> exact after one rank-3 step
    w = WORKLOADS["U8k"]
    gen = hmx.BlockGenerator(w.spec(), [[0.0, 0.0, 0.0]], [[0.3, -0.2, 0.9]])
    f = hmx.aca_vector(gen, hmx.ACAConfig(eps_aca=1e-4))
    A = gen.dense()
    assert f.rank == 3 and f.steps == 1 and f.converged
    assert np.linalg.norm(A - f.dense()) <= 1e-12 * np.linalg.norm(A)


def test_recompress_duplicated_columns_drops_rank():
    # duplicated columns -> rank strictly drops
    rng = np.random.default_rng(0)
    u = rng.standard_normal((60, 4)) + 1j * rng.standard_normal((60, 4))
    v = rng.standard_normal((50, 4)) + 1j * rng.standard_normal((50, 4))
    f = hmx.LowRankFactor(np.hstack([u, u[:, :2]]), np.hstack([v, v[:, :2]]))
    g = hmx.recompress(f, 1e-10)
    assert g.rank == 4
    np.testing.assert_allclose(g.dense(), f.dense(), rtol=0, atol=1e-10 * np.abs(f.dense()).max())


def test_dense_utilities():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(30) + 1j * rng.standard_normal(30)
    y = rng.standard_normal(20) + 1j * rng.standard_normal(20)
    assert hmx.numerical_rank(np.outer(x, y.conj()), 1e-4) == 1
    assert hmx.numerical_rank(np.eye(5), 1e-4) == 5
    a2 = np.outer(x, y) + np.outer(x[::-1], y[::-1] * 1j)
    f = hmx.aca_full(a2, hmx.ACAConfig(eps_aca=1e-10))  # exact rank 2
    assert f.rank == 2 and np.linalg.norm(a2 - f.dense()) <= 1e-10 * np.linalg.norm(a2)
    assert hmx.aca_full(np.zeros((7, 5)), hmx.ACAConfig()).rank == 0
    a5 = (rng.standard_normal((80, 5)) + 1j * rng.standard_normal((80, 5))) @ rng.standard_normal((5, 60))
    r = hmx.randomized_svd(a5, 1e-8)  # rank 5 +- oversampling, trimmed by recompress
    assert r.converged and r.rank >= 5 and np.linalg.norm(a5 - r.dense()) <= 1e-8 * np.linalg.norm(a5)
    assert hmx.recompress(r, 1e-8).rank == 5
    assert hmx.randomized_svd(np.zeros((9, 9)), 1e-8).rank == 0
    # aca_full cannot beat the SVD optimum
    pb = Problem("H4k", 1024)
    b = _admissible_leaf(pb)
    _, r0, r1, c0, c1 = pb.table[b][:5]
    A = hmx.BlockGenerator(pb.spec, pb.pts[r0:r1], pb.pts[c0:c1]).dense()
    assert hmx.aca_full(A, hmx.ACAConfig(eps_aca=1e-4)).rank >= hmx.numerical_rank(A, 1e-4)
