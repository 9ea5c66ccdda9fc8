"""SPEC.md:444-445 rank-trend invariants on the device-assembled sphere (elasto U, eta = 3,
leaf 32, eps 1e-4):

* fixed-omega rank stability: max_rank_after varies by <= 15% across >= 3 refinements of the
  sphere at a fixed frequency (PAPER Table 2 pattern);
* fixed-density rank growth: at 10 points per S-wavelength, max_rank_after grows by a factor in
  [1.5, 2.5] each time omega doubles (N quadruples).
"""

import pytest

import paper_1706_09384_b200 as hmx
from paper_1706_09384_b200.configs import WORKLOADS, ks_ten_per_wavelength

pytestmark = pytest.mark.gpu


def _max_rank(n_points, ks):
    w = WORKLOADS["U8k"]
    cl = hmx.make_geometry("sphere", n_points, 1.0, d=3)
    ct = hmx.build_cluster_tree(cl, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    mat = hmx.Material.from_lame(1.0, 1.0, 1.0, ks)
    H, rep = hmx.assemble(hmx.KernelSpec.elasto_u(mat), cl, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    return rep.max_rank_after


def test_fixed_frequency_rank_stability():
    ranks = [_max_rank(n, 3.0) for n in (4096, 8192, 16384, 32768)]
    print("omega = 3, N = 4k..32k: max ranks", ranks)
    assert max(ranks) <= 1.15 * min(ranks), ranks


def test_fixed_density_rank_growth():
    ns = (2048, 8192, 32768)
    ranks = [_max_rank(n, ks_ten_per_wavelength(n)) for n in ns]
    print("10 points per S-wavelength, N =", ns, "max ranks", ranks)
    for a, b in zip(ranks, ranks[1:]):
        assert 1.5 <= b / a <= 2.5, ranks
