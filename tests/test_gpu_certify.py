"""Opt-in per-leaf certification (ACAConfig(certify=True)): after assembly every admissible leaf is
regenerated on the device and the leaves with ||A_b - U V^H||_F > eps ||A_b||_F are re-compressed at
tighter tolerances and spliced back (hmx_hmatrix_splice), so that every leaf meets the north_star
bar eps (the reference's SPEC.md:329 promises 3 eps; the default assembly keeps that behaviour)."""

import numpy as np
import pytest

import paper_1706_09384_b200 as hmx
from paper_1706_09384_b200.hmatrix import block_errors, splice
from tests._problems import Problem

pytestmark = pytest.mark.gpu


def _rel(H, pb):
    err2, norm2 = block_errors(H, pb.spec, pb.cloud)
    adm = pb.table[:, 0] == 1
    return np.sqrt(err2[adm] / norm2[adm])


@pytest.mark.parametrize("tag", ["U32k", "T65k", "U131k"])
def test_certified_assembly_every_leaf_within_eps(tag):
    pb = Problem(tag)
    H0, _ = pb.device_h()
    r0 = _rel(H0, pb)
    H, rep = pb.device_h(certify=True)
    r = _rel(H, pb)
    cr = H.certify_report
    print(f"{tag}: {int((r0 > pb.w.eps).sum())} leaves above eps by default (worst {r0.max() / pb.w.eps:.2f} eps), "
          f"certified: worst {r.max() / pb.w.eps:.3f} eps, rounds {cr['rounds']}")
    assert cr["leaves_above_eps"] == int((r0 > pb.w.eps).sum())
    assert r.max() <= pb.w.eps and cr["leaves_still_above_eps"] == 0
    # untouched leaves keep their factors; the H-matvec of the certified H is no worse
    info0, info = H0.block_info(), H.block_info()
    kept = (info["flags"] & 256) == 0
    np.testing.assert_array_equal(info["rank_after"][kept], info0["rank_after"][kept])
    x = pb.rhs(0)
    y0, y = hmx.matvec(H0, x), hmx.matvec(H, x)
    assert np.linalg.norm(y - y0) <= 3 * pb.w.eps * np.linalg.norm(y0)


def test_splice_identity_and_replacement():
    pb = Problem("U8k", 2048)
    H, _ = pb.device_h()
    adm = np.flatnonzero(pb.table[:, 0] == 1)
    idx = adm[::7]
    from paper_1706_09384_b200.shard import LeafSubset

    Hs, _ = hmx.assemble(pb.spec, pb.cloud, pb.ct, LeafSubset(pb.bt, idx), hmx.ACAConfig(eps_aca=pb.w.eps))
    x = pb.rhs(3)
    # the same factors spliced in: bitwise the same matvec
    Hx = splice(H, Hs, idx)
    np.testing.assert_array_equal(hmx.matvec(Hx, x), hmx.matvec(H, x))
    # tighter factors spliced in: those leaves change, the others do not
    Ht, _ = hmx.assemble(pb.spec, pb.cloud, pb.ct, LeafSubset(pb.bt, idx), hmx.ACAConfig(eps_aca=1e-7))
    Hy = splice(H, Ht, idx)
    for b in (idx[0], adm[1]):
        f = Hy.block(int(b))
        g = (Ht.block(0) if b == idx[0] else H.block(int(b)))
        np.testing.assert_array_equal(f.dense(), g.dense())
    with pytest.raises(ValueError):
        splice(H, Hs, idx[:-1])  # length mismatch
    with pytest.raises(ValueError):
        splice(H, Hs, idx[::-1])  # leaves do not match
