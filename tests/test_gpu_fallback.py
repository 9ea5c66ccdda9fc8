"""The randomized-SVD fallback of the vector ACA on the device.

A coplanar traction block -- plate points, normals (0, 0, 1) -- has n . z_hat = 0 for every pair,
so every 3 x 3 sub-block of T is a combination of n z_hat^T and z_hat n^T: rank 2, sigma_3 = 0
("ElastoT coplanar block where all 3x3 subblocks are singular").  aca_vector signals
FallbackNeeded on it; randomized_svd compresses it; assemble routes every such leaf through the
device fallback instead of failing (pivot exhaustion only if the fallback fails too).
"""

import numpy as np
import pytest

import paper_1706_09384_b200 as hmx
from oracle import hmatrix as OH
from tests._problems import oracle_params

pytestmark = pytest.mark.gpu


def _plate_t(n_side=40, leaf=32):
    cl = hmx.make_geometry("plate", n_side, 1.0, d=3)
    mat = hmx.Material.from_lame(1.0, 1.0, 1.0, 12.0)
    spec = hmx.KernelSpec.elasto_t(mat)
    ct = hmx.build_cluster_tree(cl, leaf)
    bt = hmx.build_block_tree(ct, ct, 3.0)
    return cl, spec, ct, bt


def test_coplanar_t_block_needs_fallback_and_rsvd_compresses_it():
    cl, spec, ct, bt = _plate_t()
    t = bt.leaf_table
    adm = np.flatnonzero(t[:, 0] == 1)
    b = adm[np.argmax((t[adm, 2] - t[adm, 1]) * (t[adm, 4] - t[adm, 3]))]
    _, r0, r1, c0, c1 = t[b][:5]
    gen = hmx.BlockGenerator(spec, ct.points_tree[r0:r1], ct.points_tree[c0:c1], ct.normals_tree[c0:c1])
    with pytest.raises(hmx.FallbackNeeded):
        hmx.aca_vector(gen, hmx.ACAConfig(eps_aca=1e-4))
    A = gen.dense()
    f = hmx.randomized_svd(gen, 1e-4, seed=7)
    assert f.converged
    assert np.linalg.norm(A - f.dense()) <= 1e-4 * np.linalg.norm(A)
    g = hmx.recompress(f, 1e-4)
    assert g.rank <= f.rank and np.linalg.norm(A - g.dense()) <= 3e-4 * np.linalg.norm(A)


def test_assemble_routes_fallback_leaves_through_rsvd():
    cl, spec, ct, bt = _plate_t()
    H, rep = hmx.assemble(spec, cl, ct, bt, hmx.ACAConfig(eps_aca=1e-4))
    st = H.stats()
    t = bt.leaf_table
    adm = np.flatnonzero(t[:, 0] == 1)
    assert st["n_fallback"] == len(adm) > 0  # every coplanar admissible leaf
    info = H.block_info()
    assert np.all(info["flags"][adm] & 8)
    # every fallback leaf within the compression bar against its dense block
    k = spec.c_kernel()
    worst = 0.0
    for b in adm:
        _, r0, r1, c0, c1 = t[b][:5]
        X, Y, NY = ct.points_tree[r0:r1], ct.points_tree[c0:c1], ct.normals_tree[c0:c1]
        A = hmx.elasto_t_block(k.kp, k.ks, k.lam, k.mu, k.scale, X, Y, NY)
        worst = max(worst, np.linalg.norm(A - H.block(int(b)).dense()) / np.linalg.norm(A))
    assert worst <= 3e-4, worst
    # ranks against the oracle's own fallback (numpy range finder + QR/SVD recompression)
    params = oracle_params(spec)
    oh = OH.assemble("T", params, ct.points_tree, ct.normals_tree, ct.permutation, t, 1e-4,
                     self_shift=float(cl.size), workers=4)
    assert oh.fallback[adm].all()
    assert np.abs(info["rank_after"][adm] - oh.rank_after[adm]).max() <= 2
    # the matvec of the assembled H against the dense operator
    rng = np.random.default_rng(0)
    x = rng.standard_normal(3 * cl.size) + 1j * rng.standard_normal(3 * cl.size)
    Ad = OH.dense_matrix("T", params, ct.points_tree, ct.normals_tree, float(cl.size))
    yd = OH.from_tree(oh, Ad @ OH.to_tree(oh, x))
    assert np.linalg.norm(hmx.matvec(H, x) - yd) <= 3e-4 * np.linalg.norm(yd)
