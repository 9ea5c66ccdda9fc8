"""hmx_hlu_truncate (the H-arithmetic truncation of the H-LU engine: direct / dense-form / range-sketch routes) against numpy's SVD truncation
on random factor pairs: full-rank, numerically low-rank with dependent columns, K above
the row count, single columns; Frobenius and spectral rules."""

import numpy as np
import pytest
import torch

from oracle.lowrank import truncation_rank
from paper_1706_09384_b200 import hierarchical_lu as HL

pytestmark = pytest.mark.gpu


def _case(rng, dm, dn, K, r_true=None, decay=None):
    def g(*s):
        return rng.standard_normal(s) + 1j * rng.standard_normal(s)
    if r_true is None:
        U, V = g(dm, K), g(dn, K)
        if decay is not None:
            U = U * (decay ** np.arange(K))[None, :]
    else:
        U = g(dm, r_true) @ g(r_true, K)
        V = g(dn, r_true) @ g(r_true, K)
    return U, V


@pytest.mark.parametrize("rule", ["frobenius", "spectral"])
def test_truncate_batch_matches_svd(rule):
    rng = np.random.default_rng(0)
    cases = [(40, 30, 10, None, None), (96, 96, 60, None, 0.7), (35, 40, 88, None, 0.8), (200, 150, 20, 5, None),
             (64, 64, 1, None, None), (300, 120, 130, None, 0.9), (50, 70, 0, None, None)]
    items, ref = [], []
    for dm, dn, K, rt, dec in cases:
        U, V = _case(rng, dm, dn, K, rt, dec)
        items.append((torch.as_tensor(U, device="cuda"), torch.as_tensor(V, device="cuda")))
        ref.append(U @ V.conj().T)
    eps = 1e-6
    out = HL.truncate_pairs(items, eps, rule)
    for (u, v), A, (dm, dn, K, _, _) in zip(out, ref, cases):
        s = np.linalg.svd(A, compute_uv=False)
        r_ref = truncation_rank(s, eps, rule)
        assert abs(u.shape[1] - r_ref) <= 1, (dm, dn, K, u.shape[1], r_ref)
        B = (u @ v.mH).cpu().numpy()
        nA = max(np.linalg.norm(A), 1e-300)
        tol = 3 * eps if rule == "frobenius" else 3 * eps * np.sqrt(min(dm, dn))
        assert np.linalg.norm(B - A) <= tol * nA + 1e-300, (dm, dn, K, np.linalg.norm(B - A) / nA)


def test_sketched_dense_form():
    """Dense-form pairs above the sketch threshold (K >= min(dm, dn) > 112) go through the
    range sketch: same truncation rank (+-1) and error as the SVD truncation, also when the
    numerical rank is near the sketch width and for the adjoint orientation."""
    rng = np.random.default_rng(1)
    eps = 1e-4
    cases = [(150, 200, 260, 30), (260, 140, 300, 60), (200, 200, 400, 85), (130, 144, 232, 5)]
    items, ref = [], []
    for dm, dn, K, r in cases:
        s = np.exp(-np.arange(K) / (r / 4.0))   # singular-value decay: numerical rank ~ r
        U = (rng.standard_normal((dm, K)) + 1j * rng.standard_normal((dm, K))) * s
        V = rng.standard_normal((dn, K)) + 1j * rng.standard_normal((dn, K))
        items.append((torch.as_tensor(U, device="cuda"), torch.as_tensor(V, device="cuda")))
        ref.append(U @ V.conj().T)
    out = HL.truncate_pairs(items, eps)
    for (u, v), A, c in zip(out, ref, cases):
        sv = np.linalg.svd(A, compute_uv=False)
        r_ref = truncation_rank(sv, eps, "frobenius")
        assert abs(u.shape[1] - r_ref) <= 1, (c, u.shape[1], r_ref)
        err = np.linalg.norm((u @ v.mH).cpu().numpy() - A) / np.linalg.norm(A)
        assert err <= 1.5 * eps, (c, err)
