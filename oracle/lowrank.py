"""Oracle: ACA (scalar + sigma_3 vector), randomized SVD, recompression.  TEST INFRASTRUCTURE.

The reference module that holds these (``hmatx/lowrank.py``) is absent from
the mount; this file restates SPEC.md:243-354 and
PAPER.md:261-382, 431-443.  Every choice SPEC leaves open is pinned here and
is mirrored 1:1 by the CUDA ACA kernel (``csrc/aca.cu``):

1. first pivot row = block-local point 0;
2. column pivot = argmax over ALL column points of sigma_3 of the d x d
   residual sub-block in the current row strip (|.| for d = 1); next row pivot
   = argmax over UNVISITED row points of sigma_3 of the pre-update residual
   column strip; ties -> lowest index (``np.argmax``);
3. zero residual row (max_j sigma_1 <= floor * sigma1_max, floor =
   ``sigma3_floor``) -> mark it visited and continue with the lowest unvisited
   row without adding rank; no unvisited row left -> converged;
4. sigma_3 of the chosen pivot <= floor * sigma1_max on a non-zero row ->
   ``FallbackNeeded``; sigma1_max = largest sigma_1 of any
   candidate sub-block seen so far;
5. ||B_k||_F^2 exact incremental: ||B_{k-1}||^2 + 2 Re tr((U^H u)(v^H V))
   + tr((u^H u)(v^H v));
6. stop when ||u_k||_F ||v_k||_F <= eps ||B_k||_F;
7. max_rank default min(d m, d n); reaching max_rank stops with
   converged False unless it equals min(d m, d n) (then B_k interpolates every
   row or every column: exact);
8. recompression truncation: ``"frobenius"`` (default) keeps the smallest r
   with sqrt(sum_{i>r} s_i^2) <= eps * sqrt(sum s_i^2) -- this is the
   postcondition SPEC.md:321 states; ``"spectral"`` keeps s_i > eps * s_1
   (Eq. num_rank).  SURVEY 0.6 records the conflict.
"""

from dataclasses import dataclass, field

import numpy as np

from . import kernels


class FallbackNeeded(RuntimeError):
    """Vector ACA found only (near-)singular pivot sub-blocks (``errors.py:12-16``)."""


@dataclass
class ACAResult:
    U: np.ndarray          # (d m, K)
    V: np.ndarray          # (d n, K)   block ~= U V^H
    steps: int             # ACA steps (rank K = d * steps)
    converged: bool
    pivots: list = field(default_factory=list)   # [(row_pt, col_pt), ...]


class BlockGen:
    """Row / column strips of one kernel block."""

    def __init__(self, kind, params, X, Y, NY=None, self_shift=None):
        self.kind, self.params = kind, params
        self.X, self.Y, self.NY = X, Y, NY
        self.self_shift = self_shift
        self.d = 1 if kind == "H" else 3
        self.m, self.n = X.shape[0], Y.shape[0]

    def _eval(self, X, Y, NY):
        out = kernels.block(self.kind, self.params, X, Y, NY, self.self_shift)
        if out is None:
            raise ValueError("singular evaluation")
        return out

    def row(self, i):
        """d x (d n) strip of point row i."""
        return self._eval(self.X[i : i + 1], self.Y, self.NY)

    def col(self, j):
        """(d m) x d strip of point column j."""
        NY = None if self.NY is None else self.NY[j : j + 1]
        return self._eval(self.X, self.Y[j : j + 1], NY)

    def dense(self):
        return self._eval(self.X, self.Y, self.NY)


def _sub_svals(strip_blocks):
    """(cnt, d, d) -> sigma_1, sigma_d per sub-block."""
    if strip_blocks.shape[1] == 1:
        a = np.abs(strip_blocks[:, 0, 0])
        return a, a
    sv = np.linalg.svd(strip_blocks, compute_uv=False)
    return sv[:, 0], sv[:, -1]


def aca(gen, eps, max_rank=None, sigma3_floor=1e-12):
    """Partially pivoted ACA; d = 1 is ``aca_partial``, d = 3
    ``aca_vector``.  Returns an :class:`ACAResult`."""
    d, m, n = gen.d, gen.m, gen.n
    if max_rank is None:
        max_rank = min(d * m, d * n)
    Ucols, Vcols = [], []
    U = np.zeros((d * m, 0), complex)
    V = np.zeros((d * n, 0), complex)
    visited = np.zeros(m, bool)
    normB2 = 0.0
    s1max = 0.0
    steps = 0
    converged = False
    pivots = []
    i = 0
    while True:
        visited[i] = True
        row = gen.row(i)                                   # (d, d n)
        if steps:
            row = row - U[d * i : d * i + d, :] @ V.conj().T
        sub = row.reshape(d, n, d).transpose(1, 0, 2)      # sub-block j: row[:, d j : d j + d]
        s1, s3 = _sub_svals(sub)
        rmax = float(s1.max())
        s1max = max(s1max, rmax)
        if rmax <= sigma3_floor * s1max or s1max == 0.0:
            # zero residual row: next unvisited row, no rank added (decision 3)
            free = np.flatnonzero(~visited)
            if free.size == 0:
                converged = True
                break
            i = int(free[0])
            continue
        j = int(np.argmax(s3))
        if s3[j] <= sigma3_floor * s1max:
            raise FallbackNeeded("all pivot sub-blocks singular")
        P = sub[j]
        col = gen.col(j)                                   # (d m, d)
        if steps:
            col = col - U @ V[d * j : d * j + d, :].conj().T
        _, cs3 = _sub_svals(col.reshape(m, d, d))
        u = col @ np.linalg.inv(P)
        v = row.conj().T
        if steps:
            cross = np.trace((U.conj().T @ u) @ (v.conj().T @ V)).real
        else:
            cross = 0.0
        normB2 = normB2 + 2.0 * cross + np.trace((u.conj().T @ u) @ (v.conj().T @ v)).real
        U = np.concatenate([U, u], axis=1)
        V = np.concatenate([V, v], axis=1)
        steps += 1
        pivots.append((i, j))
        if np.linalg.norm(u) * np.linalg.norm(v) <= eps * np.sqrt(max(normB2, 0.0)):
            converged = True
            break
        if d * steps >= max_rank:
            # full rank min(dm, dn) reached -> interpolation is exact
            converged = d * steps >= min(d * m, d * n)
            break
        cs3 = np.where(visited, -1.0, cs3)
        if not (~visited).any():
            converged = True
            break
        i = int(np.argmax(cs3))
    return ACAResult(U=U, V=V, steps=steps, converged=converged, pivots=pivots)


def aca_full(A, eps, max_rank=None):
    """Fully pivoted ACA on a dense matrix; returns (U, V, converged)."""
    R = np.array(A, dtype=complex)
    m, n = R.shape
    if max_rank is None:
        max_rank = min(m, n)
    nA = np.linalg.norm(R)
    Us, Vs = [], []
    while np.linalg.norm(R) > eps * nA and len(Us) < max_rank:
        k = int(np.argmax(np.abs(R)))
        i, j = divmod(k, n)
        u = R[:, j] / R[i, j]
        v = R[i, :].conj()
        Us.append(u); Vs.append(v)
        R = R - np.outer(u, v.conj())
    conv = np.linalg.norm(R) <= eps * nA
    U = np.array(Us).T if Us else np.zeros((m, 0), complex)
    V = np.array(Vs).T if Vs else np.zeros((n, 0), complex)
    return U, V, bool(conv)


def numerical_rank(A, eps):
    """Smallest r with sigma_{r+1} <= eps sigma_1 (Eq. num_rank)."""
    s = np.linalg.svd(A, compute_uv=False)
    if s.size == 0 or s[0] == 0.0:
        return 0
    return int(np.count_nonzero(s > eps * s[0]))


def truncation_rank(s, eps, rule="frobenius"):
    """Kept rank for singular values ``s`` (descending) -- decision 8."""
    if s.size == 0 or s[0] == 0.0:
        return 0
    if rule == "spectral":
        return int(np.count_nonzero(s > eps * s[0]))
    # tail[r] = sum_{i >= r} s_i^2 ; smallest r with tail[r] <= eps^2 * total
    sq = s * s
    tail = np.concatenate([np.cumsum(sq[::-1])[::-1], [0.0]])
    ok = np.flatnonzero(tail <= (eps * eps) * tail[0])
    return int(ok[0])


def recompress(U, V, eps, rule="frobenius"):
    """QR(U), QR(V), SVD(R_U R_V^H), truncate, U' = Q_U P S^1/2, V' = Q_V L S^1/2
    (SPEC.md:318-326)."""
    if U.shape[1] == 0:
        return U.copy(), V.copy()
    Qu, Ru = np.linalg.qr(U)
    Qv, Rv = np.linalg.qr(V)
    P, s, Lh = np.linalg.svd(Ru @ Rv.conj().T)
    r = truncation_rank(s, eps, rule)
    root = np.sqrt(s[:r])
    return (Qu @ P[:, :r]) * root, (Qv @ Lh.conj().T[:, :r]) * root


def randomized_svd(A, eps, oversample=10, max_rank=None, seed=0):
    """Adaptive range finder with a Gaussian test matrix.

    Rank doubles from 8 until ||A - Q Q^H A||_F <= eps ||A||_F (the block is
    regenerated densely, as SPEC allows "matvec or dense").  Returns (U, V, conv).
    """
    A = np.asarray(A, dtype=complex)
    m, n = A.shape
    cap = min(m, n) if max_rank is None else max_rank
    nA = np.linalg.norm(A)
    if nA == 0.0:
        return np.zeros((m, 0), complex), np.zeros((n, 0), complex), True
    rng = np.random.default_rng(seed)
    k = 8
    while True:
        kk = min(k + oversample, min(m, n))
        Om = rng.standard_normal((n, kk)) + 1j * rng.standard_normal((n, kk))
        Q, _ = np.linalg.qr(A @ Om)
        B = Q.conj().T @ A
        err = np.linalg.norm(A - Q @ B)
        if err <= eps * nA or kk >= cap:
            return Q, B.conj().T, bool(err <= eps * nA)
        k *= 2
