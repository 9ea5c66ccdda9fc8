"""Oracle: H-matrix assemble / matvec / storage report (CPU).  TEST INFRASTRUCTURE.

Restates SPEC.md:356-439 (reference ``hmatx/hmatrix.py`` is absent from the
mount).  Dense leaves come from ``oracle.kernels`` (= the reference's
``_kernelcore_np`` numerics) with the self-block rule zeta = N_c
(SPEC.md:226); admissible leaves run ``oracle.lowrank.aca`` then
``recompress`` with eps_ACA, switching to ``randomized_svd`` when the vector
ACA signals ``FallbackNeeded``.

``matvec`` follows SPEC.md:391-399: x in original point order, permuted to
tree order with the cluster-tree permutation, leaf contributions accumulated
in ``BlockTree.leaves()`` order, result permuted back.
"""

import math
import multiprocessing as mp
from dataclasses import dataclass, field

import numpy as np

from . import kernels, lowrank

DENSE, ADMISSIBLE = 0, 1


@dataclass
class OracleH:
    kind: str
    d: int
    n_points: int
    perm: np.ndarray            # (N,) tree slot -> original point
    table: np.ndarray           # (nb, 5) kind, r0, r1, c0, c1 (points, tree order)
    payload: list               # dense (d m, d n) array  or  (U, V)
    steps: np.ndarray           # ACA steps per block (0 for dense)
    rank_before: np.ndarray     # d * steps (or rSVD rank)
    rank_after: np.ndarray
    converged: np.ndarray       # bool
    fallback: np.ndarray        # bool: rSVD used
    n_leaf: int = 0
    c_sp: int = 0
    pivots: list = field(default_factory=list)


_G = {}


def _leaf(b):
    g = _G
    k, r0, r1, c0, c1 = (int(t) for t in g["table"][b])
    X = g["pts"][r0:r1]
    Y = g["pts"][c0:c1]
    NY = None if g["nrm"] is None else g["nrm"][c0:c1]
    if k == DENSE:
        out = kernels.block(g["kind"], g["params"], X, Y, NY, g["self_shift"])
        if out is None:
            raise ValueError("singular evaluation")
        return b, out, 0, 0, 0, True, False, []
    gen = lowrank.BlockGen(g["kind"], g["params"], X, Y, NY, g["self_shift"])
    fb = False
    try:
        res = lowrank.aca(gen, g["eps"], g["max_rank"], g["sigma3_floor"])
        U, V, steps, conv, piv = res.U, res.V, res.steps, res.converged, res.pivots
    except lowrank.FallbackNeeded:
        fb = True
        U, V, conv = lowrank.randomized_svd(gen.dense(), g["eps"], seed=b)
        steps, piv = 0, []
    kb = U.shape[1]
    Ur, Vr = lowrank.recompress(U, V, g["eps"], g["rule"])
    return b, (Ur, Vr), steps, kb, Ur.shape[1], conv, fb, piv


def _init(state, single_thread=False):
    _G.clear()
    _G.update(state)
    if single_thread:
        # one BLAS thread per pool worker: the pool already uses every core
        from threadpoolctl import threadpool_limits
        _G["_limits"] = threadpool_limits(1)


def assemble(kind, params, points_tree, normals_tree, perm, table, eps, *,
             max_rank=None, sigma3_floor=1e-12, self_shift=None, rule="frobenius",
             workers=1, n_leaf=0):
    """Assemble the oracle H-matrix.  ``workers > 1`` runs
    leaves in a fork pool (SPEC.md:456 allows leaf-parallel assembly)."""
    d = 1 if kind == "H" else 3
    N = points_tree.shape[0]
    state = dict(kind=kind, params=params, pts=points_tree, nrm=normals_tree,
                 table=np.asarray(table), eps=eps, max_rank=max_rank,
                 sigma3_floor=sigma3_floor,
                 self_shift=float(N) if self_shift is None else self_shift, rule=rule)
    nb = len(table)
    if workers > 1:
        ctx = mp.get_context("fork")
        # big blocks first for balance
        cost = (table[:, 2] - table[:, 1]) + (table[:, 4] - table[:, 3])
        order = np.argsort(-cost, kind="stable").tolist()
        with ctx.Pool(workers, initializer=_init, initargs=(state, True)) as pool:
            results = pool.map(_leaf, order, chunksize=8)
    else:
        _init(state)
        results = [_leaf(b) for b in range(nb)]
    results.sort(key=lambda t: t[0])
    payload = [t[1] for t in results]
    return OracleH(
        kind=kind, d=d, n_points=N, perm=np.asarray(perm), table=np.asarray(table),
        payload=payload,
        steps=np.array([t[2] for t in results], dtype=np.int64),
        rank_before=np.array([t[3] for t in results], dtype=np.int64),
        rank_after=np.array([t[4] for t in results], dtype=np.int64),
        converged=np.array([t[5] for t in results], dtype=bool),
        fallback=np.array([t[6] for t in results], dtype=bool),
        n_leaf=n_leaf,
        pivots=[t[7] for t in results],
    )


def to_tree(h, x):
    return x.reshape(h.n_points, h.d)[h.perm].reshape(-1)


def from_tree(h, y_tree):
    y = np.empty_like(y_tree)
    y.reshape(h.n_points, h.d)[h.perm] = y_tree.reshape(h.n_points, h.d)
    return y


def matvec_tree(h, xt):
    d = h.d
    yt = np.zeros(h.d * h.n_points, dtype=complex)
    for (k, r0, r1, c0, c1), p in zip(h.table, h.payload):
        xs = xt[d * c0 : d * c1]
        if k == DENSE:
            yt[d * r0 : d * r1] += p @ xs
        else:
            U, V = p
            if U.shape[1]:
                yt[d * r0 : d * r1] += U @ (V.conj().T @ xs)
    return yt


def matvec(h, x):
    """y = A_H x, x in original point order."""
    x = np.asarray(x, dtype=complex)
    if x.shape != (h.d * h.n_points,):
        raise ValueError("dimension mismatch")
    return from_tree(h, matvec_tree(h, to_tree(h, x)))


def dense_matrix(kind, params, points_tree, normals_tree, self_shift):
    """Full (dN, dN) kernel matrix in tree order (for dense checks, small N)."""
    out = kernels.block(kind, params, points_tree, points_tree, normals_tree, self_shift)
    if out is None:
        raise ValueError("singular evaluation")
    return out


def storage_report(h):
    """N_s, tau, max ranks, and the section-5.1 bound."""
    d = h.d
    ns = 0
    for (k, r0, r1, c0, c1), ra in zip(h.table, h.rank_after):
        m, n = r1 - r0, c1 - c0
        ns += d * d * m * n if k == DENSE else int(ra) * d * (m + n)
    N = d * h.n_points
    rmax_after = int(h.rank_after.max()) if len(h.rank_after) else 0
    rmax_before = int(h.rank_before.max()) if len(h.rank_before) else 0
    bound = None
    if h.n_leaf and h.c_sp:
        nl = d * h.n_leaf
        bound = 2 * h.c_sp * max(rmax_after, nl) * N * (math.log2(N) - math.log2(nl) + 1)
    return dict(n_stored=int(ns), n_dense_equiv=N * N, tau=ns / float(N * N),
                max_rank_before=rmax_before, max_rank_after=rmax_after, bound=bound)


def matvec_tree_threads(h, xt, pool, chunks):
    """Leaf-parallel oracle matvec ("matvec parallelizes across
    sibling blocks with per-output-range accumulation"): ``chunks`` is a list
    of leaf-index lists; each worker thread accumulates its own y, the partial
    vectors are summed in chunk order (deterministic).  numpy's BLAS calls
    release the GIL, so the threads overlap the GEMV work."""
    d = h.d

    def work(idx):
        yt = np.zeros(h.d * h.n_points, dtype=complex)
        for b in idx:
            k, r0, r1, c0, c1 = h.table[b]
            p = h.payload[b]
            xs = xt[d * c0 : d * c1]
            if k == DENSE:
                yt[d * r0 : d * r1] += p @ xs
            elif p[0].shape[1]:
                yt[d * r0 : d * r1] += p[0] @ (p[1].conj().T @ xs)
        return yt

    parts = list(pool.map(work, chunks))
    y = parts[0]
    for p in parts[1:]:
        y += p
    return y
