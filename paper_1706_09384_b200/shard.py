"""Row-sharded H-matrix over several processes.

One process per GPU.  The rows [0, N) (tree order) are cut at points no leaf
straddles into one contiguous owned range per rank, balanced on the leaf
cost; rank p owns every leaf whose row range lies in its range.  The
admissible and dense leaves are independent, so the
assembly shards with no collective at all.  The H-matvec has one exchange
step: every rank applies its own leaves to the replicated x, which fills
exactly its owned rows of y, and one all-gather of the owned segments (d N
complex128 in total, 1.5 MB at U32k) hands every rank the full y.  GMRES runs
replicated on every rank on top of that matvec; every rank holds the same y,
so all ranks take the same Krylov steps and stop together without further
collectives.

The collective goes through ``torch.distributed`` (NCCL on the GPUs, gloo in
the CPU tests); the per-rank compute is the C-ABI (``hmx_assemble`` on a leaf
subset, ``hmx_matvec`` on device pointers).
"""

import numpy as np

from .solve import GmresConfig, GmresResult


def leaf_cost(table, d, rank_est=None):
    """Per-leaf matvec-byte proxy: d^2 m n for dense leaves, r d (m + n) for
    admissible ones (r from ``rank_est`` per leaf, default 2 d log2-size)."""
    t = np.asarray(table)
    m = (t[:, 2] - t[:, 1]).astype(np.float64)
    n = (t[:, 4] - t[:, 3]).astype(np.float64)
    if rank_est is None:
        rank_est = 2.0 * d * np.log2(np.maximum(m + n, 2.0))
    cost = np.where(t[:, 0] == 0, d * d * m * n, np.asarray(rank_est, np.float64) * d * (m + n))
    return cost


def safe_row_cuts(table, n_points):
    """Tree-order row positions p in [0, N] that no leaf straddles (no leaf has r0 < p < r1):
    cutting the rows there gives every leaf to exactly one owner of its whole row range."""
    t = np.asarray(table)
    diff = np.zeros(int(n_points) + 2, np.int64)
    np.add.at(diff, t[:, 1] + 1, 1)
    np.add.at(diff, t[:, 2], -1)
    inside = np.cumsum(diff)[: int(n_points) + 1]
    return np.flatnonzero(inside == 0)


def partition_row_ranges(table, n_parts, n_points, cost=None, d=3):
    """Split the rows [0, N) (tree order) into ``n_parts`` contiguous owned ranges at safe cut
    points, each near an equal share of the cumulative leaf cost; every leaf goes to the owner of
    its row range.  Returns (parts, bounds): sorted leaf-index arrays (together a partition of
    range(len(table))) and the n_parts + 1 row bounds."""
    t = np.asarray(table)
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    if cost is None:
        cost = leaf_cost(t, d)
    cost = np.asarray(cost, np.float64)
    N = int(n_points)
    safe = safe_row_cuts(t, N)
    # cumulative cost of the leaves lying entirely below each safe point
    per_row_end = np.zeros(N + 1)
    np.add.at(per_row_end, t[:, 2], cost)
    cum = np.cumsum(per_row_end)[safe]
    total = float(cost.sum())
    bounds = [0]
    for k in range(1, n_parts):
        target = total * k / n_parts
        j = int(np.argmin(np.abs(cum - target)))
        bounds.append(max(int(safe[j]), bounds[-1]))
    bounds.append(N)
    bounds = np.asarray(bounds, np.int64)
    owner = np.searchsorted(bounds, t[:, 1], side="right") - 1
    parts = [np.flatnonzero(owner == k) for k in range(n_parts)]
    return parts, bounds


def partition_block_rows(table, n_parts, cost=None, d=3, n_points=None):
    """The leaf parts of :func:`partition_row_ranges` (n_points defaults to the table's extent)."""
    t = np.asarray(table)
    N = int(t[:, 2].max()) if n_points is None else int(n_points)
    return partition_row_ranges(t, n_parts, N, cost=cost, d=d)[0]


class LeafSubset:
    """Block-tree stand-in carrying a subset of the leaf table (what
    ``hmatrix.assemble`` reads from a block tree)."""

    def __init__(self, bt, idx):
        self.idx = np.asarray(idx, np.int64)
        self.leaf_table = np.ascontiguousarray(np.asarray(bt.leaf_table)[self.idx])
        self.table = np.ascontiguousarray(np.asarray(bt.table)[self.idx])  # + row / column node ids
        self.rows, self.cols, self.eta = bt.rows, bt.cols, bt.eta


class RowExchange:
    """The matvec's exchange step: rank k computed the rows it owns (tree rows
    [bounds[k], bounds[k+1]), i.e. original dofs d perm[t] + a); one all-gather of the owned
    segments hands every rank the full y (d N complex128, half the bytes of an all-reduce)."""

    def __init__(self, bounds, perm, d, rank, world, device="cpu", group=None):
        import torch

        perm = np.asarray(perm, np.int64)
        self.world, self.rank, self.group = world, rank, group
        dofs = [(d * perm[bounds[k]:bounds[k + 1]][:, None] + np.arange(d)[None, :]).ravel() for k in range(world)]
        self.counts = [len(x) for x in dofs]
        self.L = max(max(self.counts), 1)
        self.own = torch.as_tensor(dofs[rank], device=device)
        self.all = torch.as_tensor(np.concatenate(dofs), device=device)

    def __call__(self, y_local):
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return y_local
        seg = torch.zeros(self.L, dtype=y_local.dtype, device=y_local.device)
        seg[: self.counts[self.rank]] = y_local[self.own]
        outs = [torch.empty_like(seg) for _ in range(self.world)]
        dist.all_gather([torch.view_as_real(o) for o in outs], torch.view_as_real(seg), group=self.group)
        y = torch.empty_like(y_local)
        y[self.all] = torch.cat([o[:c] for o, c in zip(outs, self.counts)])
        return y


def sharded_matvec(local_apply, x, exchange):
    """y = sum_p A_p x: ``local_apply(x)`` returns this rank's product (non-zero only on its
    owned rows); ``exchange`` (a RowExchange) assembles the full y on every rank."""
    return exchange(local_apply(x))


class ShardedHMatrix:
    """This rank's row range of a row-sharded H-matrix."""

    def __init__(self, local, part_idx, n_points, d, bounds=None, exchange=None, group=None):
        self.local = local  # HMatrix of this rank's leaves (None: no leaves)
        self.part_idx = part_idx
        self.n_points = n_points
        self.d = d
        self.bounds = bounds
        self.exchange = exchange
        self.group = group

    def apply_local(self, x):
        import torch

        if self.local is None:
            return torch.zeros_like(x)
        from .hmatrix import matvec

        return matvec(self.local, x)

    def matvec(self, x):
        """x: CUDA complex128 tensor in original point order (replicated)."""
        return sharded_matvec(self.apply_local, x, self.exchange)


def assemble_sharded(spec, cloud, ct, bt, cfg, rank, world, group=None, device=0, cost=None):
    """Assemble rank ``rank``'s owned row range (no collective)."""
    from .hmatrix import assemble

    parts, bounds = partition_row_ranges(bt.leaf_table, world, cloud.size, cost=cost, d=spec.d)
    idx = parts[rank]
    local = None
    if len(idx):
        local, _ = assemble(spec, cloud, ct, LeafSubset(bt, idx), cfg, device=device)
    ex = RowExchange(bounds, ct.permutation, spec.d, rank, world, device=f"cuda:{device}", group=group)
    return ShardedHMatrix(local, idx, cloud.size, spec.d, bounds=bounds, exchange=ex, group=group)


def _givens(a, b):
    """Complex Givens rotation (oracle/solve.py givens; csrc/gmres.cu)."""
    if b == 0:
        return 1.0, 0.0 + 0.0j, a
    if a == 0:
        return 0.0, np.conj(b) / abs(b), abs(b) + 0.0j
    t = np.hypot(abs(a), abs(b))
    ph = a / abs(a)
    return abs(a) / t, ph * np.conj(b) / t, ph * t


def gmres(apply, b, cfg=GmresConfig()):
    """Restarted GMRES on torch tensors with an arbitrary operator (the
    sharded matvec): x0 = 0, MGS Arnoldi, complex Givens rotations, stop on
    |g_{j+1}| <= tol ||b||, explicit residual at each restart -- the
    algorithm of csrc/gmres.cu / oracle/solve.py.  Every reduction result is
    replicated, so all ranks follow the same iteration."""
    import torch

    m = int(cfg.restart)
    bnorm = float(torch.linalg.vector_norm(b))
    x = torch.zeros_like(b)
    hist = []
    if bnorm == 0.0:
        return GmresResult(x=x, iters=0, history=hist, converged=True)
    iters = 0
    beta = bnorm
    r = b
    converged = False
    while True:
        V = [r / beta]
        Hm = np.zeros((m + 1, m), np.complex128)
        g = np.zeros(m + 1, np.complex128)
        cs = np.zeros(m)
        sn = np.zeros(m, np.complex128)
        g[0] = beta
        k = 0
        done = False
        for j in range(m):
            w = apply(V[j])
            iters += 1
            for i in range(j + 1):
                h = torch.vdot(V[i], w)
                w = w - h * V[i]
                Hm[i, j] = complex(h)
            hn = float(torch.linalg.vector_norm(w))
            Hm[j + 1, j] = hn
            for i in range(j):
                t0 = cs[i] * Hm[i, j] + sn[i] * Hm[i + 1, j]
                Hm[i + 1, j] = -np.conj(sn[i]) * Hm[i, j] + cs[i] * Hm[i + 1, j]
                Hm[i, j] = t0
            c, s, rr = _givens(Hm[j, j], Hm[j + 1, j])
            cs[j], sn[j] = c, s
            Hm[j, j], Hm[j + 1, j] = rr, 0.0
            g[j + 1] = -np.conj(s) * g[j]
            g[j] = c * g[j]
            res = abs(g[j + 1])
            hist.append(res / bnorm)
            k = j + 1
            if res <= cfg.tol * bnorm:
                done = True
                break
            if iters >= cfg.max_iters or hn == 0.0:
                break
            V.append(w / hn)
        y = np.zeros(k, np.complex128)
        for i in range(k - 1, -1, -1):
            s = g[i] - np.dot(Hm[i, i + 1:k], y[i + 1:k])
            y[i] = s / Hm[i, i]
        for i in range(k):
            x = x + complex(y[i]) * V[i]
        if done:
            converged = True
            break
        if iters >= cfg.max_iters:
            break
        r = b - apply(x)
        beta = float(torch.linalg.vector_norm(r))
        if beta <= cfg.tol * bnorm:
            converged = True
            break
    return GmresResult(x=x, iters=iters, history=hist, converged=converged)
