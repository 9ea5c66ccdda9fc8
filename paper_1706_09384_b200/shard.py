"""Block-row sharded H-matrix over several processes.

One process per GPU.  The admissible and dense leaves are independent
(SPEC.md:344, 456), so the assembly shards with no collective at all: rank p
assembles only the leaves of its block-row stripe.  The H-matvec has one
exchange step: every rank applies its own leaves to the replicated x and the
partial products are summed with one all-reduce of y (d N complex128, 1.5 MB
at U32k).  GMRES runs replicated on every rank on top of that matvec; the
all-reduce hands every rank the same y, so all ranks take the same Krylov
steps and stop together without further collectives.

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


def partition_block_rows(table, n_parts, cost=None, d=3):
    """Split the leaf list into ``n_parts`` block-row stripes: leaves ordered by
    (row start, row stop desc, column start), cut into contiguous runs of
    near-equal cumulative cost.  Returns a list of sorted leaf-index arrays
    (together a partition of range(len(table)))."""
    t = np.asarray(table)
    nb = len(t)
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    if cost is None:
        cost = leaf_cost(t, d)
    order = np.lexsort((t[:, 3], -t[:, 2], t[:, 1]))
    cum = np.cumsum(np.asarray(cost, np.float64)[order])
    total = cum[-1] if nb else 0.0
    # part p takes the leaves whose cumulative cost ends in (p/P, (p+1)/P] of the total
    bounds = np.searchsorted(cum, total * np.arange(1, n_parts) / n_parts, side="left")
    parts = np.split(order, bounds)
    return [np.sort(p) for p in parts]


class LeafSubset:
    """Block-tree stand-in carrying a subset of the leaf table (what
    ``hmatrix.assemble`` reads from a block tree)."""

    def __init__(self, bt, idx):
        self.idx = np.asarray(idx, np.int64)
        self.leaf_table = np.ascontiguousarray(np.asarray(bt.leaf_table)[self.idx])
        self.table = np.ascontiguousarray(np.asarray(bt.table)[self.idx])  # + row / column node ids
        self.rows, self.cols, self.eta = bt.rows, bt.cols, bt.eta


def allreduce_sum(y, group=None):
    """In-place sum of a complex128 torch tensor over the process group (the
    matvec's exchange step); identity on a single process."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return y
    v = torch.view_as_real(y)  # NCCL / gloo reduce real tensors
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    return y


def sharded_matvec(local_apply, x, group=None):
    """y = sum_p A_p x: ``local_apply(x)`` returns this rank's partial product
    (a torch tensor), summed over the group."""
    return allreduce_sum(local_apply(x), group)


class ShardedHMatrix:
    """This rank's stripe of a block-row sharded H-matrix."""

    def __init__(self, local, part_idx, n_points, d, group=None):
        self.local = local  # HMatrix of this rank's leaves (None: no leaves)
        self.part_idx = part_idx
        self.n_points = n_points
        self.d = d
        self.group = group

    def apply_local(self, x):
        import torch

        if self.local is None:
            return torch.zeros_like(x)
        from .hmatrix import matvec

        return matvec(self.local, x)

    def matvec(self, x):
        """x: CUDA complex128 tensor in original point order (replicated)."""
        return sharded_matvec(self.apply_local, x, self.group)


def assemble_sharded(spec, cloud, ct, bt, cfg, rank, world, group=None, device=0, cost=None):
    """Assemble rank ``rank``'s block-row stripe (no collective)."""
    from .hmatrix import assemble

    parts = partition_block_rows(bt.leaf_table, world, cost=cost, d=spec.d)
    idx = parts[rank]
    local = None
    if len(idx):
        local, _ = assemble(spec, cloud, ct, LeafSubset(bt, idx), cfg, device=device)
    return ShardedHMatrix(local, idx, cloud.size, spec.d, group)


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
