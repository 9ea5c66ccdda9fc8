"""Block-row sharding on CPU: the leaf partition, and the
sharded matvec / replicated GMRES over a world-size-2 gloo group with a CPU
operator built from a real block tree (every leaf a slice of one dense matrix,
so the leaves of all ranks together cover it exactly once)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1706_09384_b200 as hmx
from paper_1706_09384_b200.shard import (RowExchange, gmres, leaf_cost, partition_row_ranges, safe_row_cuts,
                                         sharded_matvec)


def _tree(n=400, leaf=16):
    cloud = hmx.make_geometry("sphere", n, 1.0, d=1)
    ct = hmx.build_cluster_tree(cloud, leaf)
    bt = hmx.build_block_tree(ct, ct, 3.0)
    return np.asarray(bt.leaf_table)[:, :5].astype(np.int64)


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_partition_covers_and_balances(parts):
    t = _tree()
    n = int(t[:, 2].max())
    cost = leaf_cost(t, 1)
    ps, bounds = partition_row_ranges(t, parts, n, cost=cost, d=1)
    assert len(ps) == parts and bounds[0] == 0 and bounds[-1] == n and np.all(np.diff(bounds) >= 0)
    allidx = np.concatenate(ps)
    assert np.array_equal(np.sort(allidx), np.arange(len(t)))  # a partition of the leaves
    safe = set(safe_row_cuts(t, n).tolist())
    assert all(int(b) in safe for b in bounds)
    for k, p in enumerate(ps):  # each part owns whole leaves inside its row range
        assert np.all(t[p, 1] >= bounds[k]) and np.all(t[p, 2] <= bounds[k + 1])
    loads = np.array([cost[p].sum() for p in ps])
    # cuts only at safe points: a part can be off the mean by at most the cost between two
    # neighbouring safe cuts
    per_end = np.zeros(n + 1)
    np.add.at(per_end, t[:, 2], cost)
    cum = np.cumsum(per_end)[sorted(safe)]
    assert loads.max() - loads.sum() / parts <= np.diff(cum).max() + 1e-9


def test_safe_cuts_are_cluster_boundaries():
    t = _tree()
    n = int(t[:, 2].max())
    safe = safe_row_cuts(t, n)
    assert safe[0] == 0 and safe[-1] == n
    for p in safe:
        assert not np.any((t[:, 1] < p) & (p < t[:, 2]))


def _operator(n, seed=3):
    rng = np.random.default_rng(seed)
    a = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    return a + 4.0 * np.eye(n)


def _local_apply(a, table, idx):
    def apply(x):
        xn = x.numpy()
        y = np.zeros_like(xn)
        for b in idx:
            _, r0, r1, c0, c1 = table[b]
            y[r0:r1] += a[r0:r1, c0:c1] @ xn[c0:c1]
        return torch.from_numpy(y)

    return apply


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = _tree()
    n = int(t[:, 2].max())
    a = _operator(n)
    parts, bounds = partition_row_ranges(t, world, n, d=1)
    idx = parts[rank]
    local = _local_apply(a, t, idx)
    ex = RowExchange(bounds, np.arange(n), 1, rank, world)  # identity permutation: tree = original order
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.standard_normal(n) + 1j * rng.standard_normal(n))
    y = sharded_matvec(local, x, ex)
    res = gmres(lambda v: sharded_matvec(local, v, ex), x, hmx.GmresConfig(tol=1e-10, restart=7))
    # a non-trivial permutation: rows owned in tree order, y gathered in original order
    perm = np.random.default_rng(5).permutation(n)
    ex2 = RowExchange(bounds, perm, 1, rank, world)
    inv = np.argsort(perm)

    def local_perm(x):  # y_orig[perm[i]] = (A x_tree)[i] restricted to this rank's leaves
        yt = local(torch.from_numpy(x.numpy()[perm]))
        return torch.from_numpy(yt.numpy()[inv])

    y2 = sharded_matvec(local_perm, x, ex2)
    q.put((rank, len(idx), y.numpy(), res.iters, res.x.numpy(), res.converged, y2.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_matvec_and_gmres_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in range(2)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t = _tree()
    n = int(t[:, 2].max())
    a = _operator(n)
    rng = np.random.default_rng(11)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert res[0][1] > 0 and res[1][1] > 0 and res[0][1] + res[1][1] == len(t)
    perm = np.random.default_rng(5).permutation(n)
    y_perm = (a @ x[perm])[np.argsort(perm)]
    for _, _, y, _, _, _, y2 in res:
        np.testing.assert_allclose(y, a @ x, rtol=0, atol=1e-12 * np.abs(a @ x).max())
        np.testing.assert_allclose(y2, y_perm, rtol=0, atol=1e-12 * np.abs(y_perm).max())
    # both ranks got the same y bit for bit, hence the same Krylov steps
    assert np.array_equal(res[0][2], res[1][2])
    assert res[0][3] == res[1][3] and np.array_equal(res[0][4], res[1][4])
    # single-process GMRES on the full operator: same iteration count, same solution
    ref = gmres(lambda v: torch.from_numpy(a @ v.numpy()), torch.from_numpy(x), hmx.GmresConfig(tol=1e-10, restart=7))
    assert res[0][5] and ref.converged
    assert abs(res[0][3] - ref.iters) <= 1
    np.testing.assert_allclose(res[0][4], ref.x.numpy(), rtol=0, atol=1e-8 * np.abs(ref.x.numpy()).max())
    assert np.linalg.norm(a @ res[0][4] - x) <= 1e-9 * np.linalg.norm(x)
