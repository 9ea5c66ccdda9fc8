"""Row-range sharding on one GPU: every part of a 2-, 3- and 4-way partition is
assembled through the C-ABI on its leaf subset; the stripes' device matvecs sum
to the full H-matvec, and the replicated torch GMRES over the (world-size-1)
sharded operator takes the device GMRES's iteration count."""

import numpy as np
import pytest
import torch

import paper_1706_09384_b200 as hmx
from paper_1706_09384_b200.shard import LeafSubset, ShardedHMatrix, assemble_sharded, gmres, partition_block_rows
from tests._problems import Problem

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag,n,parts", [("U8k", 2048, 2), ("T65k", 2048, 4), ("H4k", 4096, 3)])
def test_stripes_sum_to_full_matvec(tag, n, parts):
    pb = Problem(tag, n)
    H, _ = pb.device_h()
    x = torch.from_numpy(pb.rhs(1)).cuda()
    y_full = hmx.matvec(H, x)
    y = torch.zeros_like(x)
    cfg = hmx.ACAConfig(eps_aca=pb.w.eps)
    for idx in partition_block_rows(pb.table, parts, d=pb.d):
        Hp, _ = hmx.assemble(pb.spec, pb.cloud, pb.ct, LeafSubset(pb.bt, idx), cfg)
        # each stripe's leaves compress exactly as in the full assembly
        np.testing.assert_array_equal(Hp.block_info()["rank_after"], H.block_info()["rank_after"][idx])
        y += hmx.matvec(Hp, x)
    err = float(torch.linalg.vector_norm(y - y_full) / torch.linalg.vector_norm(y_full))
    assert err <= 1e-13, err


def test_sharded_gmres_world1_matches_device_gmres():
    pb = Problem("U8k", 2048)
    sh = assemble_sharded(pb.spec, pb.cloud, pb.ct, pb.bt, hmx.ACAConfig(eps_aca=pb.w.eps), rank=0, world=1)
    assert isinstance(sh, ShardedHMatrix) and len(sh.part_idx) == len(pb.table)
    b = pb.rhs(0)
    res = gmres(sh.matvec, torch.from_numpy(b).cuda(), hmx.GmresConfig(tol=1e-4, restart=50))
    ref = hmx.solve_gmres(sh.local, b, hmx.GmresConfig(tol=1e-4, restart=50))
    assert res.converged and ref.converged
    assert abs(res.iters - ref.iters) <= 1
    r = b - hmx.matvec(sh.local, res.x.cpu().numpy())
    assert np.linalg.norm(r) <= 1e-4 * np.linalg.norm(b) * 1.01
