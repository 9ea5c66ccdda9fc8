"""Assemble configs on the GPU and dump per-leaf (table, steps, ranks) to
gpurun_out/blocks_<tag>.npz for offline cost modelling."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

for tag in sys.argv[1:]:
    w = WORKLOADS[tag]
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    info = H.block_info()
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez(f"gpurun_out/blocks_{tag}.npz", table=bt.table, **info)
    print(tag, H.stats())
