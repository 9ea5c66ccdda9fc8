"""Per-leaf flag census of one assembly (QL fallback / regularised counts).

    python tools/asm_flags.py U32k
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

for tag in sys.argv[1:] or ["U32k"]:
    w = WORKLOADS[tag]
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    f = H.block_info()["flags"]
    print(tag, "leaves", len(f), "QL fallback (bit 32)", int(np.sum((f & 32) != 0)), "QL unconverged (64)",
          int(np.sum((f & 64) != 0)), "regularised (16)", int(np.sum((f & 16) != 0)), "max rank", rep.max_rank_after)
    del H
