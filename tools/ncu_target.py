"""Small ncu target: assemble one config, run a few H-matvecs.

    python tools/ncu_target.py U32k [n_matvec]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "U32k"
nmv = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = WORKLOADS[tag]
cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
ct = hmx.build_cluster_tree(cloud, w.n_leaf)
bt = hmx.build_block_tree(ct, ct, w.eta)
H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
rng = np.random.default_rng(0)
n = w.d * w.n_points
x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
for _ in range(nmv):
    y = hmx.matvec(H, x)
print(tag, "ok", rep.max_rank_after, float(np.linalg.norm(y)))
