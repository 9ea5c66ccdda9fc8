"""Reproduce bench.py's T65k time-to-solve conditions: a U32k H-matrix stays
resident while T65k is assembled."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

keep = []
for tag in sys.argv[1:] or ["U32k", "T65k"]:
    w = WORKLOADS[tag]
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    t0 = time.perf_counter()
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    st = H.stats()
    print(f"{tag}: total {st['t_total_ms']:.1f} ms passes {st['aca_passes']} wall {1e3 * (time.perf_counter() - t0):.1f}",
          flush=True)
    keep.append(H)
