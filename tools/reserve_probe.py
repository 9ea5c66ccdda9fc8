"""First / repeated assembly times in one process with and without the context's reserved region.

    python tools/reserve_probe.py T65k [1|0]     (0 = no reserved region)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200 import _lib  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "T65k"
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
w = WORKLOADS[tag]
cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
ct = hmx.build_cluster_tree(cloud, w.n_leaf)
bt = hmx.build_block_tree(ct, ct, w.eta)
t0 = time.perf_counter()
_lib.context(0)
t1 = time.perf_counter()
tw = _lib.reserve(0, 0.0) if frac > 0 else 0.0
print(f"context {t1 - t0:.3f} s, reserve {tw:.3f} s", flush=True)
for r in range(3):
    t0 = time.perf_counter()
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    st = H.stats()
    print(f"{tag} rep {r}: device {st['t_total_ms']:.1f} ms, wall {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del H
