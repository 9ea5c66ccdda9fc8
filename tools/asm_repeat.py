"""Assemble one config several times in one process (timing stability probe)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "U32k"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = WORKLOADS[tag]
cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
ct = hmx.build_cluster_tree(cloud, w.n_leaf)
bt = hmx.build_block_tree(ct, ct, w.eta)
tot = []
for r in range(reps):
    t0 = time.perf_counter()
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    st = H.stats()
    print(f"{tag} rep {r}: total {st['t_total_ms']:.1f} ms  aca {st['t_aca_ms']:.1f}  recompress "
          f"{st['t_recompress_ms']:.1f}  form {st['t_form_ms']:.1f}  wall {1e3 * (time.perf_counter() - t0):.1f}",
          flush=True)
    del H
    if r > 0:
        tot.append(st["t_total_ms"])
if tot:
    import statistics
    print(f"{tag} summary over reps 1..{reps - 1}: min {min(tot):.1f} ms  median {statistics.median(tot):.1f} ms")
