"""Exhaustive per-leaf compression error of one config; dumps the worst leaves.

    python tools/worst_leaves.py U131k [out.npz]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests._problems import Problem  # noqa: E402
from paper_1706_09384_b200.hmatrix import block_errors  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "U131k"
out = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/worst_{tag}.npz"
pb = Problem(tag)
H, _ = pb.device_h()
t0 = time.perf_counter()
err2, norm2 = block_errors(H, pb.spec, pb.cloud)
t1 = time.perf_counter()
info = H.block_info()
adm = np.flatnonzero(pb.table[:, 0] == 1)
ratio = np.sqrt(err2[adm] / norm2[adm]) / pb.w.eps
order = np.argsort(-ratio)
print(f"{tag}: block_errors {1e3 * (t1 - t0):.1f} ms; {len(adm)} admissible; worst {ratio[order[0]]:.3f} eps; "
      f">1 eps {np.mean(ratio > 1) * 100:.2f}%; >3 eps {np.sum(ratio > 3)}")
for q in order[:12]:
    b = adm[q]
    _, r0, r1, c0, c1 = pb.table[b][:5]
    print(f"  leaf {b}: m {r1 - r0} n {c1 - c0} ratio {ratio[q]:.3f} steps {info['steps'][b]} "
          f"rank {info['rank_before'][b]} -> {info['rank_after'][b]} flags {info['flags'][b]}")
np.savez(out, adm=adm, ratio=ratio, steps=info["steps"], rank_before=info["rank_before"],
         rank_after=info["rank_after"], flags=info["flags"], table=pb.table)
