"""bench.py's T65k conditions: U32k assembled twice and released (cache handed
back), then T65k assembled `reps` times; prints each assembly's device time.

    HMX_VERBOSE=1 python tools/first_call_probe.py 3
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200 import _lib  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2


def asm(tag):
    w = WORKLOADS[tag]
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    t0 = time.perf_counter()
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    st = H.stats()
    print(f"{tag}: total {st['t_total_ms']:.1f} ms aca {st['t_aca_ms']:.1f} form {st['t_form_ms']:.1f} "
          f"wall {1e3 * (time.perf_counter() - t0):.1f}", file=sys.stderr, flush=True)
    return H


for _ in range(2):
    H = asm("U32k")
    del H
_lib.lib().hmx_ctx_release_cache(_lib.context(0))
for _ in range(reps):
    H = asm("T65k")
    del H
