"""Small end-to-end run for compute-sanitizer (memcheck / racecheck)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from tests._problems import Problem  # noqa: E402

for tag, n in [("H4k", 600), ("U8k", 400), ("T65k", 300)]:
    pb = Problem(tag, n)
    H, rep = pb.device_h()
    x = pb.rhs(0)
    y = hmx.matvec(H, x)
    res = hmx.solve_gmres(H, x, hmx.GmresConfig(tol=1e-4, restart=50))
    print(tag, n, rep.max_rank_after, res.iters, float(np.linalg.norm(y)))
