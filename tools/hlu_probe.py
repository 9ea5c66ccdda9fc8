"""Time the device H-LU (hlu + triangular_solve) on a workload at a given size and
report consistency ||L U x - A_H x|| / ||A_H x||, the solve residual and the factor storage.
usage: python tools/hlu_probe.py TAG N [eps_lu ...]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200 import hierarchical_lu as HL  # noqa: E402
from tests._problems import Problem  # noqa: E402

tag, n = sys.argv[1], int(sys.argv[2])
prof = "p" in sys.argv[3:]
epss = [float(e) for e in sys.argv[3:] if e != "p"] or [1e-4]
pb = Problem(tag, n)
H, rep = pb.device_h()
b = pb.rhs(0)
y = hmx.matvec(H, b)
for eps in epss:
    for rep_i in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = HL.hlu(H, eps)
        t1 = time.perf_counter()
        x = HL.triangular_solve(f, b)
        t2 = time.perf_counter()
    cons = np.linalg.norm(HL.lu_matvec(f, b) - y) / np.linalg.norm(y)
    res = np.linalg.norm(hmx.matvec(H, x) - b) / np.linalg.norm(b)
    print(f"{tag}@{n} dofs {pb.d * n} eps_lu {eps:g}: hlu {t1 - t0:.3f} s (copy {f.stats['copy_s']:.3f}, "
          f"factor {f.stats['factor_s']:.3f}), solve {1e3 * (t2 - t1):.1f} ms, consistency {cons:.2e}, "
          f"residual {res:.2e}, truncations {f.stats["n_truncations"]} in {f.stats["n_truncate_calls"]} calls, getrf {f.stats['n_getrf']}, "
          f"max rank {f.stats['max_rank']}, storage {f.storage() * 16 / 1e6:.1f} MB "
          f"(H {rep.n_stored * 16 / 1e6:.1f} MB); truncate calls {f.stats['truncate_s']:.3f} s, "
          f"call K max p50/p90/max {f.stats['truncate_kmax_p50_p90_max']}, dense images {f.stats['dense_image_GB']:.2f} GB", flush=True)
    if prof and eps == epss[-1]:
        import cProfile
        import pstats
        cProfile.run("HL.hlu(H, eps)", "/tmp/hlu.prof")
        pstats.Stats("/tmp/hlu.prof").sort_stats("tottime").print_stats(15)
