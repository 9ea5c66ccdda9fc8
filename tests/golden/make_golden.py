"""Generate the golden fixtures from the REFERENCE itself (run in the build
container, where /root/reference is mounted; the fixtures are committed and
travel to the GPU box, the reference does not).

    python tests/golden/make_golden.py

* geometry_<case>.npz : permutation + leaf table (kind, r0, r1, c0, c1) of the
  reference ``build_cluster_tree`` / ``build_block_tree`` / ``leaves()``
  (geometry.py:182-295) for a few clouds;
* config_partitions.json : SHA-256 of the reference permutation and leaf table
  at every BASELINE.json configuration (H4k, U8k, U32k, U131k, T65k), with the
  leaf counts (the full tables are too large to commit);
* kernels.npz : outputs of the reference kernel core
  (_kernelcore_np.py:37-130) on seeded points, with and without coincident
  pairs / self shift.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hmatx import _kernelcore_np as R  # noqa: E402
from hmatx import geometry as G  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

GEOMETRY_CASES = {
    # name: (kind, n, n_leaf, eta)
    "sphere1000_l16_e3": ("sphere", 1000, 16, 3.0),
    "sphere4096_l32_e3": ("sphere", 4096, 32, 3.0),   # the H4k partition
    "plate30_l8_e05": ("plate", 30, 8, 0.5),
    "plate20_l1_e3": ("plate", 20, 1, 3.0),
}


def leaf_table(bt):
    return np.array([(1 if isinstance(l, G.AdmissibleLeaf) else 0, l.row.start, l.row.stop, l.col.start,
                      l.col.stop) for l in bt.leaves()], dtype=np.int64)


def config_partitions():
    """Reference tree + partition at the five BASELINE sizes (geometry.py:182-295)."""
    import hashlib
    import json

    cases = {"H4k": (4096, 32), "U8k": (8192, 32), "U32k": (32768, 32), "U131k": (131072, 64),
             "T65k": (65536, 32)}
    out = {}
    for tag, (n, leaf) in cases.items():
        cl = G.make_geometry("sphere", n, 1.0)
        ct = G.build_cluster_tree(cl, leaf)
        bt = G.build_block_tree(ct, ct, 3.0)
        perm = np.ascontiguousarray(ct.permutation.astype("<i8"))
        tab = np.ascontiguousarray(leaf_table(bt).astype("<i8"))
        out[tag] = {"n_points": n, "n_leaf": leaf, "eta": 3.0,
                    "perm_sha256": hashlib.sha256(perm.tobytes()).hexdigest(),
                    "table_sha256": hashlib.sha256(tab.tobytes()).hexdigest(),
                    "n_leaves": int(len(tab)), "n_admissible": int((tab[:, 0] == 1).sum()),
                    "depth": int(ct.depth), "c_sp": int(G.sparsity_pattern(bt))}
        print(tag, out[tag])
    with open(os.path.join(HERE, "config_partitions.json"), "w") as f:
        json.dump(out, f, indent=1)


def main():
    for name, (kind, n, leaf, eta) in GEOMETRY_CASES.items():
        cl = G.make_geometry(kind, n, 1.0)
        ct = G.build_cluster_tree(cl, leaf)
        bt = G.build_block_tree(ct, ct, eta)
        np.savez_compressed(os.path.join(HERE, f"geometry_{name}.npz"), kind=kind, n=n, n_leaf=leaf, eta=eta,
                            perm=ct.permutation.astype(np.int64), table=leaf_table(bt),
                            c_sp=G.sparsity_pattern(bt), depth=ct.depth)
    rng = np.random.default_rng(20260101)
    X = rng.standard_normal((12, 3))
    Y = rng.standard_normal((15, 3))
    Y[4] = X[7]
    NY = rng.standard_normal((15, 3))
    NY /= np.linalg.norm(NY, axis=1)[:, None]
    out = dict(X=X, Y=Y, NY=NY)
    out["H"] = R.scalar_block(11.3, X, Y, self_shift=4096.0)
    out["H_lap"] = R.scalar_block(0.0, X, Y, self_shift=4096.0)
    out["U"] = R.elasto_u_block(9.262, 16.042, 1 / 16.042**2, X, Y, self_shift=8192.0)
    out["U_low"] = R.elasto_u_block(2.0 / np.sqrt(3.0), 2.0, 0.25, X * 0.01, Y * 0.01, self_shift=1.0)
    out["T"] = R.elasto_t_block(26.197, 45.375, 1.0, 1.0, 1 / 45.375**2, X, Y, NY, self_shift=65536.0)
    out["H_none_is_none"] = np.array(R.scalar_block(11.3, X, Y) is None)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    config_partitions()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
