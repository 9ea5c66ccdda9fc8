"""ncu target for the per-pair FP64 flop count: one eval_block launch per
kernel kind over exactly 512 x 512 point pairs (no coincident points)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402

rng = np.random.default_rng(0)
X = rng.standard_normal((512, 3))
Y = rng.standard_normal((512, 3)) + 10.0
NY = rng.standard_normal((512, 3))
NY /= np.linalg.norm(NY, axis=1)[:, None]
hmx.scalar_block(11.3, X, Y)
hmx.elasto_u_block(18.5, 32.1, 1 / 32.1**2, X, Y)
hmx.elasto_t_block(26.2, 45.4, 1.0, 1.0, 1 / 45.4**2, X, Y, NY)
print("pairs per launch", 512 * 512)
