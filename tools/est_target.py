"""ncu target: assemble one config and run the delta_{H,F} estimator once."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests._problems import Problem  # noqa: E402
from paper_1706_09384_b200.hmatrix import block_errors  # noqa: E402

pb = Problem(sys.argv[1] if len(sys.argv) > 1 else "U32k")
H, _ = pb.device_h()
err2, norm2 = block_errors(H, pb.spec, pb.cloud)
print("ok", float(err2.sum()), float(norm2.sum()))
