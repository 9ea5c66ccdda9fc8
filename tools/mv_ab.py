"""A/B the U32k H-matvec of several libhmx builds in one process each.

    HMX_LIB=... python tools/mv_ab.py [K]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200 import _lib  # noqa: E402
from tests._problems import Problem  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
pb = Problem("U32k")
H, _ = pb.device_h()
st = H.stats()
n = pb.d * pb.N
X = torch.randn(n, dtype=torch.complex128, device="cuda")
Y = torch.empty_like(X)
H.use_stream(torch.cuda.current_stream().cuda_stream)
L = _lib.lib()
for _ in range(5):
    L.hmx_matvec(H.handle, C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()), 1)
torch.cuda.synchronize()
L.hmx_profile_begin(H.handle)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    L.hmx_matvec(H.handle, C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()), 1)
e1.record()
torch.cuda.synchronize()
nc = C.c_int64()
ph = np.zeros(4)
L.hmx_profile_end(H.handle, C.byref(nc), _lib.ptr(ph))
ms = e0.elapsed_time(e1) / K
ph /= max(nc.value, 1)
print(f"{os.path.basename(os.environ.get('HMX_LIB', 'default'))}: {ms:.4f} ms/matvec = "
      f"{st['matvec_bytes'] / ms / 1e6:.0f} GB/s; phase1 {ph[1]:.4f} ms ({st['phase1_bytes'] / ph[1] / 1e6:.0f} GB/s) "
      f"phase2 {ph[2]:.4f} ms ({st['phase2_bytes'] / ph[2] / 1e6:.0f} GB/s) y0 {complex(Y[0]):.6e}")
