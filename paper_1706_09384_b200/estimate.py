"""A-posteriori residual estimator (PAPER Eq.
(est_direct)): ``estimate(h, spec, cloud, b, x0, with_dense_oracle) ->
EstimatorReport``.

* delta = ||b - A_H x0||_2 from one device H-matvec;
* delta_{H,F} = ||A - A_H||_F by blockwise regeneration of every admissible
  leaf on the device (``hmx_block_errors``; dense leaves contribute 0);
* bound = (delta + delta_{H,F} ||x0||_2) / ||b||_2;
* true_residual = ||b - A x0||_2 / ||b||_2 from the dense kernel matrix, only
  when ``with_dense_oracle`` (row blocks evaluated by ``hmx_eval_block``).
"""

import math
from dataclasses import dataclass

import numpy as np

from .hmatrix import block_errors, matvec
from .kernels import assemble_dense

# dense-oracle limit: (d N)^2 complex entries evaluated row block by row block
DENSE_ORACLE_MAX_DOFS = 40000


@dataclass(frozen=True)
class EstimatorReport:
    """SPEC.md:474-477."""

    delta: float
    delta_h_frob: float
    norm_b: float
    norm_x0: float
    bound: float
    true_residual: float | None = None
    norm_a_frob: float | None = None


def delta_h_frob(h, spec, cloud):
    """(delta_{H,F}, ||A||_F, per-leaf err2, per-leaf norm2)."""
    err2, norm2 = block_errors(h, spec, cloud)
    return math.sqrt(float(err2.sum())), math.sqrt(float(norm2.sum())), err2, norm2


def _dense_residual(h, spec, cloud, b, x0, rows_per_block=2048):
    from .geometry import PointCloud

    d = spec.d
    n = d * cloud.size
    if n > DENSE_ORACLE_MAX_DOFS:
        raise ValueError(f"dense oracle limited to {DENSE_ORACLE_MAX_DOFS} dofs")
    shift = h.self_shift if h.self_shift is not None else float(cloud.size)
    r = np.array(b, dtype=np.complex128, copy=True)
    for p0 in range(0, cloud.size, rows_per_block):
        p1 = min(cloud.size, p0 + rows_per_block)
        rows = PointCloud(points=cloud.points[p0:p1], normals=None if cloud.normals is None
                          else cloud.normals[p0:p1])
        blk = assemble_dense(spec, rows, cloud, self_shift=shift)
        r[d * p0:d * p1] -= blk @ x0
    return float(np.linalg.norm(r))


def estimate(h, spec, cloud, b, x0, with_dense_oracle=False):
    """SPEC.md:507-515."""
    b = np.ascontiguousarray(b, dtype=np.complex128)
    x0 = np.ascontiguousarray(x0, dtype=np.complex128)
    nb = float(np.linalg.norm(b))
    nx = float(np.linalg.norm(x0))
    delta = float(np.linalg.norm(b - matvec(h, x0)))
    dhf, na, _, _ = delta_h_frob(h, spec, cloud)
    bound = (delta + dhf * nx) / nb if nb > 0 else (0.0 if delta == 0.0 and dhf * nx == 0.0 else math.inf)
    tr = None
    if with_dense_oracle:
        tr = _dense_residual(h, spec, cloud, b, x0) / nb if nb > 0 else 0.0
    return EstimatorReport(delta=delta, delta_h_frob=dhf, norm_b=nb, norm_x0=nx, bound=bound, true_residual=tr,
                           norm_a_frob=na)
