"""Iterative solve -- the reference's ``hmatx.solve.solve_gmres``
run device-resident by ``hmx_gmres`` (``csrc/gmres.cu``)."""

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class GmresConfig:
    """tol > 0, restart >= 1."""

    tol: float = 1e-4
    restart: int = 50
    max_iters: int = 1000

    def __post_init__(self):
        if not self.tol > 0:
            raise ValueError("tol must be positive")
        if self.restart < 1:
            raise ValueError("restart must be >= 1")


@dataclass
class GmresResult:
    x: np.ndarray
    iters: int
    history: list
    converged: bool

    def __iter__(self):  # (x, iters, history) unpacking, as SPEC.md:497
        return iter((self.x, self.iters, self.history))


def solve_gmres(h, b, cfg=GmresConfig()):
    """Restarted, unpreconditioned GMRES; returns (x, iters, history) (plus
    ``.converged`` on the result object)."""
    n = h.d * h.n_points
    b = np.ascontiguousarray(b, dtype=np.complex128)
    if b.shape != (n,):
        raise ValueError("dimension mismatch")
    x = np.empty_like(b)
    cap = max(1, int(cfg.max_iters))
    hist = np.zeros(cap, np.float64)
    iters = C.c_int64()
    hlen = C.c_int64()
    conv = C.c_int32()
    _lib.check(_lib.lib().hmx_gmres(h.handle, _lib.ptr(b), _lib.ptr(x), cfg.tol, cfg.restart, cfg.max_iters, 0,
                                    C.byref(iters), _lib.ptr(hist), cap, C.byref(hlen), C.byref(conv)),
               "hmx_gmres")
    return GmresResult(x=x, iters=int(iters.value), history=hist[: min(cap, hlen.value)].tolist(),
                       converged=bool(conv.value))
