"""Kernel parameters and the kernel-core seam, on the GPU.

Types follow SPEC.md:156-175 (``Material``, ``Wavenumbers``, ``KernelSpec``);
the three block functions keep the reference kernel-core signatures
(``/root/reference/pkg/src/hmatx/_kernelcore_np.py:37, 89, 105``) and return
convention (new C-contiguous complex128 array, or ``None`` when an exact r == 0
pair exists and ``self_shift`` is None), computed by ``hmx_eval_block``
(``csrc/dense.cu``) on the device.
"""

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import SingularEvaluationError

HELMHOLTZ, ELASTO_U, ELASTO_T = 0, 1, 2


@dataclass(frozen=True)
class Wavenumbers:
    kp: float
    ks: float


@dataclass(frozen=True)
class Material:
    """rho, mu, Poisson ratio nu, circular frequency omega."""

    rho: float
    mu: float
    nu: float
    omega: float

    def __post_init__(self):
        if not (self.rho > 0 and self.mu > 0 and self.omega > 0):
            raise ValueError("rho, mu, omega must be positive")
        if not (-1.0 < self.nu < 0.5):
            raise ValueError("nu must lie in (-1, 0.5)")

    @property
    def lam(self):
        return 2.0 * self.mu * self.nu / (1.0 - 2.0 * self.nu)

    @property
    def wavenumbers(self):
        """kp^2 = rho w^2/(lambda + 2 mu), ks^2 = rho w^2/mu."""
        w2 = self.rho * self.omega**2
        return Wavenumbers(kp=math.sqrt(w2 / (self.lam + 2.0 * self.mu)), ks=math.sqrt(w2 / self.mu))

    @property
    def scale(self):
        return 1.0 / (self.rho * self.omega**2)

    @classmethod
    def from_lame(cls, rho, mu, lam, omega):
        return cls(rho=rho, mu=mu, nu=lam / (2.0 * (lam + mu)), omega=omega)


@dataclass(frozen=True)
class KernelSpec:
    """variant in {"laplace", "helmholtz", "elasto_u", "elasto_t"}."""

    variant: str
    kappa: float = 0.0
    material: Material | None = None

    @classmethod
    def laplace(cls):
        return cls("laplace", 0.0)

    @classmethod
    def helmholtz(cls, kappa):
        return cls("helmholtz", float(kappa))

    @classmethod
    def elasto_u(cls, material):
        return cls("elasto_u", material=material)

    @classmethod
    def elasto_t(cls, material):
        return cls("elasto_t", material=material)

    @property
    def d(self):
        return 1 if self.variant in ("laplace", "helmholtz") else 3

    @property
    def kind(self):
        return {"laplace": HELMHOLTZ, "helmholtz": HELMHOLTZ, "elasto_u": ELASTO_U,
                "elasto_t": ELASTO_T}[self.variant]

    def c_kernel(self):
        k = _lib.HmxKernel()
        k.kind = self.kind
        k.kappa = self.kappa
        if self.material is not None:
            w = self.material.wavenumbers
            k.kp, k.ks = w.kp, w.ks
            k.lam, k.mu = self.material.lam, self.material.mu
            k.scale = self.material.scale
        return k


def _eval(kern, X, Y, NY, self_shift, device=0):
    X = _lib.f64c(X)
    Y = _lib.f64c(Y)
    if X.ndim != 2 or X.shape[1] != 3 or Y.ndim != 2 or Y.shape[1] != 3:
        raise ValueError("X, Y must have shape (., 3)")
    d = 1 if kern.kind == HELMHOLTZ else 3
    out = np.empty((d * X.shape[0], d * Y.shape[0]), dtype=np.complex128)
    nrm = None if NY is None else _lib.f64c(NY, Y.shape)
    st = _lib.lib().hmx_eval_block(
        _lib.context(device), C.byref(kern), _lib.ptr(X), X.shape[0], _lib.ptr(Y), Y.shape[0],
        _lib.ptr(nrm), 0 if self_shift is None else 1, 0.0 if self_shift is None else float(self_shift),
        _lib.ptr(out))
    if st == 4:  # HMX_ESINGULAR -> reference returns None
        return None
    _lib.check(st, "hmx_eval_block")
    return out


def scalar_block(kappa, X, Y, self_shift=None):
    """(m, n) e^{i kappa r}/(4 pi r) (``_kernelcore_np.py:37-49``)."""
    k = _lib.HmxKernel()
    k.kind, k.kappa = HELMHOLTZ, float(kappa)
    return _eval(k, X, Y, None, self_shift)


def elasto_u_block(kp, ks, scale, X, Y, self_shift=None):
    """(3m, 3n) displacement tensor (``_kernelcore_np.py:89-102``)."""
    k = _lib.HmxKernel()
    k.kind, k.kp, k.ks, k.scale = ELASTO_U, float(kp), float(ks), float(scale)
    return _eval(k, X, Y, None, self_shift)


def elasto_t_block(kp, ks, lam, mu, scale, X, Y, NY, self_shift=None):
    """(3m, 3n) traction tensor, column normals NY (``_kernelcore_np.py:105-130``)."""
    k = _lib.HmxKernel()
    k.kind, k.kp, k.ks, k.lam, k.mu, k.scale = ELASTO_T, float(kp), float(ks), float(lam), float(mu), float(scale)
    return _eval(k, X, Y, NY, self_shift)


def _single(spec, x, y, n_y=None):
    out = _eval(spec.c_kernel(), np.reshape(x, (1, 3)), np.reshape(y, (1, 3)),
                None if n_y is None else np.reshape(n_y, (1, 3)), None)
    if out is None:
        raise SingularEvaluationError("singular evaluation")
    return out


def eval_scalar(spec, x, y):
    """SPEC.md:178-186."""
    return complex(_single(spec, x, y)[0, 0])


def eval_elasto_u(m, x, y):
    """SPEC.md:188-196."""
    return _single(KernelSpec.elasto_u(m), x, y)


def eval_elasto_t(m, x, y, n_y):
    """SPEC.md:198-206."""
    return _single(KernelSpec.elasto_t(m), x, y, n_y)


def assemble_dense(spec, rows, cols, self_shift=None):
    """Dense (d N_r) x (d N_c) kernel matrix of two clouds;
    coincident points need ``self_shift`` or raise."""
    NY = cols.normals if spec.variant == "elasto_t" else None
    if spec.variant == "elasto_t" and NY is None:
        raise ValueError("ElastoT requires column normals")
    out = _eval(spec.c_kernel(), rows.points, cols.points, NY, self_shift)
    if out is None:
        raise SingularEvaluationError("coincident points without a self-block rule")
    return out
