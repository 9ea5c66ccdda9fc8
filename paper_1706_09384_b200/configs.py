"""The BASELINE.json workloads (synthetic Fibonacci-sphere stand-ins).

Parameters follow BASELINE.md section 4 / SURVEY.md 8(d):

* rho = mu = lambda = 1 (nu = 0.25) for every elastodynamic config;
* "10 points per S-wavelength" = kappa_s = 2 pi / (10 h), h = sqrt(4 pi / N)
  (BASELINE.json writes "kappa_s about 45" for N_c = 32,768; that value is the
  N_c = 65,536 one -- we follow the stated rule, kappa_s = 32.085);
* omega = kappa_s sqrt(mu / rho), kappa_p = kappa_s / sqrt(3), scale = 1/(rho omega^2);
* eta = 3 (strict <, geometry.py:113), eps_ACA = 1e-4, self shift zeta = N_c
  (SPEC.md:226), RHS seed 0 (BASELINE.json names none).
"""

import math
from dataclasses import dataclass, field

SEED = 0


def ks_ten_per_wavelength(n_points):
    h = math.sqrt(4.0 * math.pi / n_points)
    return 2.0 * math.pi / (10.0 * h)


@dataclass(frozen=True)
class Workload:
    tag: str
    kind: str            # "H" | "U" | "T"
    n_points: int
    n_leaf: int
    eta: float = 3.0
    eps: float = 1e-4
    kappa: float = 0.0   # Helmholtz wavenumber (kind "H")
    ks: float = 0.0      # S wavenumber (kinds "U"/"T")
    rho: float = 1.0
    mu: float = 1.0
    lam: float = 1.0
    runs: tuple = field(default=("assemble", "matvec", "gmres"))

    @property
    def d(self):
        return 1 if self.kind == "H" else 3

    @property
    def omega(self):
        return self.ks * math.sqrt(self.mu / self.rho)

    @property
    def kp(self):
        # kp^2 = rho omega^2 / (lambda + 2 mu)
        return math.sqrt(self.rho * self.omega**2 / (self.lam + 2.0 * self.mu))

    @property
    def scale(self):
        return 1.0 / (self.rho * self.omega**2)

    def params(self):
        """Kernel parameter dict (oracle convention)."""
        if self.kind == "H":
            return {"kappa": self.kappa}
        return {"kp": self.kp, "ks": self.ks, "lam": self.lam, "mu": self.mu,
                "scale": self.scale}

    def spec(self):
        """The hmatx KernelSpec of this workload (Material from rho, mu, lambda, omega)."""
        from .kernels import KernelSpec, Material

        if self.kind == "H":
            return KernelSpec.helmholtz(self.kappa)
        mat = Material.from_lame(self.rho, self.mu, self.lam, self.omega)
        return KernelSpec.elasto_u(mat) if self.kind == "U" else KernelSpec.elasto_t(mat)

    def with_points(self, n_points, rescale_ks=True):
        """Same physics at another size (kappa_s rescaled for 10 pts/lambda_s
        when the original was on that rule)."""
        ks = self.ks
        if rescale_ks and self.kind != "H" and self.tag != "U131k":
            ks = ks_ten_per_wavelength(n_points)
        return Workload(tag=f"{self.tag}@{n_points}", kind=self.kind, n_points=n_points,
                        n_leaf=self.n_leaf, eta=self.eta, eps=self.eps, kappa=self.kappa,
                        ks=ks, rho=self.rho, mu=self.mu, lam=self.lam, runs=self.runs)


WORKLOADS = {
    "H4k": Workload("H4k", "H", 4096, 32, kappa=11.3),
    "U8k": Workload("U8k", "U", 8192, 32, ks=ks_ten_per_wavelength(8192)),
    "U32k": Workload("U32k", "U", 32768, 32, ks=ks_ten_per_wavelength(32768),
                     runs=("assemble", "matvec")),
    # the other reading of config 3's "kappa_s about 45" (the N_c = 65,536 ten-points rule value)
    "U32k45": Workload("U32k45", "U", 32768, 32, ks=ks_ten_per_wavelength(65536), runs=("assemble", "matvec")),
    "U131k": Workload("U131k", "U", 131072, 64, ks=2.0, runs=("assemble", "matvec")),
    "T65k": Workload("T65k", "T", 65536, 32, ks=ks_ten_per_wavelength(65536),
                     runs=("assemble", "gmres")),
}
