"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no spectra, no DST, no exponentials, no
DFT, no time stepping): only the problem parameters of BASELINE.json's five configs and
seeded initial data / random space-time vectors (recipe: DESIGN.md "Inputs").  Both the
oracle side and the CUDA side receive the same float64 arrays from here.

The paper's workloads are analytic initial conditions on (0,1)^d Dirichlet grids
(PAPER.md:917, :1028, :1253); BASELINE.json:7-11 scales them up.  Sine modes are
evaluated at the grid points x_i = i h, h = 1/(n+1), with the angle index reduced
exactly, sin(pi ((k i) mod 2(n+1)) / (n+1)), so each mode is sampled without argument
rounding drift.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    n: int
    a: float
    c: float
    T: float
    nt: int
    alpha: float
    scheme: int = 0  # 0: exponential Euler / ETD1, 1: ETD2
    q: tuple = field(default_factory=tuple)  # N(u) = sum_p q[p] u^p
    solvers: tuple = ("fixed_point",)
    tol: float = 1e-12  # reading R9
    seed: int = 0
    a_im: float = 0.0  # imaginary parts of a, c: complex state (NEXT-4, Schroedinger)
    c_im: float = 0.0

    @property
    def is_complex(self) -> bool:
        return self.a_im != 0.0 or self.c_im != 0.0

    @property
    def dt(self) -> float:
        return self.T / self.nt

    @property
    def N(self) -> int:
        return self.n ** self.dim

    @property
    def nst(self) -> int:
        return self.N * self.nt

    @property
    def shape(self) -> tuple:
        return (self.n,) * self.dim

    def scaled(self, n: int, nt: int, name: str | None = None) -> "Config":
        """Same problem family on a smaller grid (same T, a, c, alpha, N(u))."""
        return replace(self, n=n, nt=nt, name=name or f"{self.name}@n{n}nt{nt}")


CUBIC = (0.0, 0.0, 0.0, -1.0)  # N(u) = -u^3 (BASELINE.json:9, :11)

CONFIGS = {
    # BASELINE.json:7 -- 1D linear heat u_t = u_xx - u
    "c1": Config("c1", 1, 63, 1.0, 1.0, 1.0, 32, 1e-2, solvers=("fixed_point", "gmres"), seed=1),
    # BASELINE.json:8 -- 2D linear u_t = 0.5 Lap u - u
    "c2": Config("c2", 2, 255, 0.5, 1.0, 1.0, 64, 1e-3, solvers=("fixed_point", "gmres"), seed=2),
    # BASELINE.json:9 -- 2D u_t = Lap u - u - u^3, exponential Euler (ETD1) Picard
    "c3": Config("c3", 2, 511, 1.0, 1.0, 0.5, 128, 1e-3, scheme=0, q=CUBIC, seed=3),
    # BASELINE.json:10 -- 3D linear u_t = Lap u - u, GMRES (tol 1e-10: reading R9)
    "c4": Config("c4", 3, 255, 1.0, 1.0, 1.0, 64, 1e-4, solvers=("gmres", "fixed_point"), tol=1e-10, seed=4),
    # BASELINE.json:11 -- 2D u_t = 0.1 Lap u - 0.5 u - u^3, ETD2 Picard
    "c5": Config("c5", 2, 2047, 0.1, 0.5, 1.0, 256, 1e-3, scheme=1, q=CUBIC, seed=5),
    # NEXT-1: the paper's own nonlinear iteration -- IF scheme (6.1) solved by
    # the IMEX-type Exp-ParaDiag iteration (7.2)/(7.3) -- on the
    # c3 and c5 problems (not BASELINE.json configs)
    # NEXT-2: the exponential BDF2 all-at-once system (4.1)-(4.5)
    # on the c1 / c2 problems (linear; nt unknowns u_2..u_{nt+1})
    "c1bdf2": Config("c1bdf2", 1, 63, 1.0, 1.0, 1.0, 32, 1e-2, scheme=3, solvers=("fixed_point", "gmres"), seed=1),
    "c2bdf2": Config("c2bdf2", 2, 255, 0.5, 1.0, 1.0, 64, 1e-3, scheme=3, solvers=("fixed_point", "gmres"), seed=2),
    "c3if": Config("c3if", 2, 511, 1.0, 1.0, 0.5, 128, 1e-3, scheme=2, q=CUBIC, seed=3),
    "c5if": Config("c5if", 2, 2047, 0.1, 0.5, 1.0, 256, 1e-3, scheme=2, q=CUBIC, seed=5),
    # NEXT-4: complex coefficients, the paper's Schroedinger tests.
    # c6se: 1D, a = i, c = 2i, u0 = sin(pi x), h = 1/128, dt = 0.01
    "c6se": Config("c6se", 1, 127, 0.0, 0.0, 2.56, 256, 1e-3, solvers=("gmres", "fixed_point"), a_im=1.0,
                   c_im=2.0, seed=6),
    # c7se: 2D, a = i, c = 200i, Gaussian wave packet u0 (the paper
    # runs it with BDF2 on h = 1/40 -- here exponential Euler on a 1023^2 grid)
    "c7se": Config("c7se", 2, 1023, 0.0, 0.0, 0.64, 128, 1e-3, solvers=("fixed_point", "gmres"), a_im=1.0,
                   c_im=200.0, seed=7),
    # c7bdf2: the same packet with the paper's own setup for it -- exponential BDF2 (scheme 3),
    # dt = 0.05, alpha_opt = 0.0001953125, GMRES; h = 1/1024
    "c7bdf2": Config("c7bdf2", 2, 1023, 0.0, 0.0, 6.4, 128, 0.0001953125, scheme=3,
                     solvers=("gmres", "fixed_point"), tol=1e-10, a_im=1.0, c_im=200.0, seed=7),
}


def sine_table(n: int, kmax: int) -> np.ndarray:
    """S[k-1, i-1] = sin(pi k i/(n+1)) for k = 1..kmax, i = 1..n (mode samples, not a transform)."""
    k = np.arange(1, kmax + 1, dtype=np.int64)[:, None]
    i = np.arange(1, n + 1, dtype=np.int64)[None, :]
    q = (k * i) % (2 * (n + 1))
    return np.sin(np.pi * q / (n + 1))


def _sum_of_modes(n: int, dim: int, ks: np.ndarray, coef: np.ndarray) -> np.ndarray:
    """sum_m coef[m] prod_axis sin(pi k[m,axis] x_axis), array indexed [z][y][x]."""
    kmax = int(ks.max())
    S = sine_table(n, kmax)
    u = np.zeros((n,) * dim)
    for k, c in zip(ks, coef):
        f = S[k[0] - 1]
        if dim >= 2:
            f = np.multiply.outer(S[k[1] - 1], f)
        if dim == 3:
            f = np.multiply.outer(S[k[2] - 1], f)
        u += c * f
    return u


def initial_condition(cfg: Config) -> np.ndarray:
    """u_0 for a config (recipes: DESIGN.md "Inputs")."""
    n, dim = cfg.n, cfg.dim
    if cfg.name.startswith("c1"):
        S = sine_table(n, 3)
        return S[0] + 0.5 * S[2]  # sin(pi x) + 0.5 sin(3 pi x)
    if cfg.name.startswith("c2") or cfg.name.startswith("c4"):
        nmodes = 16 if cfg.name.startswith("c2") else 32
        rng = np.random.default_rng(cfg.seed)
        kmax = min(32, n)
        ks = rng.integers(1, kmax + 1, size=(nmodes, dim))
        coef = rng.standard_normal(nmodes)
        return _sum_of_modes(n, dim, ks, coef)
    if cfg.name.startswith("c3"):
        rng = np.random.default_rng(cfg.seed)
        u = rng.uniform(-0.5, 0.5, size=(n,) * dim)
        w = 2.0 / 3.0
        for _ in range(4):  # damped Jacobi smoothing passes, zero Dirichlet ghosts
            p = np.pad(u, 1)
            nb = p[:-2, 1:-1] + p[2:, 1:-1] + p[1:-1, :-2] + p[1:-1, 2:]
            u = (1.0 - w) * u + w * nb / 4.0
        return u
    if cfg.name.startswith("c6"):
        return sine_table(n, 1)[0].astype(np.complex128)  # sin(pi x)
    if cfg.name.startswith("c7"):
        # exp(-((x-1/2)^2 + (y-1/2)^2) / (2 mu^2)) exp(-5 i (x - 1/2)), mu = 0.05
        x = np.arange(1, n + 1) / (n + 1) - 0.5
        mu = 0.05
        gx = np.exp(-x * x / (2 * mu * mu)) * np.exp(-5j * x)
        gy = np.exp(-x * x / (2 * mu * mu))
        return np.multiply.outer(gy, gx)  # [y][x]
    if cfg.name.startswith("c5"):
        rng = np.random.default_rng(cfg.seed)
        K = min(64, n)
        g = rng.standard_normal((64, 64))[:K, :K]  # [ky-1][kx-1]
        k = np.arange(1, K + 1, dtype=np.float64)
        amp = g / (k[:, None] ** 2 + k[None, :] ** 2)
        S = sine_table(n, K)  # [k-1][i-1]
        return S.T @ amp @ S  # [y][x] = sum_{ky,kx} amp sin(ky pi y) sin(kx pi x)
    raise ValueError(cfg.name)


def random_spacetime(cfg: Config, seed: int | None = None, scale: float = 1.0) -> np.ndarray:
    """Seeded standard-normal space-time vector [nt][n..n] (parity inputs, seeds 100+cfg)."""
    rng = np.random.default_rng(100 + cfg.seed if seed is None else seed)
    if cfg.is_complex:  # complex state: independent N(0,1) real and imaginary parts
        re = rng.standard_normal((cfg.nt,) + cfg.shape)
        return scale * (re + 1j * rng.standard_normal((cfg.nt,) + cfg.shape))
    return scale * rng.standard_normal((cfg.nt,) + cfg.shape)


def random_slice(cfg: Config, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal(cfg.shape)


def sparse_spacetime(cfg: Config, nmodes: int = 8, seed: int = 77):
    """A space-time vector [nt][n..n] that is a sum of nmodes fixed sine modes with seeded
    N(0,1) coefficients per slice (full-size parity input whose DST coefficients are
    nonzero only on those modes).  Returns (U, ks) with ks[m] = (k_x, k_y[, k_z])."""
    rng = np.random.default_rng(seed)
    kmax = min(64, cfg.n)
    ks = rng.integers(1, kmax + 1, size=(nmodes, cfg.dim))
    coef = rng.standard_normal((cfg.nt, nmodes))
    S = sine_table(cfg.n, kmax)
    phi = np.empty((nmodes,) + cfg.shape)
    for m, k in enumerate(ks):
        f = S[k[0] - 1]
        if cfg.dim >= 2:
            f = np.multiply.outer(S[k[1] - 1], f)
        if cfg.dim == 3:
            f = np.multiply.outer(S[k[2] - 1], f)
        phi[m] = f
    U = (coef @ phi.reshape(nmodes, -1)).reshape((cfg.nt,) + cfg.shape)
    return U, ks

