"""Analysis harness around the hot path: the convergence theory of the
paper evaluated per configuration, to validate the alpha each config uses.

TEST / ANALYSIS INFRASTRUCTURE, like the rest of oracle/: only tests/, tools and bench.py's
CPU legs may import it; the product package never does.

* Thm 2.1 / 3.1: the fixed-point contraction factor
  psi_max = |alpha| e^{lambda_max T} / (1 - |alpha| e^{lambda_max T}) and the exact per-mode
  residual history r^k_J = (-psi_J)^k r^0_J (psi_J = alpha E_J^{Nt} / (1 - alpha E_J^{Nt})),
  which predicts the fixed-point iteration count of a linear problem exactly;
* Thm 3.3 / Lemma 3.4 / Thm 3.14: GMRES terminates in at most
  N_x + 1 iterations; Elman bound (4 alpha (1 - alpha))^{k/2} when alpha < 2/(3 + sqrt(Nt))
  (the constant as in the proofs, reading R12);
* the alpha min-max problem (minmax): the objective
  max_omega |alpha e^{-(a|omega|^2 + c) T} / (1 - alpha e^{-(a|omega|^2 + c) T})| over
  |omega_i| <= pi/h, evaluated on a grid; it is increasing in alpha (its max sits at
  omega = 0 for a > 0, c >= 0), so the min over (0, 1) has no interior minimiser (reading
  R19): alpha is then bounded below only by the round-off of Gamma_alpha,
  eps * cond(Gamma_alpha) = eps * alpha^{-(Nt-1)/Nt} (reported alongside).

    python -m oracle.analysis            # one JSON line per config of synth.CONFIGS
"""
from __future__ import annotations

import json
import math

import numpy as np

from . import Spec, apply_A, axis_eigs, dst, spec as _spec

EPS = float(np.finfo(np.float64).eps)


def lambda_max(s: Spec) -> float:
    """Largest real part of sigma(L_h): a dim lambda_1 - c (lambda_1 the smallest-magnitude
    Dirichlet eigenvalue, reading R1; the real part for complex a, c)."""
    return s.a * s.dim * float(axis_eigs(s.n).max()) - s.c


def psi_max(s: Spec) -> float:
    """Thm 2.1: per-iteration error contraction bound; for the BDF2
    system (scheme 3) Thm 4.1's rho <= alpha / (1 - alpha)."""
    if s.scheme == 3:
        return s.alpha / (1.0 - s.alpha)
    e = abs(s.alpha) * math.exp(lambda_max(s) * s.T)
    return e / (1.0 - e)


def fp_iterations_bound(s: Spec, tol: float) -> int:
    """Smallest k with psi_max^k < tol (an upper bound on the fixed-point count)."""
    p = psi_max(s)
    return 1 if p <= 0.0 else max(1, math.ceil(math.log(tol) / math.log(p) - 1e-12))


def fp_history_exact(s: Spec, u0: np.ndarray, kmax: int = 60) -> np.ndarray:
    """Exact relative residual history of Richardson (3.2) for a LINEAR real problem from
    U^0 = 0: r^0 = (A u0, 0, ..., 0) and r^k = (-psi_J)^k r^0 per DST mode J (the derivation
    of Thm 2.1 with the residual in the first time slot), so
    ||r^k|| / ||r^0|| = sqrt(sum_J psi_J^{2k} c_J^2) / ||c||, c = V A u0."""
    assert not s.q and s.scheme in (0, 1), "linear first-order problems only"
    c = dst(s, apply_A(s, u0)).reshape(-1)
    lam = axis_eigs(s.n)
    mu = s.a * _mode_sum(lam, s.dim) - s.c
    eT = np.exp(mu * s.T)
    psi = np.abs(s.alpha * eT / (1.0 - s.alpha * eT))
    r0 = np.sqrt((c * c).sum())
    return np.array([np.sqrt(((psi ** k * c) ** 2).sum()) / r0 for k in range(kmax + 1)])


def fp_iterations_exact(s: Spec, u0: np.ndarray, tol: float, kmax: int = 60) -> int:
    """The fixed-point iteration count the stop rule of reading R8 gives: the first k with
    rho_k < tol."""
    h = fp_history_exact(s, u0, kmax)
    below = np.nonzero(h < tol)[0]
    return int(below[0]) if len(below) else kmax


def _mode_sum(lam: np.ndarray, dim: int) -> np.ndarray:
    """sum over axes of lambda_{j_axis}, modes in [z][y][x] order (x fastest), flattened."""
    out = lam.copy()
    for _ in range(1, dim):
        out = np.add.outer(lam, out).reshape(-1)
    return out


def elman_alpha_limit(nt: int) -> float:
    """alpha < 2/(3 + sqrt(Nt)) for the Elman bound (Lemmas 3.9-3.13 as proved, R12)."""
    return 2.0 / (3.0 + math.sqrt(nt))


def gmres_iterations_bound(s: Spec, tol: float) -> int:
    """min(N_x + 1 (Thm 3.3), the Elman bound's k (Thm 3.14) when it applies)."""
    n_bound = s.N + 1
    if s.alpha < elman_alpha_limit(s.nt):
        rate = math.sqrt(4.0 * s.alpha * (1.0 - s.alpha))
        k = math.ceil(math.log(tol) / math.log(rate) - 1e-12)
        return min(n_bound, max(1, k))
    return n_bound


def minmax_objective(alpha: float, s: Spec, n_omega: int = 257) -> float:
    """The objective of (minmax) on a grid of |omega_i| <= pi/h in dim
    dimensions ("the formula in higher dimensions is straightforward": |omega|^2 summed)."""
    h = 1.0 / (s.n + 1)
    w = np.linspace(-math.pi / h, math.pi / h, n_omega)
    w2 = w * w
    acc = w2
    for _ in range(1, s.dim):
        acc = np.add.outer(w2, acc).reshape(-1)
    e = alpha * np.exp(-(s.a * acc + s.c) * s.T)
    return float(np.abs(-e / (1.0 - e)).max())


def alpha_minmax(s: Spec, lo: float = 1e-12, hi: float = 1.0 - 1e-9, iters: int = 200) -> float:
    """Golden-section search of the (minmax) objective over log alpha in [lo, hi]; the
    objective is increasing (R19), so this returns ~lo: there is no interior optimum."""
    g = (math.sqrt(5.0) - 1.0) / 2.0
    a, b = math.log(lo), math.log(hi)
    f = lambda x: minmax_objective(math.exp(x), s)  # noqa: E731
    c, d = b - g * (b - a), a + g * (b - a)
    fc, fd = f(c), f(d)
    for _ in range(iters):
        if fc <= fd:
            b, d, fd = d, c, fc
            c = b - g * (b - a)
            fc = f(c)
        else:
            a, c, fc = c, d, fd
            d = a + g * (b - a)
            fd = f(d)
    return math.exp(0.5 * (a + b))


def roundoff_floor(s: Spec) -> float:
    """eps * cond(Gamma_alpha) = eps alpha^{-(Nt-1)/Nt}: the relative accuracy one
    preconditioner apply can reach (the floor small alpha runs into)."""
    return EPS * s.alpha ** (-(s.nt - 1) / s.nt)


def report(cfg) -> dict:
    s = _spec(cfg)
    out = {
        "config": cfg.name, "alpha": s.alpha, "nt": s.nt, "T": s.T,
        "lambda_max": lambda_max(s), "psi_max": psi_max(s),
        "fp_iterations_bound": fp_iterations_bound(s, cfg.tol),
        "elman_alpha_limit": elman_alpha_limit(s.nt),
        "elman_applies": s.alpha < elman_alpha_limit(s.nt),
        "gmres_iterations_bound": gmres_iterations_bound(s, cfg.tol),
        "minmax_objective_at_alpha": minmax_objective(s.alpha, s),
        "minmax_objective_increasing": minmax_objective(s.alpha / 2, s) < minmax_objective(s.alpha, s)
        < minmax_objective(min(2 * s.alpha, 0.5), s),
        "roundoff_floor": roundoff_floor(s),
        "tol": cfg.tol,
    }
    return out


def main():
    import synth

    for cfg in synth.CONFIGS.values():
        print(json.dumps(report(cfg)))


if __name__ == "__main__":
    main()
