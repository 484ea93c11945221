"""Seeded random problems (dimension, grid, Nt, coefficients, alpha, scheme, real or complex)
through the C-ABI against the oracle: one preconditioner apply and one residual each, at
the north_star tolerance (relative max error <= 1e-11)."""
from __future__ import annotations

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

DEV = torch.device("cuda:0")


def draw(seed):
    rng = np.random.default_rng(seed)
    dim = int(rng.integers(1, 4))
    nmax = {1: 11, 2: 7, 3: 4}[dim]  # n + 1 = 2^k, k <= nmax (3-D kept small for the oracle)
    n = 2 ** int(rng.integers(2, nmax + 1)) - 1
    if dim == 3:
        n = min(n, 15)
    nt = 2 ** int(rng.integers(2, 9))
    while n ** dim * nt * nt > 1e8 and nt > 4:  # keep the oracle's O(N Nt^2) DFT to ~1 s
        nt //= 2
    cx = rng.random() < 0.4
    scheme = int(rng.choice([0, 3])) if cx else int(rng.choice([0, 1, 2, 3]))
    q = () if (cx or scheme == 3 or rng.random() < 0.4) else (0.0, 0.5 * rng.standard_normal(), 0.0, -1.0)
    a = float(10 ** rng.uniform(-3, 0))
    c = float(rng.uniform(0, 2))
    a_im = float(rng.uniform(-2, 2)) if cx else 0.0
    c_im = float(rng.uniform(-50, 50)) if cx else 0.0
    T = float(10 ** rng.uniform(-2, 0.5))
    alpha = float(10 ** rng.uniform(-4, -0.5))
    return synth.Config(f"fuzz{seed}", dim, n, a, c, T, nt, alpha, scheme=scheme, q=q, a_im=a_im, c_im=c_im,
                        seed=seed)


def relmax(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


@pytest.mark.parametrize("seed", range(120))
def test_fuzz_precond_and_residual(orc, seed):
    cfg = draw(seed)
    s = orc.spec(cfg)
    plan = Plan(Problem.from_config(cfg))
    dt = torch.complex128 if cfg.is_complex else torch.float64
    R = synth.random_spacetime(cfg)
    S = plan.precond_apply(torch.from_numpy(R).to(DEV, dt)).cpu().numpy()
    want = orc.cplx_precond(s, R) if cfg.is_complex else orc.precond(s, R)[0]
    assert relmax(S, want) < 1e-11, cfg  # north_star's tolerance, for every draw
    u0 = synth.random_slice(cfg, seed + 1000)
    if cfg.is_complex:
        u0 = u0 + 1j * synth.random_slice(cfg, seed + 2000)
    U = synth.random_spacetime(cfg, seed=seed + 3000, scale=0.3)
    Rg, rn2 = plan.residual(torch.from_numpy(np.asarray(u0)).to(DEV, dt), torch.from_numpy(U).to(DEV, dt), norm=True)
    if cfg.is_complex:
        wr, wn2 = orc.cplx_residual(s, u0, U)
    else:
        wr, wn2 = orc.residual(s, u0, U)
    assert relmax(Rg.cpu().numpy(), wr) < 1e-11, cfg
    assert abs(rn2 - wn2) <= 1e-11 * wn2, cfg


@pytest.mark.parametrize("seed", range(200, 236))
def test_fuzz_solvers(orc, seed):
    """Linear random problems, all three solvers: identical iteration counts (unless a
    residual of the history lies within 12 % of the tolerance, where round-off may decide) and
    solutions within 1e-9."""
    cfg = draw(seed)
    cfg = synth.Config(cfg.name, cfg.dim, min(cfg.n, 63 if cfg.dim < 3 else 7), cfg.a, cfg.c, cfg.T,
                       min(cfg.nt, 64), max(cfg.alpha, 1e-3), scheme=cfg.scheme, q=(), a_im=cfg.a_im,
                       c_im=cfg.c_im, seed=seed)
    s = orc.spec(cfg)
    dt = torch.complex128 if cfg.is_complex else torch.float64
    u0 = synth.random_slice(cfg, seed)
    if cfg.is_complex:
        u0 = u0 + 1j * synth.random_slice(cfg, seed + 1)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=21)
    tol = 1e-11
    pre = "cplx_" if cfg.is_complex else ""
    runs = (("fixed_point", lambda: plan.fixed_point_solve(torch.from_numpy(np.asarray(u0)).to(DEV, dt), tol=tol,
                                                            maxit=60),
             lambda: getattr(orc, pre + "fixed_point")(s, u0, tol=tol, maxit=60)),
            ("gmres", lambda: plan.gmres_solve(torch.from_numpy(np.asarray(u0)).to(DEV, dt), tol=tol, restart=20,
                                               maxit=60),
             lambda: getattr(orc, pre + "gmres")(s, u0, tol=tol, restart=20, maxit=60)),
            ("bicgstab", lambda: plan.bicgstab_solve(torch.from_numpy(np.asarray(u0)).to(DEV, dt), tol=tol,
                                                     maxit=60),
             lambda: getattr(orc, pre + "bicgstab")(s, u0, tol=tol, maxit=60)))
    for name, gpu, ref in runs:
        U, rep = gpu()
        Uo, st, its, hist = ref()
        assert st == 0 and rep["converged"], (name, cfg)
        borderline = np.any(np.abs(np.log(np.maximum(hist, 1e-300) / tol)) < np.log(1.12))
        if borderline:
            assert abs(rep["iterations"] - its) <= 1, (name, cfg)
        else:
            assert rep["iterations"] == its, (name, cfg, rep["hist"], list(hist))
        assert relmax(U.cpu().numpy(), Uo) < 1e-9, (name, cfg)


@pytest.mark.parametrize("seed", range(300, 316))
def test_fuzz_picard(orc, seed):
    """Nonlinear random problems (ETD1 / ETD2 / IF-IMEX, N(u) = q1 u - u^3): the Picard sweep
    takes the oracle's iterations (borderline rule as above) to the oracle's fixed point."""
    rng = np.random.default_rng(seed)
    dim = int(rng.integers(1, 3))
    n = int(2 ** rng.integers(3, 8 if dim == 1 else 6) - 1)
    nt = int(2 ** rng.integers(2, 6))
    cfg = synth.Config(f"pic{seed}", dim, n, float(10 ** rng.uniform(-2, 0)), float(rng.uniform(0.2, 1.5)),
                       float(10 ** rng.uniform(-1.5, -0.3)), nt, float(10 ** rng.uniform(-3, -1.5)),
                       scheme=int(rng.choice([0, 1, 2])), q=(0.0, float(rng.uniform(-0.5, 0.5)), 0.0, -1.0), seed=seed)
    s = orc.spec(cfg)
    u0 = 0.5 * synth.random_slice(cfg, seed)
    plan = Plan(Problem.from_config(cfg))
    tol = 1e-11
    U, rep = plan.fixed_point_solve(torch.from_numpy(u0).to(DEV), tol=tol, maxit=80)
    Uo, st, its, hist = orc.fixed_point(s, u0, tol=tol, maxit=80)
    assert st == 0 and rep["converged"], cfg
    borderline = np.any(np.abs(np.log(np.maximum(hist, 1e-300) / tol)) < np.log(1.12))
    assert abs(rep["iterations"] - its) <= (1 if borderline else 0), (cfg, rep["hist"], list(hist))
    assert relmax(U.cpu().numpy(), Uo) < 1e-9, cfg
