"""GPU parity at BASELINE.json's full sizes, in the launch configurations bench.py times.

* c2 (255^2 x 64, BASELINE.json:8) and c3 (511^2 x 128, :9): the oracle finishes a whole
  residual / preconditioner apply in seconds (c2) or about a minute (c3), so the primitives
  are compared element by element at the north_star tolerance (relative max error <= 1e-11,
  reading R9), and the c2 solves (fixed point, GMRES(20)) with identical iteration counts and
  solutions within 1e-9.
* c5 (2047^2 x 256, :11): one ETD2 Picard sweep of the resident state -- stage 3 (the TMA line
  kernels) and K1 (k_time_tma<256, ...> in its ETD2 form, the kernel the bench times) -- from
  a nonlinear state, compared at sampled DST modes with the oracle's per-mode residual
  (PAPER.md:181-183 with the ETD2 Phi terms, reading R6) and per-mode Steps (a)-(c)
  (PAPER.md:188-197); the N-hat history the residual needs is taken by the oracle's own sums
  (orc_dst_sample of orc_nonlin of each physical slice).
* the largest line (n + 1 = 4096): the converged GPU Picard solution satisfies the oracle's
  all-at-once equations at sampled modes.
* c4 (255^3 x 64, :10): the preconditioner apply and the residual on inputs made of a few
  separable sine modes, against the oracle's per-mode formulas at those modes, every other
  mode at round-off; GMRES(3) from a separable u0 against the sequential solution E_J^t u-hat_0.
"""
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


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(DEV)


def H(t):
    return t.detach().cpu().numpy()


def relmax(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def primitives_parity(orc, cfg):
    s = orc.spec(cfg)
    plan = Plan(Problem.from_config(cfg))
    R = synth.random_spacetime(cfg)
    S = H(plan.precond_apply(T(R)))
    want, leak = orc.precond(s, R)
    assert leak < 1e-8
    assert relmax(S, want) < 1e-11
    del S, want
    u0 = synth.initial_condition(cfg)
    U = synth.random_spacetime(cfg, scale=0.5)
    Rg, rn2 = plan.residual(T(u0), T(U), norm=True)
    wr, wn2 = orc.residual(s, u0, U)
    assert relmax(H(Rg), wr) < 1e-11
    assert abs(rn2 - wn2) < 1e-11 * wn2


def test_c2_full_size_primitives(orc):
    primitives_parity(orc, synth.CONFIGS["c2"])


@pytest.mark.slow
def test_c3_full_size_primitives(orc):
    primitives_parity(orc, synth.CONFIGS["c3"])


def test_c2_full_size_solves(orc):
    cfg = synth.CONFIGS["c2"]
    s = orc.spec(cfg)
    u0 = synth.initial_condition(cfg)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=21)
    U, rep = plan.fixed_point_solve(T(u0), tol=cfg.tol, maxit=50)
    Uo, st, its, hist = orc.fixed_point(s, u0, tol=cfg.tol, maxit=50)
    assert st == 0 and rep["converged"] and rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9
    U, rep = plan.gmres_solve(T(u0), tol=cfg.tol, restart=20, maxit=50)
    Uo, st, its, hist = orc.gmres(s, u0, tol=cfg.tol, restart=20, maxit=50)
    assert st == 0 and rep["converged"] and rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9


def _oracle_mode_data(orc, s, u0, U, J):
    """DST coefficients at the modes J of u0 and of every slice of U, and of N(u_m) for
    m = 0..nt-1 (u_0 = u0), all by the oracle's plain sums."""
    uh0 = orc.dst_sample(s, u0, J)
    uh = orc.dst_sample_batch(s, U, J)  # [nt][len(J)]
    nh = np.empty_like(uh)
    nh[0] = orc.dst_sample(s, orc.nonlin(s, u0), J)
    for m in range(1, s.nt):
        nh[m] = orc.dst_sample(s, orc.nonlin(s, U[m - 1]), J)
    return uh0, uh, nh


def test_c5_full_size_etd2_sweep_sampled(orc):
    """One ETD2 Picard sweep at c5's full size, through stage 3 and K1's ETD2 form."""
    cfg = synth.CONFIGS["c5"]
    s = orc.spec(cfg)
    u0 = synth.initial_condition(cfg)
    U, ks = synth.sparse_spacetime(cfg, nmodes=6)
    U *= 0.2  # |u| ~ 1: the cube is a genuinely nonlinear, mode-mixing term
    plan = Plan(Problem.from_config(cfg))
    plan.load_state(T(u0), T(U))
    plan.sweep()
    rn2 = plan.sweep_norm2()
    Ud = torch.empty((cfg.nt,) + cfg.shape, dtype=torch.float64, device=DEV)
    plan.store_state(Ud)
    U2 = H(Ud)
    del Ud, plan
    n = cfg.n
    # 3 modes of U, 2 modes only the cube reaches (k_x + k_x' + k_x'' etc.), 1 far mode
    J = [int((k[1] - 1) * n + (k[0] - 1)) for k in ks[:3]]
    J += [int((ks[0][1] - 1) * n + (min(3 * ks[0][0], n) - 1)), int(2 * n + 4), int(1500 * n + 1900)]
    uh0, uh, nh = _oracle_mode_data(orc, s, u0, U, J)
    uh2 = orc.dst_sample_batch(s, U2, J)
    scale = np.abs(uh).max()
    for m, j in enumerate(J):
        r = orc.mode_residual(s, j, uh[:, m], uh0[m], nh[:, m])
        want = uh[:, m] + orc.mode_precond(s, j, r)
        assert np.abs(uh2[:, m] - want).max() < 1e-11 * scale, j
    assert np.isfinite(rn2) and rn2 > 0


def test_max_line_length_picard_solution_satisfies_oracle_equations(orc):
    """n + 1 = 4096 (the largest line the kernels take), 2D ETD2: the GPU Picard solution U
    satisfies the oracle's all-at-once residual equations at sampled modes (the residual the
    oracle computes from U's own DST coefficients is at round-off relative to U)."""
    cfg = synth.CONFIGS["c5"].scaled(4095, 4)
    s = orc.spec(cfg)
    u0 = synth.initial_condition(cfg)
    plan = Plan(Problem.from_config(cfg))
    U, rep = plan.fixed_point_solve(T(u0), tol=1e-12, maxit=30)
    assert rep["converged"]
    U = H(U)
    del plan
    n = cfg.n
    J = [0, 1, n + 1, 3 * n + 5, 60 * n + 63, 4000 * n + 4000]
    uh0, uh, nh = _oracle_mode_data(orc, s, u0, U, J)
    scale = max(np.abs(uh).max(), np.abs(uh0).max())
    for m, j in enumerate(J):
        r = orc.mode_residual(s, j, uh[:, m], uh0[m], nh[:, m])
        assert np.abs(r).max() < 1e-11 * scale, j



def test_c4_full_size_primitives_sampled(orc):
    """c4 (255^3 x 64, BASELINE.json:10, 3-D, the GMRES config) at full size: the
    preconditioner apply and the residual on inputs made of a few separable sine modes, whose
    DST coefficients are known, against the oracle's per-mode Steps (a)-(c)
    and per-mode residual; the outputs are taken to the DST basis by the
    plan's own DST (parity-tested separately) and every other mode must stay at round-off.
    (c4's own u0 decays by ~1e-17 per step, so its GMRES solution is checked at reduced size.)"""
    cfg = synth.CONFIGS["c4"]
    s = orc.spec(cfg)
    n, nt = cfg.n, cfg.nt
    ks = [(1, 1, 1), (2, 3, 1), (5, 1, 7), (40, 90, 3)]  # (k_x, k_y, k_z)
    x = np.arange(1, n + 1) / (n + 1)
    Sk = lambda k: np.sin(np.pi * k * x)  # noqa: E731
    J = [(kz - 1) * n * n + (ky - 1) * n + (kx - 1) for kx, ky, kz in ks]
    # the orthonormal DST's coefficient of one separable mode (oracle sums, one call per mode)
    unit = np.array([orc.dst_sample(s, np.multiply.outer(Sk(kz), np.multiply.outer(Sk(ky), Sk(kx))), [j])[0]
                     for (kx, ky, kz), j in zip(ks, J)])
    F = [torch.from_numpy(np.stack([Sk(k[a]) for k in ks])).to(DEV) for a in range(3)]  # [mode][n] per axis
    rng = np.random.default_rng(44)

    def field(C):  # sum_m C[m, t] phi_m as [t][z][y][x] on the device
        return torch.einsum("mt,mz,my,mx->tzyx", T(C), F[2], F[1], F[0]).contiguous()

    def spectral_at(Y):  # the plan's DST of every slice, at the sampled modes; + the rest
        Yh = plan.dst(Y).reshape(Y.shape[0], -1)
        at = H(Yh[:, J])
        Yh[:, J] = 0.0
        return at, float(Yh.abs().max())

    plan = Plan(Problem.from_config(cfg))
    C = rng.standard_normal((len(ks), nt))
    S = plan.precond_apply(field(C))
    got, rest = spectral_at(S)
    want = np.stack([orc.mode_precond(s, j, C[m] * unit[m]) for m, j in enumerate(J)], 1)
    scale = np.abs(want).max()
    assert np.abs(got - want).max() < 1e-11 * scale and rest < 1e-11 * scale
    del S
    D = 0.5 * rng.standard_normal((len(ks), nt))
    e0 = rng.standard_normal(len(ks))
    u0 = field(e0[:, None])[0]
    R, rn2 = plan.residual(u0, field(D), norm=True)
    got, rest = spectral_at(R)
    want = np.stack([orc.mode_residual(s, j, D[m] * unit[m], e0[m] * unit[m]) for m, j in enumerate(J)], 1)
    scale = np.abs(want).max()
    assert np.abs(got - want).max() < 1e-11 * scale and rest < 1e-11 * scale
    assert abs(rn2 - float((want ** 2).sum())) < 1e-11 * rn2


def test_c4_full_size_gmres_separable_modes(orc):
    """GMRES(3) at c4's full size (the bench's GMRES configuration) from a u0 made of three
    slowly decaying separable modes: the solution of the all-at-once system is the sequential
    one, u-hat_t(J) = E_J^(t+1) u-hat_0(J) (slice t holds u_{t+1}), with the
    oracle's E_J; every other mode stays at round-off."""
    cfg = synth.CONFIGS["c4"]
    s = orc.spec(cfg)
    n, nt = cfg.n, cfg.nt
    ks = [(1, 1, 1), (2, 1, 1), (1, 2, 2)]
    x = np.arange(1, n + 1) / (n + 1)
    Sk = lambda k: np.sin(np.pi * k * x)  # noqa: E731
    J = [(kz - 1) * n * n + (ky - 1) * n + (kx - 1) for kx, ky, kz in ks]
    e0 = np.array([1.0, -0.7, 0.4])
    u0 = sum(c * np.multiply.outer(Sk(kz), np.multiply.outer(Sk(ky), Sk(kx))) for c, (kx, ky, kz) in zip(e0, ks))
    uh0 = orc.dst_sample(s, u0, J)
    E = orc.mode_tables(s)[1].reshape(-1)[J]
    plan = Plan(Problem.from_config(cfg), krylov_vectors=4)
    plan.set_zero_guess(True)
    U, rep = plan.gmres_solve(T(u0), tol=cfg.tol, restart=3, maxit=20)
    assert rep["converged"]
    Uh = plan.dst(U).reshape(nt, -1)
    got = H(Uh[:, J])
    Uh[:, J] = 0.0
    want = np.stack([E ** (t + 1) * uh0 for t in range(nt)])
    scale = np.abs(uh0).max()
    assert np.abs(got - want).max() < 1e-9 * scale and float(Uh.abs().max()) < 1e-11 * scale
