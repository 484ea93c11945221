"""Pins for the complex-coefficient oracle (oracle/oracle_cplx.c; the paper's Schroedinger
tests a = i, c = 2i): every check is against something other than the oracle
itself -- dense complex matrices assembled from the FD stencil (scipy expm / solve),
unitarity, the per-mode closed form of the fixed-point residual, the real oracle on the real
and imaginary parts when the coefficients are real, GMRES termination."""
from __future__ import annotations

import numpy as np
import pytest
import scipy.linalg as sla

from test_oracle_pins import alpha_circulant, lapnd, rel


def cspec(orc, dim, n, a=1j, c=2j, T=0.5, nt=8, alpha=1e-2):
    a, c = complex(a), complex(c)
    return orc.Spec(dim, n, a.real, c.real, T, nt, alpha, 0, (), a.imag, c.imag)


def Lc(s):
    a, c = s.a + 1j * s.a_im, s.c + 1j * s.c_im
    return a * lapnd(s.n, s.dim) - c * np.eye(s.N)


def dense_Qalpha_c(s, alpha):
    A = sla.expm(s.dt * Lc(s))
    return np.eye(s.N * s.nt) - np.kron(alpha_circulant(s.nt, alpha), A)


def crandn(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


COEFS = [(1j, 2j), (0.3 + 1j, 0.5 - 0.2j), (1j, 200j)]


@pytest.mark.parametrize("a,c", COEFS)
@pytest.mark.parametrize("dim,n", [(1, 9), (2, 4)])
def test_cplx_sequential_vs_dense_expm(orc, a, c, dim, n):
    s = cspec(orc, dim, n, a, c, T=0.2, nt=6)
    u0 = crandn(np.random.default_rng(1), (n,) * dim)
    U = orc.cplx_sequential(s, u0)
    L = Lc(s)
    for k in range(1, s.nt + 1):
        want = sla.expm(k * s.dt * L) @ u0.reshape(-1)
        assert rel(U[k - 1].reshape(-1), want) < 1e-12


def test_cplx_schroedinger_is_unitary_and_sine_mode_phase(orc):
    """a = i, c = 2i: e^{dt L} is unitary, and u0 = sin(pi x) (the paper's initial condition,
    PAPER.md:983) is the first discrete mode, so u_n = e^{i n dt (lam_1 - 2)} u0 with lam_1
    the smallest-magnitude eigenvalue of the dense stencil."""
    n = 31
    s = cspec(orc, 1, n, 1j, 2j, T=0.16, nt=16)
    x = np.arange(1, n + 1) / (n + 1)
    u0 = np.sin(np.pi * x).astype(np.complex128)
    U = orc.cplx_sequential(s, u0)
    lam1 = np.linalg.eigvalsh(lapnd(n, 1)).max()
    for k in range(1, s.nt + 1):
        assert abs(np.linalg.norm(U[k - 1]) - np.linalg.norm(u0)) < 1e-13 * np.linalg.norm(u0)
        want = np.exp(1j * k * s.dt * (lam1 - 2.0)) * u0
        assert rel(U[k - 1], want) < 1e-11


@pytest.mark.parametrize("a,c", COEFS)
def test_cplx_residual_and_Q_vs_dense(orc, a, c):
    s = cspec(orc, 2, 3, a, c, T=0.3, nt=5)
    rng = np.random.default_rng(2)
    u0, U = crandn(rng, (3, 3)), crandn(rng, (5, 3, 3))
    A = sla.expm(s.dt * Lc(s))
    R, r2 = orc.cplx_residual(s, u0, U)
    Uf = U.reshape(5, -1)
    for k in range(5):
        prev = u0.reshape(-1) if k == 0 else Uf[k - 1]
        assert rel(R[k].reshape(-1), A @ prev - Uf[k]) < 1e-12
    assert abs(r2 - np.vdot(R, R).real) < 1e-12 * r2
    Q = np.eye(45) - np.kron(alpha_circulant(5, 0.0), A)
    assert rel(orc.cplx_apply_Q(s, U).reshape(-1), Q @ U.reshape(-1)) < 1e-12


@pytest.mark.parametrize("alpha", [0.3, 1e-2, 1e-4])
@pytest.mark.parametrize("a,c", COEFS)
@pytest.mark.parametrize("dim,n,nt", [(1, 5, 8), (1, 6, 7), (2, 3, 6)])
def test_cplx_precond_vs_dense_solve(orc, alpha, a, c, dim, n, nt):
    s = cspec(orc, dim, n, a, c, T=0.5, nt=nt, alpha=alpha)
    R = crandn(np.random.default_rng(3), (nt,) + (n,) * dim)
    S = orc.cplx_precond(s, R)
    want = np.linalg.solve(dense_Qalpha_c(s, alpha), R.reshape(-1))
    kappa = alpha ** (-(nt - 1) / nt)
    assert rel(S.reshape(-1), want) < 1e-15 * kappa * 50


def test_cplx_reduces_to_real_oracle_for_real_coefficients(orc):
    """a, c real: every complex operator acts on Re and Im separately as the real one."""
    s = cspec(orc, 2, 5, 0.7, 0.4, T=0.4, nt=6, alpha=0.05)
    sr = orc.Spec(2, 5, 0.7, 0.4, 0.4, 6, 0.05)
    rng = np.random.default_rng(4)
    u0, U = crandn(rng, (5, 5)), crandn(rng, (6, 5, 5))
    R, _ = orc.cplx_residual(s, u0, U)
    Rre, _ = orc.residual(sr, u0.real, U.real)
    Rim, _ = orc.residual(sr, u0.imag, U.imag)
    assert rel(R, Rre + 1j * Rim) < 1e-14
    S = orc.cplx_precond(s, R)
    Sre, _ = orc.precond(sr, R.real)
    Sim, _ = orc.precond(sr, R.imag)
    assert rel(S, Sre + 1j * Sim) < 1e-13


@pytest.mark.parametrize("a,c", COEFS)
def test_cplx_fixed_point_history_closed_form(orc, a, c):
    """r^k = (P - Q) P^{-1} r^{k-1} stays in the first time slot; per eigenmode J of the
    stencil the factor is -psi_J, psi_J = alpha e^{z_J T} / (1 - alpha e^{z_J T}),
    z_J = a lam_J - c complex (the derivation of Thm 2.1, with complex z)."""
    s = cspec(orc, 1, 12, a, c, T=0.4, nt=8, alpha=0.05)
    u0 = crandn(np.random.default_rng(5), 12)
    lam, W = np.linalg.eigh(lapnd(12, 1))
    z = (s.a + 1j * s.a_im) * lam - (s.c + 1j * s.c_im)
    c0 = W.T @ (sla.expm(s.dt * Lc(s)) @ u0)
    eT = np.exp(z * s.T)
    psi = s.alpha * eT / (1 - s.alpha * eT)
    U, st, its, hist = orc.cplx_fixed_point(s, u0, tol=1e-13)
    assert st == 0
    r0 = np.linalg.norm(c0)
    for k in range(len(hist)):
        want = np.linalg.norm(np.abs(psi) ** k * c0) / r0
        assert abs(hist[k] - want) < 1e-9 * want + 1e-15
    assert rel(U, orc.cplx_sequential(s, u0)) < 1e-11


@pytest.mark.parametrize("a,c", COEFS)
def test_cplx_gmres_terminates_and_matches_sequential(orc, a, c):
    """Thm 3.3 over C: at most N + 1 iterations."""
    s = cspec(orc, 1, 5, a, c, T=0.6, nt=6, alpha=0.3)
    u0 = crandn(np.random.default_rng(6), 5)
    U, st, its, hist = orc.cplx_gmres(s, u0, tol=1e-13, restart=50, maxit=50)
    assert st == 0 and its <= s.N + 1
    assert rel(U, orc.cplx_sequential(s, u0)) < 1e-11


def test_cplx_gmres_schroedinger_one_iteration(orc):
    """a = i, c = 2i, u0 = sin(pi x), dt = 0.01 -- 'the proposed method
    converges in just one iteration' (u0 is one eigenmode, so the Krylov space is one
    complex dimension)."""
    n = 127
    s = cspec(orc, 1, n, 1j, 2j, T=0.64, nt=64, alpha=1e-4)
    x = np.arange(1, n + 1) / (n + 1)
    u0 = np.sin(np.pi * x)
    U, st, its, hist = orc.cplx_gmres(s, u0, tol=1e-10, restart=20, maxit=20)
    assert st == 0 and its == 1
    assert rel(U, orc.cplx_sequential(s, u0)) < 1e-9


def test_cplx_bicgstab_on_dense_system(orc):
    """BiCGStab over C written out on the dense complex system Q_alpha^{-1} Q (test-side,
    Hermitian inner products np.vdot) takes the oracle's steps: same history, same x."""
    s = cspec(orc, 1, 4, 0.3 + 1j, 0.5 + 2j, T=0.5, nt=4, alpha=0.3)
    rng = np.random.default_rng(4)
    u0 = crandn(rng, 4)
    A = sla.expm(s.dt * Lc(s))
    Q = np.eye(16) - np.kron(alpha_circulant(4, 0.0), A)
    Qa = dense_Qalpha_c(s, s.alpha)
    B = np.linalg.solve(Qa, Q)
    f = np.zeros(16, dtype=complex)
    f[:4] = A @ u0
    b = np.linalg.solve(Qa, f)
    x = np.zeros_like(b)
    r = b.copy()
    rh = r.copy()
    beta0 = np.linalg.norm(r)
    rho_prev = al = om = 1.0
    p = np.zeros_like(b)
    v = np.zeros_like(b)
    hist = [1.0]
    for _ in range(30):
        rho = np.vdot(rh, r)
        beta = (rho / rho_prev) * (al / om)
        p = r + beta * (p - om * v)
        v = B @ p
        al = rho / np.vdot(rh, v)
        sv = r - al * v
        if np.linalg.norm(sv) / beta0 < 1e-13:
            x = x + al * p
            hist.append(np.linalg.norm(sv) / beta0)
            break
        t = B @ sv
        om = np.vdot(t, sv) / np.vdot(t, t).real
        x = x + al * p + om * sv
        r = sv - om * t
        rho_prev = rho
        hist.append(np.linalg.norm(r) / beta0)
        if hist[-1] < 1e-13:
            break
    U, st, its, h = orc.cplx_bicgstab(s, u0, tol=1e-13, maxit=30)
    assert st == 0 and its == len(hist) - 1 and its >= 2
    big = np.array(hist) > 1e-10
    assert np.allclose(h[big], np.array(hist)[big], rtol=1e-8)
    assert rel(U.reshape(-1), x) < 1e-10
    assert rel(U, orc.cplx_sequential(s, u0)) < 1e-10


@pytest.mark.parametrize("a,c", COEFS)
def test_cplx_bicgstab_matches_gmres_and_sequential(orc, a, c):
    s = cspec(orc, 2, 4, a, c, T=0.4, nt=8, alpha=0.2)
    u0 = crandn(np.random.default_rng(7), (4, 4))
    Ub, st, its, _ = orc.cplx_bicgstab(s, u0, tol=1e-12, maxit=60)
    Ug, st2, _, _ = orc.cplx_gmres(s, u0, tol=1e-12, restart=30, maxit=60)
    assert st == 0 and st2 == 0
    assert rel(Ub, Ug) < 1e-9 and rel(Ub, orc.cplx_sequential(s, u0)) < 1e-9


# ------------------------------------------------------------------------------------------
# complex exponential BDF2 (scheme 3, the 2D Schroedinger test of :1064)
# ------------------------------------------------------------------------------------------
def cspec3(orc, dim, n, a, c, T=0.5, nt=8, alpha=1e-2):
    a, c = complex(a), complex(c)
    return orc.Spec(dim, n, a.real, c.real, T, nt, alpha, 3, (), a.imag, c.imag)


def dense_R_c(s, alpha):
    """R_alpha = I - 4/3 (C_0^alpha (x) A) + 1/3 (C_1^alpha (x) A^2);
    alpha = 0 gives R."""
    A = sla.expm(s.dt * Lc(s))
    L = s.nt
    C0 = np.diag(np.ones(L - 1), -1)
    C1 = np.diag(np.ones(L - 2), -2)
    C0[0, L - 1] = alpha
    C1[0, L - 2] = alpha
    C1[1, L - 1] = alpha
    return np.eye(L * s.N) - 4 / 3 * np.kron(C0, A) + 1 / 3 * np.kron(C1, A @ A)


@pytest.mark.parametrize("a,c", COEFS)
def test_cplx_bdf2_sequential_is_exact(orc, a, c):
    """(4.1) from u_1 = A u_0 gives 4/3 A^n - 1/3 A^2 A^{n-2} = A^n exactly (R16)."""
    s = cspec3(orc, 1, 9, a, c, T=0.3, nt=6)
    u0 = crandn(np.random.default_rng(21), 9)
    U = orc.cplx_sequential(s, u0)
    for i in range(s.nt):
        assert rel(U[i], sla.expm((i + 2) * s.dt * Lc(s)) @ u0) < 1e-11


@pytest.mark.parametrize("a,c", COEFS)
def test_cplx_bdf2_residual_and_R_vs_dense(orc, a, c):
    s = cspec3(orc, 2, 3, a, c, T=0.3, nt=5)
    rng = np.random.default_rng(22)
    u0, U = crandn(rng, (3, 3)), crandn(rng, (5, 3, 3))
    A = sla.expm(s.dt * Lc(s))
    u1 = A @ u0.reshape(-1)
    f = np.zeros(45, dtype=complex)
    f[:9] = 4 / 3 * A @ u1 - 1 / 3 * A @ A @ u0.reshape(-1)
    f[9:18] = -1 / 3 * A @ A @ u1
    R, _ = orc.cplx_residual(s, u0, U)
    assert rel(R.reshape(-1), f - dense_R_c(s, 0.0) @ U.reshape(-1)) < 1e-12
    assert rel(orc.cplx_apply_Q(s, U).reshape(-1), dense_R_c(s, 0.0) @ U.reshape(-1)) < 1e-12


@pytest.mark.parametrize("alpha", [0.3, 1e-2, 1e-4])
@pytest.mark.parametrize("a,c", COEFS)
@pytest.mark.parametrize("dim,n,nt", [(1, 5, 8), (2, 3, 6)])
def test_cplx_bdf2_precond_vs_dense_solve(orc, alpha, a, c, dim, n, nt):
    s = cspec3(orc, dim, n, a, c, T=0.5, nt=nt, alpha=alpha)
    R = crandn(np.random.default_rng(23), (nt,) + (n,) * dim)
    S = orc.cplx_precond(s, R)
    want = np.linalg.solve(dense_R_c(s, alpha), R.reshape(-1))
    kappa = alpha ** (-(nt - 1) / nt)
    assert rel(S.reshape(-1), want) < 1e-15 * kappa * 200


@pytest.mark.parametrize("a,c", COEFS)
def test_cplx_bdf2_solvers_reach_sequential(orc, a, c):
    s = cspec3(orc, 2, 4, a, c, T=0.4, nt=8, alpha=0.05)
    u0 = crandn(np.random.default_rng(24), (4, 4))
    Us = orc.cplx_sequential(s, u0)
    for solve in (lambda: orc.cplx_fixed_point(s, u0, tol=1e-13, maxit=80),
                  lambda: orc.cplx_gmres(s, u0, tol=1e-13, restart=40, maxit=80),
                  lambda: orc.cplx_bicgstab(s, u0, tol=1e-13, maxit=80)):
        U, st, its, _ = solve()
        assert st == 0 and rel(U, Us) < 1e-10


@pytest.mark.parametrize("n,nt", [(31, 16), (31, 32), (31, 64), (63, 16)])
def test_cplx_bdf2_gmres_three_iterations(orc, n, nt):
    """the 2D Schroedinger equation (a = i, c = 200i, the Gaussian packet of
    :1066, dt = 0.05, alpha_opt = 0.0001953125) with the BDF2 preconditioner: GMRES
    "consistently converges in just three iterations, regardless of the window size" (the
    tolerance is not printed: any tol in [1e-11, 1e-8] gives 3 here; h = 1/32, 1/64 instead
    of 1/40, which the power-of-two DST does not take)."""
    s = cspec3(orc, 2, n, 1j, 200j, T=0.05 * nt, nt=nt, alpha=0.0001953125)
    x = np.arange(1, n + 1) / (n + 1) - 0.5
    g = np.exp(-x * x / (2 * 0.05 ** 2))
    u0 = np.multiply.outer(g, g * np.exp(-5j * x))
    U, st, its, hist = orc.cplx_gmres(s, u0, tol=1e-10, restart=20, maxit=20)
    assert st == 0 and its == 3
    assert rel(U, orc.cplx_sequential(s, u0)) < 1e-9
