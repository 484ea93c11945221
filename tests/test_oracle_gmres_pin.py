"""Exact pin of the oracle's GMRES(m) (oracle/oracle.c orc_gmres, oracle/oracle_cplx.c
orc_cplx_gmres): iteration count and the whole relative residual history.

PAPER.md:284-289 (Sec. 3.2) runs GMRES on the preconditioned system Q_alpha^{-1} Q U =
Q_alpha^{-1} f; reading R11 fixes the variant (left preconditioning, restart m, zero
initial guess, stop on the preconditioned residual relative to the initial one, iterations =
Arnoldi matvecs, happy breakdown counts as converged).  The replica below is written here,
independently of the oracle: it assembles B = Q_alpha^{-1} Q and b = Q_alpha^{-1} f as dense
Kronecker matrices from the FD stencil (scipy expm, numpy solve), orthogonalises with
modified Gram-Schmidt and takes the residual estimate min_y ||beta e1 - H_j y|| from a dense
least-squares solve instead of Givens rotations.  The two agree in exact arithmetic; an
off-by-one in the oracle's counter or stop test, a dropped restart residual or a wrong
rotation changes the count or the history and fails here.
"""
from __future__ import annotations

import numpy as np
import pytest
import scipy.linalg as sla

from test_oracle_pins import Lh, alpha_circulant, bdf2_dense, rel, spec


def dense_gmres(B, b, tol, m, maxit):
    """Left-preconditioned GMRES(m) on B x = b from x = 0 (test-side, R11)."""
    x = np.zeros_like(b)
    hist = [1.0]
    its = 0
    beta0 = None
    while its < maxit:
        r = b - B @ x
        beta = np.linalg.norm(r)
        if beta0 is None:
            beta0 = beta
        if beta0 == 0 or beta / beta0 < tol:
            break
        V = [r / beta]
        H = np.zeros((m + 1, m), dtype=b.dtype)
        done = False
        y = np.zeros(0, dtype=b.dtype)
        for j in range(m):
            if its >= maxit:
                break
            w = B @ V[j]
            for i in range(j + 1):  # modified Gram-Schmidt (the oracle uses CGS2)
                H[i, j] = np.vdot(V[i], w)
                w = w - H[i, j] * V[i]
            hn = np.linalg.norm(w)
            H[j + 1, j] = hn
            e1 = np.zeros(j + 2, dtype=b.dtype)
            e1[0] = beta
            y, *_ = np.linalg.lstsq(H[: j + 2, : j + 1], e1, rcond=None)
            res = np.linalg.norm(e1 - H[: j + 2, : j + 1] @ y)
            its += 1
            hist.append(res / beta0)
            if res / beta0 < tol or hn == 0:
                done = True
                break
            V.append(w / hn)
        x = x + np.array(V[: len(y)]).T @ y
        if done:
            break
    return x, its, np.array(hist)


def check_history(hist_orc, its_orc, hist_ref, its_ref, tol):
    assert its_orc == its_ref, (its_orc, its_ref, hist_orc, hist_ref)
    # no residual within 12 % of the tolerance: the count is decided with a margin
    assert np.all(np.abs(np.log(np.asarray(hist_ref[1:]) / tol)) > np.log(1.12))
    # every entry to 1e-8 relative, plus an absolute 1e-16 for the round-off floor of a
    # relative residual (entries below 1e-13 are round-off and skipped)
    big = np.asarray(hist_ref) > 1e-13
    assert np.allclose(np.asarray(hist_orc)[big], np.asarray(hist_ref)[big], rtol=1e-8, atol=1e-16)


def exp_euler_system(s, u0, A):
    C0 = np.diag(np.ones(s.nt - 1), -1)
    Q = np.eye(s.nt * s.N, dtype=A.dtype) - np.kron(C0, A)
    Qa = np.eye(s.nt * s.N, dtype=A.dtype) - np.kron(alpha_circulant(s.nt, s.alpha), A)
    f = np.zeros(s.nt * s.N, dtype=A.dtype)
    f[: s.N] = A @ u0.reshape(-1)  # f = (A u_0, 0, ..., 0)
    return np.linalg.solve(Qa, Q), np.linalg.solve(Qa, f)


@pytest.mark.parametrize(
    "dim,n,a,c,T,nt,alpha,restart,tol",
    [
        (1, 6, 0.05, 0.0, 0.5, 8, 0.3, 50, 1e-12),  # unrestarted: 6 <= N + 1 (Thm 3.3)
        (1, 8, 0.01, 0.0, 1.0, 8, 0.5, 50, 1e-12),  # unrestarted: 8 <= N + 1
        (1, 6, 0.05, 0.0, 0.5, 8, 0.3, 3, 1e-12),   # restart 3: three restart cycles
        (1, 6, 0.02, 0.0, 0.5, 8, 0.45, 2, 1e-12),  # restart 2: seven cycles
        (2, 3, 0.02, 0.0, 0.5, 8, 0.35, 3, 1e-12),  # 2D Kronecker operator, restarted
    ],
)
def test_gmres_count_and_history_exact(orc, dim, n, a, c, T, nt, alpha, restart, tol):
    s = spec(orc, dim, n, a=a, c=c, T=T, nt=nt, alpha=alpha)
    u0 = np.random.default_rng(3).standard_normal((n,) * dim)
    A = sla.expm(s.dt * Lh(s))
    B, b = exp_euler_system(s, u0, A)
    maxit = 60
    x, its, hist = dense_gmres(B, b, tol, restart, maxit)
    U, st, its_o, hist_o = orc.gmres(s, u0, tol=tol, restart=restart, maxit=maxit)
    assert st == 0
    assert its >= 3  # a non-trivial history
    check_history(hist_o, its_o, hist, its, tol)
    assert rel(U.reshape(-1), x) < 1e-9


def test_gmres_maxit_cut(orc):
    """maxit reached: the oracle stops after exactly maxit matvecs, reports NOT_CONVERGED (7),
    and its history is the replica's first maxit + 1 entries."""
    s = spec(orc, 1, 6, a=0.05, c=0.0, T=0.5, nt=8, alpha=0.3)
    u0 = np.random.default_rng(3).standard_normal(6)
    A = sla.expm(s.dt * Lh(s))
    B, b = exp_euler_system(s, u0, A)
    _, its, hist = dense_gmres(B, b, 1e-14, 3, 5)
    U, st, its_o, hist_o = orc.gmres(s, u0, tol=1e-14, restart=3, maxit=5)
    assert st == 7 and its == its_o == 5
    assert np.allclose(hist_o, hist, rtol=1e-8)


def test_gmres_bdf2_count_and_history_exact(orc):
    """Exponential BDF2 (4.2)-(4.5): GMRES on R_alpha^{-1} R v =
    R_alpha^{-1} f2 (reading R16: u_1 = A u_0)."""
    s = spec(orc, 1, 5, a=0.02, c=0.0, T=0.8, nt=8, alpha=0.3, scheme=3)
    u0 = np.random.default_rng(8).standard_normal(5)
    A, Bm, R, Ra = bdf2_dense(s)
    u1 = A @ u0
    f2 = np.zeros(s.nt * s.N)
    f2[: s.N] = 4.0 / 3.0 * A @ u1 - 1.0 / 3.0 * Bm @ u0
    f2[s.N: 2 * s.N] = -1.0 / 3.0 * Bm @ u1
    for restart in (50, 3):
        x, its, hist = dense_gmres(np.linalg.solve(Ra, R), np.linalg.solve(Ra, f2), 1e-12, restart, 60)
        U, st, its_o, hist_o = orc.gmres(s, u0, tol=1e-12, restart=restart, maxit=60)
        assert st == 0 and its >= 3
        check_history(hist_o, its_o, hist, its, 1e-12)
        assert rel(U.reshape(-1), x) < 1e-9


@pytest.mark.parametrize("restart", [50, 3])
def test_cplx_gmres_count_and_history_exact(orc, restart):
    """Complex coefficients (NEXT-4, reading R18: GMRES over C, Hermitian inner product):
    a = 0.01 + 0.05i, c = 0.02 - 0.2i (slowly damped, rotating spectrum: many iterations)."""
    a, c = 0.01 + 0.05j, 0.02 - 0.2j
    s = orc.Spec(1, 5, a.real, c.real, 0.6, 8, 0.3, 0, (), a.imag, c.imag)
    rng = np.random.default_rng(9)
    u0 = rng.standard_normal(5) + 1j * rng.standard_normal(5)
    from test_oracle_pins import lapnd

    L = a * lapnd(5, 1) - c * np.eye(5)
    A = sla.expm(s.dt * L)
    B, b = exp_euler_system(s, u0, A)
    x, its, hist = dense_gmres(B, b, 1e-12, restart, 60)
    U, st, its_o, hist_o = orc.cplx_gmres(s, u0, tol=1e-12, restart=restart, maxit=60)
    assert st == 0 and its >= 3
    check_history(hist_o, its_o, hist, its, 1e-12)
    assert rel(U.reshape(-1), x) < 1e-9
