"""GPU parity for complex-coefficient plans (NEXT-4: the paper's Schroedinger tests, a = i,
c = 2i / 200i) against the complex oracle (oracle/oracle_cplx.c).
Same bars as test_gpu_parity.py: preconditioner apply / residual relative max error
<= 1e-11, solves with identical iteration counts and solution error <= 1e-9."""
from __future__ import annotations

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_04350_b200 import ExpdError, Plan, Problem  # noqa: E402

DEV = torch.device("cuda:0")


def TC(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(DEV)


def H(t):
    return t.detach().cpu().numpy()


def relmax(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def cfg_of(name, n=None, nt=None):
    c = synth.CONFIGS[name]
    return c if n is None else c.scaled(n, nt)


# nt 4 / 8: single-stage register K1; 16..256: the TMA K1 (L = 2, 3); dims 1..3
CASES = [("c6se", None, None), ("c6se", 63, 4), ("c6se", 31, 8), ("c7se", 31, 16), ("c7se", 15, 64),
         ("c7se", 31, 128), ("c7se", 7, 256),
         ("c6se", 3, 4), ("c7se", 3, 8), ("c6se", 4095, 4), ("c7se", 255, 4)]  # smallest / largest lines
CASES3 = [("c7se", 7, 32)]


def cfg3(nt):
    return synth.Config("c7se3d", 3, 7, 0.3, 0.1, 0.2, nt, 1e-2, a_im=1.0, c_im=5.0, seed=9)


@pytest.mark.parametrize("name,n,nt", CASES)
def test_cplx_precond_parity(orc, name, n, nt):
    cfg = cfg_of(name, n, nt)
    plan = Plan(Problem.from_config(cfg))
    R = synth.random_spacetime(cfg)
    S = H(plan.precond_apply(TC(R)))
    assert relmax(S, orc.cplx_precond(orc.spec(cfg), R)) < 1e-11


@pytest.mark.parametrize("nt", [8, 32])
def test_cplx_precond_parity_3d_general_coefficients(orc, nt):
    cfg = cfg3(nt)  # a = 0.3 + i, c = 0.1 + 5i: damped and oscillatory at once
    plan = Plan(Problem.from_config(cfg))
    R = synth.random_spacetime(cfg)
    assert relmax(H(plan.precond_apply(TC(R))), orc.cplx_precond(orc.spec(cfg), R)) < 1e-11


@pytest.mark.parametrize("name,n,nt", CASES)
def test_cplx_residual_parity(orc, name, n, nt):
    cfg = cfg_of(name, n, nt)
    plan = Plan(Problem.from_config(cfg))
    u0 = synth.initial_condition(cfg)
    U = synth.random_spacetime(cfg, scale=0.5)
    R, rn2 = plan.residual(TC(u0), TC(U), norm=True)
    want, wn2 = orc.cplx_residual(orc.spec(cfg), u0, U)
    assert relmax(H(R), want) < 1e-11
    assert abs(rn2 - wn2) < 1e-11 * wn2


@pytest.mark.parametrize("name,n,nt", [("c6se", None, None), ("c7se", 31, 64), ("c7se", 15, 8)])
def test_cplx_fixed_point_parity(orc, name, n, nt):
    cfg = cfg_of(name, n, nt)
    plan = Plan(Problem.from_config(cfg))
    u0 = synth.initial_condition(cfg)
    U, rep = plan.fixed_point_solve(TC(u0), tol=cfg.tol, maxit=50)
    Uo, st, its, hist = orc.cplx_fixed_point(orc.spec(cfg), u0, tol=cfg.tol, maxit=50)
    assert st == 0 and rep["converged"]
    assert rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9
    h = np.array(rep["hist"])
    big = hist > 1e-9
    assert np.allclose(h[big], hist[big], rtol=1e-6)


@pytest.mark.parametrize("name,n,nt", [("c6se", None, None), ("c7se", 31, 64), ("c7se", 15, 16)])
def test_cplx_gmres_parity(orc, name, n, nt):
    cfg = cfg_of(name, n, nt)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=21)
    u0 = synth.initial_condition(cfg)
    U, rep = plan.gmres_solve(TC(u0), tol=cfg.tol, restart=20, maxit=50)
    Uo, st, its, hist = orc.cplx_gmres(orc.spec(cfg), u0, tol=cfg.tol, restart=20, maxit=50)
    assert st == 0 and rep["converged"]
    assert rep["iterations"] == its
    if name == "c6se" and n is None:
        assert its == 1  # "converges in just one iteration"
    assert relmax(H(U), Uo) < 1e-9


def test_cplx_gmres_restart_several_iterations(orc):
    # alpha = 0.3, random u0: many modes, complex Givens over several restarts
    cfg = synth.Config("g", 1, 15, 0.2, 0.1, 0.5, 16, 0.3, a_im=1.0, c_im=2.0, seed=3)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=2)
    rng = np.random.default_rng(3)
    u0 = rng.standard_normal(15) + 1j * rng.standard_normal(15)
    U, rep = plan.gmres_solve(TC(u0), tol=1e-12, restart=2, maxit=60)
    Uo, st, its, hist = orc.cplx_gmres(orc.spec(cfg), u0, tol=1e-12, restart=2, maxit=60)
    assert rep["iterations"] == its and its > 2
    assert relmax(H(U), Uo) < 1e-9


@pytest.mark.parametrize("name,n,nt", [("c6se", None, None), ("c7se", 31, 64), ("c7se", 15, 16)])
def test_cplx_bicgstab_parity(orc, name, n, nt):
    cfg = cfg_of(name, n, nt)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=6)
    u0 = synth.initial_condition(cfg)
    U, rep = plan.bicgstab_solve(TC(u0), tol=cfg.tol, maxit=50)
    Uo, st, its, hist = orc.cplx_bicgstab(orc.spec(cfg), u0, tol=cfg.tol, maxit=50)
    assert st == 0 and rep["converged"]
    assert rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9


def test_cplx_bicgstab_several_steps(orc):
    cfg = synth.Config("b", 1, 15, 0.05, 0.0, 0.5, 16, 0.2, a_im=1.0, c_im=2.0, seed=3)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=6)
    rng = np.random.default_rng(3)
    u0 = rng.standard_normal(15) + 1j * rng.standard_normal(15)
    U, rep = plan.bicgstab_solve(TC(u0), tol=1e-12, maxit=60)
    Uo, st, its, hist = orc.cplx_bicgstab(orc.spec(cfg), u0, tol=1e-12, maxit=60)
    assert rep["iterations"] == its and its >= 3
    h = np.array(rep["hist"])
    assert np.allclose(h[hist > 1e-9], hist[hist > 1e-9], rtol=1e-6)
    assert relmax(H(U), Uo) < 1e-9


def test_cplx_full_size_sampled_modes(orc):
    """c7se at full size (1023^2 x 128, complex): the converged Picard solution in the DST
    basis is u-hat_J(t) = E_J^t u-hat_J(0) (the sequential scheme), checked on
    sampled modes; E_J from the oracle's pinned axis eigenvalues in long double."""
    cfg = synth.CONFIGS["c7se"]
    s = orc.spec(cfg)
    plan = Plan(Problem.from_config(cfg))
    u0 = synth.initial_condition(cfg)
    U, rep = plan.fixed_point_solve(TC(u0), tol=cfg.tol, maxit=20)
    assert rep["converged"]
    Uh = H(U)
    rng = np.random.default_rng(11)
    kx = rng.integers(1, 40, 6)
    ky = 2 * rng.integers(0, 20, 6) + 1  # u0 is even in y about 1/2: only odd k_y carry signal
    idx = (ky - 1) * cfg.n + (kx - 1)
    ts = np.array([0, 1, 63, 127])
    uh0 = orc.dst_sample(s, u0.real, idx) + 1j * orc.dst_sample(s, u0.imag, idx)
    got = orc.dst_sample_batch(s, Uh[ts].real, idx) + 1j * orc.dst_sample_batch(s, Uh[ts].imag, idx)
    lam = orc.axis_eigs(cfg.n).astype(np.longdouble)
    mu = lam[kx - 1] + lam[ky - 1]
    a = np.clongdouble(complex(cfg.a, cfg.a_im))
    c = np.clongdouble(complex(cfg.c, cfg.c_im))
    z = np.longdouble(cfg.dt) * (a * mu - c)
    for i, t in enumerate(ts):
        want = np.exp(z * (t + 1)) * uh0
        # scale: ||u0||_2 = ||V u0||_2 bounds every coefficient (V orthonormal)
        assert np.abs(got[i] - want.astype(np.complex128)).max() < 1e-9 * np.linalg.norm(u0)


# ------------------------------------------------------------------------------------------
# complex BDF2 (K1 form 5; the paper's 2D Schroedinger setup)
# ------------------------------------------------------------------------------------------
BDF_CASES = [("c7bdf2", 31, 32), ("c7bdf2", 15, 8), ("c7bdf2", 7, 256), ("c7bdf2", 15, 128)]


@pytest.mark.parametrize("name,n,nt", BDF_CASES)
def test_cplx_bdf2_precond_and_residual_parity(orc, name, n, nt):
    cfg = cfg_of(name, n, nt)
    s = orc.spec(cfg)
    plan = Plan(Problem.from_config(cfg))
    R = synth.random_spacetime(cfg)
    assert relmax(H(plan.precond_apply(TC(R))), orc.cplx_precond(s, R)) < 1e-11
    u0 = synth.initial_condition(cfg)
    U = synth.random_spacetime(cfg, scale=0.5)
    Rg, rn2 = plan.residual(TC(u0), TC(U), norm=True)
    want, wn2 = orc.cplx_residual(s, u0, U)
    assert relmax(H(Rg), want) < 1e-11
    assert abs(rn2 - wn2) < 1e-11 * wn2


@pytest.mark.parametrize("solver", ["fixed_point", "gmres", "bicgstab"])
def test_cplx_bdf2_solver_parity(orc, solver):
    cfg = cfg_of("c7bdf2", 31, 32)
    s = orc.spec(cfg)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=21)
    u0 = synth.initial_condition(cfg)
    if solver == "fixed_point":
        U, rep = plan.fixed_point_solve(TC(u0), tol=cfg.tol, maxit=50)
        Uo, st, its, _ = orc.cplx_fixed_point(s, u0, tol=cfg.tol, maxit=50)
    elif solver == "gmres":
        U, rep = plan.gmres_solve(TC(u0), tol=cfg.tol, restart=20, maxit=50)
        Uo, st, its, _ = orc.cplx_gmres(s, u0, tol=cfg.tol, restart=20, maxit=50)
        assert its == 3
    else:
        U, rep = plan.bicgstab_solve(TC(u0), tol=cfg.tol, maxit=50)
        Uo, st, its, _ = orc.cplx_bicgstab(s, u0, tol=cfg.tol, maxit=50)
    assert st == 0 and rep["converged"] and rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9


def test_cplx_bdf2_full_size_sampled_modes(orc):
    """c7bdf2 at full size (1023^2 x 128, complex, BDF2): GMRES converges in 3 iterations and
    the solution's DST modes are E_J^{t+2} u-hat_J(0) (BDF2 is exact on the linear problem,
    reading R16)."""
    cfg = synth.CONFIGS["c7bdf2"]
    s = orc.spec(cfg)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=5)
    u0 = synth.initial_condition(cfg)
    U, rep = plan.gmres_solve(TC(u0), tol=cfg.tol, restart=4, maxit=20)
    assert rep["converged"] and rep["iterations"] == 3
    Uh = H(U)
    rng = np.random.default_rng(12)
    kx = rng.integers(1, 40, 6)
    ky = 2 * rng.integers(0, 20, 6) + 1
    idx = (ky - 1) * cfg.n + (kx - 1)
    ts = np.array([0, 5, 127])
    uh0 = orc.dst_sample(s, u0.real, idx) + 1j * orc.dst_sample(s, u0.imag, idx)
    got = orc.dst_sample_batch(s, Uh[ts].real, idx) + 1j * orc.dst_sample_batch(s, Uh[ts].imag, idx)
    lam = orc.axis_eigs(cfg.n).astype(np.longdouble)
    mu = lam[kx - 1] + lam[ky - 1]
    z = np.longdouble(cfg.dt) * (np.clongdouble(complex(cfg.a, cfg.a_im)) * mu - np.clongdouble(complex(cfg.c, cfg.c_im)))
    for i, t in enumerate(ts):
        want = np.exp(z * (t + 2)) * uh0
        assert np.abs(got[i] - want.astype(np.complex128)).max() < 1e-9 * np.linalg.norm(u0)


# ------------------------------------------------------------------------------------------
# complex plans on the distributed schedule (a 1-rank NCCL communicator: the all-to-alls
# become local copies, the mode / time slab code path runs)
# ------------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def comm1():
    from paper_2603_04350_b200 import Comm

    c = Comm(0, 1, 0)
    yield c
    c.close()


@pytest.mark.parametrize("name,n,nt", [("c6se", 63, 32), ("c7se", 31, 64), ("c7bdf2", 31, 32)])
def test_cplx_dist1_parity(orc, comm1, name, n, nt):
    cfg = cfg_of(name, n, nt)
    s = orc.spec(cfg)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=21, comm=comm1)
    R = synth.random_spacetime(cfg)
    assert relmax(H(plan.precond_apply(TC(R))), orc.cplx_precond(s, R)) < 1e-11
    u0 = synth.initial_condition(cfg)
    U = synth.random_spacetime(cfg, scale=0.5)
    Rg, rn2 = plan.residual(TC(u0), TC(U), norm=True)
    want, wn2 = orc.cplx_residual(s, u0, U)
    assert relmax(H(Rg), want) < 1e-11 and abs(rn2 - wn2) < 1e-11 * wn2
    for solve, ref in ((lambda: plan.fixed_point_solve(TC(u0), tol=cfg.tol, maxit=50),
                        lambda: orc.cplx_fixed_point(s, u0, tol=cfg.tol, maxit=50)),
                       (lambda: plan.gmres_solve(TC(u0), tol=cfg.tol, restart=20, maxit=50),
                        lambda: orc.cplx_gmres(s, u0, tol=cfg.tol, restart=20, maxit=50)),
                       (lambda: plan.bicgstab_solve(TC(u0), tol=cfg.tol, maxit=50),
                        lambda: orc.cplx_bicgstab(s, u0, tol=cfg.tol, maxit=50))):
        Ug, rep = solve()
        Uo, st, its, _ = ref()
        assert st == 0 and rep["converged"] and rep["iterations"] == its
        assert relmax(H(Ug), Uo) < 1e-9


def test_cplx_invalid_problems():
    base = dict(dim=1, n=15, a=0.0, c=0.0, dt=0.01, nt=8, alpha=1e-2, a_im=1.0, c_im=2.0)
    with pytest.raises(ExpdError) as e:  # nonlinear complex: not built
        Plan(Problem(**{**base, "q": (0.0, 1.0)}))
    assert e.value.status == 2
    with pytest.raises(ExpdError) as e:  # Re a < 0: ill-posed
        Plan(Problem(**{**base, "a": -0.5}))
    assert e.value.status == 1
    plan = Plan(Problem(**base), krylov_vectors=6)
    with pytest.raises(ValueError):  # a complex plan takes complex128 state
        plan.fixed_point_solve(torch.ones(15, dtype=torch.float64, device=DEV))
