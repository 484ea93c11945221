"""Edge cases of the CUDA path against the oracle and the C-ABI's documented behaviour:
empty inputs, the zero problem, the largest alpha, the smallest grids and time windows, and
the binding's argument checks."""
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


def test_empty_slices_leave_output_untouched():
    cfg = synth.CONFIGS["c5"].scaled(63, 4)
    plan = Plan(Problem.from_config(cfg))
    x = torch.empty((0,) + cfg.shape, dtype=torch.float64, device=DEV)
    assert plan.dst(x).numel() == 0 and plan.nonlin_hat(x).numel() == 0


@pytest.mark.parametrize("name,n,nt", [("c2", 31, 16), ("c5", 63, 8)])
def test_zero_problem(orc, name, n, nt):
    """u0 = 0: F(0) = 0, so r^0 = 0; both the oracle and the GPU stop at once (rho := 0 when
    ||r^0|| = 0, reading R8) with U = 0."""
    cfg = synth.CONFIGS[name].scaled(n, nt)
    u0 = np.zeros(cfg.shape)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=4)
    U, rep = plan.fixed_point_solve(T(u0), tol=1e-12)
    Uo, st, its, hist = orc.fixed_point(orc.spec(cfg), u0, tol=1e-12)
    assert st == 0 and rep["converged"] and rep["iterations"] == its == 0
    assert float(U.abs().max()) == 0.0
    if not cfg.q:
        U, rep = plan.gmres_solve(T(u0), tol=1e-12, restart=3)
        assert rep["converged"] and rep["iterations"] == 0 and float(U.abs().max()) == 0.0


@pytest.mark.parametrize("dim,n,nt", [(1, 3, 4), (2, 3, 4), (3, 3, 4), (1, 7, 256)])
def test_alpha_one_and_smallest_grids(orc, dim, n, nt):
    """alpha = 1 (the largest the ABI takes: the periodic, circulant preconditioner, cond = 1)
    on the smallest grids (n + 1 = 4) and windows (Nt = 4)."""
    cfg = synth.Config("e", dim, n, 0.5, 0.3, 0.5, nt, 1.0)
    plan = Plan(Problem.from_config(cfg))
    R = synth.random_spacetime(cfg, seed=7)
    want, leak = orc.precond(orc.spec(cfg), R)
    assert leak < 1e-8 and relmax(H(plan.precond_apply(T(R))), want) < 1e-11
    u0 = synth.random_slice(cfg, 8)
    U = synth.random_spacetime(cfg, seed=9)
    Rg, rn2 = plan.residual(T(u0), T(U), norm=True)
    wr, wn2 = orc.residual(orc.spec(cfg), u0, U)
    assert relmax(H(Rg), wr) < 1e-11 and abs(rn2 - wn2) < 1e-11 * wn2


def test_binding_rejects_wrong_shapes_and_devices():
    cfg = synth.CONFIGS["c2"].scaled(15, 8)
    plan = Plan(Problem.from_config(cfg))
    u0 = torch.zeros(cfg.shape, dtype=torch.float64, device=DEV)
    with pytest.raises(ValueError):
        plan.fixed_point_solve(u0, torch.zeros((cfg.nt - 1,) + cfg.shape, dtype=torch.float64, device=DEV))
    with pytest.raises(ValueError):
        plan.fixed_point_solve(torch.zeros(cfg.N + 1, dtype=torch.float64, device=DEV))
    with pytest.raises(ValueError):
        plan.precond_apply(torch.zeros((cfg.nt,) + cfg.shape, dtype=torch.float64))  # host tensor
    with pytest.raises(ValueError):
        plan.precond_apply(torch.zeros((cfg.nt,) + cfg.shape, dtype=torch.float32, device=DEV))
    with pytest.raises(ValueError):
        plan.dst(torch.zeros(cfg.N + 3, dtype=torch.float64, device=DEV))


@pytest.mark.parametrize("name,n,nt,solver", [("c5", 63, 16, "fixed_point"), ("c2", 31, 16, "gmres"),
                                              ("c2", 31, 16, "bicgstab"), ("c7se", 31, 16, "gmres")])
def test_host_buffers_and_zero_guess(orc, name, n, nt, solver):
    """The solvers with host u0 / U (pinned and pageable): the library copies in and streams the
    solution out chunk by chunk; results identical to the device-buffer call.  With the zero
    guess set, garbage in U on entry is ignored."""
    cfg = synth.CONFIGS[name].scaled(n, nt)
    prob = Problem.from_config(cfg)
    plan = Plan(prob, krylov_vectors=6)
    u0 = torch.from_numpy(np.asarray(synth.initial_condition(cfg))).to(prob.dtype)
    kw = {"gmres": dict(restart=5)}.get(solver, {})
    solve = getattr(plan, solver + "_solve")
    Ud, rd = solve(u0.to(DEV), torch.zeros((cfg.nt,) + cfg.shape, dtype=prob.dtype, device=DEV), tol=cfg.tol, **kw)
    for pin in (True, False):
        Uh = torch.zeros((cfg.nt,) + cfg.shape, dtype=prob.dtype)
        u0h = u0.clone()
        if pin:
            Uh, u0h = Uh.pin_memory(), u0h.pin_memory()
        Uh2, rh = solve(u0h, Uh, tol=cfg.tol, **kw)
        assert Uh2.device.type == "cpu" and rh["iterations"] == rd["iterations"]
        assert float((Uh2 - Ud.cpu()).abs().max()) == 0.0
    plan.set_zero_guess(True)
    garbage = torch.full((cfg.nt,) + cfg.shape, 1e30, dtype=prob.dtype, device=DEV)
    Uz, rz = solve(u0.to(DEV), garbage, tol=cfg.tol, **kw)
    assert rz["iterations"] == rd["iterations"] and float((Uz - Ud).abs().max()) == 0.0


def test_gmres_restart_beyond_workspace_is_an_error():
    from paper_2603_04350_b200 import ExpdError

    cfg = synth.CONFIGS["c2"].scaled(15, 8)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=3)
    u0 = torch.from_numpy(synth.initial_condition(cfg)).to(DEV)
    with pytest.raises(ExpdError):
        plan.gmres_solve(u0, tol=1e-12, restart=4)
    U, rep = plan.gmres_solve(u0, tol=1e-12, restart=3)
    assert rep["converged"]


@pytest.mark.parametrize("name,n,nt,scheme_note", [("c5", 255, 16, "ETD2"), ("c3", 127, 32, "ETD1"),
                                                   ("c5if", 127, 16, "IF / IMEX"), ("c5", 63, 256, "Nt = 256")])
@pytest.mark.parametrize("device_loop", ["1", "0"])
def test_zero_guess_first_sweep_skips_stage3_bitwise(orc, monkeypatch, name, n, nt, scheme_note, device_loop):
    """From the zero guess with N(0) = 0 the first sweep's stage 3 is skipped (N-hat = V N(0) =
    0 exactly): the iterates, the history and the solution are bitwise those of the full first
    sweep (EXPD_S3_SKIP0=0), on the device loop and on the host loop, and match the oracle."""
    monkeypatch.setenv("EXPD_DEVICE_LOOP", device_loop)
    cfg = synth.CONFIGS[name].scaled(n, nt)
    plan = Plan(Problem.from_config(cfg))
    plan.set_zero_guess(True)
    u0 = T(synth.initial_condition(cfg))
    U1, r1 = plan.fixed_point_solve(u0, tol=cfg.tol, maxit=50)
    monkeypatch.setenv("EXPD_S3_SKIP0", "0")
    U2, r2 = plan.fixed_point_solve(u0, tol=cfg.tol, maxit=50)
    assert r1["iterations"] == r2["iterations"] and r1["hist"] == r2["hist"]
    assert torch.equal(U1, U2)
    Uo, st, its, _ = orc.fixed_point(orc.spec(cfg), synth.initial_condition(cfg), tol=cfg.tol, maxit=50)
    assert st == 0 and r1["iterations"] == its and relmax(H(U1), Uo) < 1e-9


def test_nonzero_constant_term_does_not_skip(orc):
    """N(0) = q0 != 0: the first sweep's N-hat is not zero, so nothing is skipped (matches the
    oracle)."""
    cfg = synth.Config("q0", 2, 63, 0.5, 1.0, 0.2, 8, 0.05, scheme=1, q=(0.3, 0.0, 0.0, -1.0))
    plan = Plan(Problem.from_config(cfg))
    plan.set_zero_guess(True)
    u0 = synth.initial_condition(synth.CONFIGS["c5"].scaled(63, 8))
    U, rep = plan.fixed_point_solve(T(u0), tol=1e-12, maxit=60)
    Uo, st, its, _ = orc.fixed_point(orc.spec(cfg), u0, tol=1e-12, maxit=60)
    assert st == 0 and rep["iterations"] == its and relmax(H(U), Uo) < 1e-9
