"""GPU parity: the CUDA path (through the C-ABI, libexpd.so) against the CPU oracle.

Tolerances (BASELINE.json:5 north_star):
  * a single preconditioner apply or residual: relative max error <= 1e-11
    (max |gpu - oracle| / max |oracle|, reading R9);
  * solves: identical iteration counts, final solution relative max error <= 1e-9.
Every input is seeded (synth/); every expected value is computed by oracle/ on the same
bytes in the same process.
"""
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


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(DEV)


def H(t):
    return t.detach().cpu().numpy()


def relmax(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def cfg_small(name, n, nt):
    return synth.CONFIGS[name].scaled(n, nt)


# ------------------------------------------------------------------------------------------
# the DST (K2/K3)
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dim,n", [(1, 3), (1, 7), (1, 63), (1, 4095), (2, 7), (2, 15), (2, 63), (2, 255),
                                   (3, 7), (3, 15)])
def test_dst_matches_oracle(orc, dim, n):
    cfg = synth.Config("t", dim, n, 1.0, 1.0, 1.0, 4, 1e-2)
    plan = Plan(Problem.from_config(cfg))
    x = np.random.default_rng(dim * 1000 + n).standard_normal((3,) + cfg.shape)
    got = H(plan.dst(T(x)))
    s = orc.spec(cfg)
    for i in range(3):
        assert relmax(got[i], orc.dst(s, x[i])) < 1e-13


@pytest.mark.parametrize("dim,n", [(2, 2047), (3, 255), (2, 4095)])  # 4095: the largest line
def test_dst_full_size_sampled(orc, dim, n):
    cfg = synth.Config("t", dim, n, 1.0, 1.0, 1.0, 4, 1e-2)
    plan = Plan(Problem.from_config(cfg))
    x = np.random.default_rng(5).standard_normal(cfg.shape)
    got = H(plan.dst(T(x))).reshape(-1)
    idx = np.random.default_rng(6).integers(0, cfg.N, 12)
    want = orc.dst_sample(orc.spec(cfg), x, idx)
    assert relmax(got[idx], want) < 1e-12 * np.sqrt(cfg.N) / np.abs(want).max() + 1e-12


def _tail_idx(cfg, seed, per=3):
    """flat indices whose strided-axis position is in the last thread's rows of the line
    transform (the transposed store writes them with direct global stores): y rows n-17..n-1
    (2-D / 3-D) and, in 3-D, z planes n-17..n-1 too (the z pass)."""
    n, rng = cfg.n, np.random.default_rng(seed)
    tail = np.arange(max(0, n - 17), n)
    out = []
    for y in tail:
        for x in rng.integers(0, n, per):
            if cfg.dim == 2:
                out.append(y * n + x)
            else:
                out.append(rng.integers(0, n) * n * n + y * n + x)  # y tail, any z
                out.append(y * n * n + rng.integers(0, n) * n + x)  # z tail, any y
    return np.array(out)


@pytest.mark.parametrize("dim,n", [(2, 255), (2, 2047), (2, 4095), (3, 255)])
def test_dst_tail_rows_sampled(orc, dim, n):
    """The strided passes' last rows (stored outside the transposed TMA box) at every line
    length class the bench and the fuzz use: sampled DST outputs against the oracle."""
    cfg = synth.Config("t", dim, n, 1.0, 1.0, 1.0, 4, 1e-2)
    plan = Plan(Problem.from_config(cfg))
    x = np.random.default_rng(15).standard_normal(cfg.shape)
    got = H(plan.dst(T(x))).reshape(-1)
    idx = _tail_idx(cfg, 16)
    want = orc.dst_sample(orc.spec(cfg), x, idx)
    assert relmax(got[idx], want) < 1e-12 * np.sqrt(cfg.N) / np.abs(want).max() + 1e-12


def test_nonlin_hat_tail_rows_sampled(orc):
    """The fused [V, N, V] pass's last rows at c5's slice size (2047^2)."""
    cfg = synth.CONFIGS["c5"].scaled(2047, 4)
    plan = Plan(Problem.from_config(cfg))
    s = orc.spec(cfg)
    uh = np.random.default_rng(65).standard_normal((1,) + cfg.shape) / np.sqrt(cfg.N)
    got = H(plan.nonlin_hat(T(uh))).reshape(-1)
    idx = _tail_idx(cfg, 66)
    want = orc.dst_sample(s, orc.nonlin(s, orc.dst(s, uh[0])), idx)
    assert np.abs(got[idx] - want).max() < 1e-12 * np.abs(got).max()


# ------------------------------------------------------------------------------------------
# stage 3: N-hat = V N(V u-hat) (K4; the TMA line kernels for n+1 >= 256)
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dim,n,ns", [(2, 31, 3), (2, 255, 3), (2, 511, 2), (3, 255, 1), (2, 1023, 1)])
def test_nonlin_hat_parity(orc, dim, n, ns):
    cfg = synth.Config("t", dim, n, 1.0, 1.0, 1.0, 8, 1e-2, q=(0.0, 0.0, 0.0, -1.0), scheme=1)
    plan = Plan(Problem.from_config(cfg))
    s = orc.spec(cfg)
    uh = np.random.default_rng(dim * 7 + n).standard_normal((ns,) + cfg.shape) / np.sqrt(cfg.N)
    got = H(plan.nonlin_hat(T(uh)))
    for i in range(ns):
        want = orc.dst(s, orc.nonlin(s, orc.dst(s, uh[i])))
        assert relmax(got[i], want) < 1e-12


def test_nonlin_hat_full_size_sampled(orc):
    # c5's slice (2047^2): the full-size launch configuration of the sweep's stage 3
    cfg = synth.CONFIGS["c5"].scaled(2047, 4)
    plan = Plan(Problem.from_config(cfg))
    s = orc.spec(cfg)
    uh = np.random.default_rng(55).standard_normal((2,) + cfg.shape) / np.sqrt(cfg.N)
    got = H(plan.nonlin_hat(T(uh))).reshape(2, -1)
    idx = np.random.default_rng(56).integers(0, cfg.N, 24)
    for i in range(2):
        want = orc.dst_sample(s, orc.nonlin(s, orc.dst(s, uh[i])), idx)
        assert np.abs(got[i][idx] - want).max() < 1e-12 * np.abs(got[i]).max()


def test_sweep_full_size_sampled(orc):
    # one fused sweep (K1: residual + preconditioner + update) at c5's full size and launch
    # configuration (linear variant of c5: stage 3 is checked separately above), compared at
    # sampled modes with the oracle's per-mode residual and Steps (a)-(c); the DST
    # coefficients of input and output are taken by the oracle's plain sums
    cfg = synth.Config("c5lin", 2, 2047, 0.1, 0.5, 1.0, 256, 1e-3, scheme=1, seed=5)
    s = orc.spec(cfg)
    u0 = synth.initial_condition(synth.CONFIGS["c5"])
    U, ks = synth.sparse_spacetime(cfg, nmodes=6)
    plan = Plan(Problem.from_config(cfg))
    plan.load_state(T(u0), T(U))
    plan.sweep()
    rn2 = plan.sweep_norm2()
    Ud = torch.empty((cfg.nt,) + cfg.shape, dtype=torch.float64, device=DEV)
    plan.store_state(Ud)
    U2 = H(Ud)
    del Ud, plan
    n = cfg.n
    J = [int((k[1] - 1) * n + (k[0] - 1)) for k in ks[:3]] + [5 * n + 7]  # 3 active modes + 1 inactive
    uh0 = orc.dst_sample(s, u0, J)
    uh = orc.dst_sample_batch(s, U, J)     # [nt][modes]
    uh2 = orc.dst_sample_batch(s, U2, J)
    scale = np.abs(uh).max()
    for m, j in enumerate(J):
        r = orc.mode_residual(s, j, uh[:, m], uh0[m])
        want = uh[:, m] + orc.mode_precond(s, j, r)
        assert np.abs(uh2[:, m] - want).max() < 1e-11 * scale, j
    assert np.isfinite(rn2) and rn2 > 0


# ------------------------------------------------------------------------------------------
# preconditioner apply (Steps (a)-(c)) and residual
# ------------------------------------------------------------------------------------------
PRECOND_CASES = [
    ("c1bdf2", None, None), ("c2bdf2", 31, 64),  # NEXT-2: BDF2 divisor
    ("c1", None, None),
    ("c2", 31, 64),
    ("c3", 31, 128),
    ("c4", 7, 64),
    ("c5", 31, 256),
    ("c2", 7, 4),
    ("c2", 7, 8),
    ("c2", 15, 16),
    ("c2", 3, 32),
]


@pytest.mark.parametrize("name,n,nt", PRECOND_CASES)
def test_precond_apply_parity(orc, name, n, nt):
    cfg = synth.CONFIGS[name] if n is None else cfg_small(name, n, nt)
    plan = Plan(Problem.from_config(cfg))
    R = synth.random_spacetime(cfg)
    S = H(plan.precond_apply(T(R)))
    want, leak = orc.precond(orc.spec(cfg), R)
    assert leak < 1e-8
    assert relmax(S, want) < 1e-11


@pytest.mark.parametrize("name,n,nt", [("c1", None, None), ("c2", 31, 64), ("c3", 31, 128), ("c4", 7, 64),
                                       ("c5", 31, 256), ("c5", 7, 4), ("c5if", 31, 256), ("c3if", 255, 8),
                                       ("c1bdf2", None, None), ("c2bdf2", 31, 64)])
def test_residual_parity(orc, name, n, nt):
    cfg = synth.CONFIGS[name] if n is None else cfg_small(name, n, nt)
    plan = Plan(Problem.from_config(cfg))
    u0 = synth.initial_condition(cfg)
    U = synth.random_spacetime(cfg, scale=0.5)
    R, rn2 = plan.residual(T(u0), T(U), norm=True)
    want, wn2 = orc.residual(orc.spec(cfg), u0, U)
    assert relmax(H(R), want) < 1e-11
    assert abs(rn2 - wn2) < 1e-11 * wn2


def test_precond_zero_and_alias(orc):
    cfg = cfg_small("c2", 15, 32)
    plan = Plan(Problem.from_config(cfg))
    Z = torch.zeros((cfg.nt,) + cfg.shape, dtype=torch.float64, device=DEV)
    assert float(plan.precond_apply(Z).abs().max()) == 0.0
    R = synth.random_spacetime(cfg)
    Rt = T(R)
    plan.precond_apply(Rt, Rt)  # S may alias R
    want, _ = orc.precond(orc.spec(cfg), R)
    assert relmax(H(Rt), want) < 1e-11


# ------------------------------------------------------------------------------------------
# solvers
# ------------------------------------------------------------------------------------------
SOLVE_CASES = [("c1", None, None), ("c2", 63, 64), ("c3", 63, 128), ("c5", 63, 256), ("c4", 15, 64),
               ("c3", 255, 16), ("c5", 255, 16),
               # NEXT-1: IF scheme (6.1) by the IMEX-type iteration (7.2)
               ("c3if", 63, 128), ("c5if", 63, 256), ("c5if", 255, 16),
               # NEXT-2: the BDF2 system (4.2) by Richardson (4.4)
               ("c1bdf2", None, None), ("c2bdf2", 63, 64)]


@pytest.mark.parametrize("name,n,nt", SOLVE_CASES)
def test_fixed_point_parity(orc, name, n, nt):
    cfg = synth.CONFIGS[name] if n is None else cfg_small(name, n, nt)
    plan = Plan(Problem.from_config(cfg))
    u0 = synth.initial_condition(cfg)
    U, rep = plan.fixed_point_solve(T(u0), tol=cfg.tol, maxit=50)
    Uo, st, its, hist = orc.fixed_point(orc.spec(cfg), u0, tol=cfg.tol, maxit=50)
    assert st == 0 and rep["converged"]
    assert rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9
    h = np.array(rep["hist"])
    big = hist > 1e-9  # above the roundoff floor the histories agree closely
    assert np.allclose(h[big], hist[big], rtol=1e-6)


@pytest.mark.parametrize("k1v", ["5124", "5123"])
@pytest.mark.parametrize("name,n,nt", [("c5", 63, 256), ("c5if", 63, 256), ("c3", 63, 256)])
def test_k1_nt256_picard_variants_match_oracle(orc, name, n, nt, k1v, monkeypatch):
    """Both K1 kernels of the Nt = 256 Picard forms (ETD2, IF/IMEX, ETD1):
    the warp-per-pair kernel (5124, the default) and the ring (5123): the oracle's iterations,
    history and solution."""
    monkeypatch.setenv("EXPD_K1V", k1v)
    test_fixed_point_parity(orc, name, n, nt)


@pytest.mark.parametrize("name,n,nt", [("c1", None, None), ("c2", 63, 64), ("c4", 15, 64), ("c1bdf2", None, None),
                                       ("c2bdf2", 63, 64)])
def test_gmres_parity(orc, name, n, nt):
    cfg = synth.CONFIGS[name] if n is None else cfg_small(name, n, nt)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=21)
    u0 = synth.initial_condition(cfg)
    U, rep = plan.gmres_solve(T(u0), tol=cfg.tol, restart=20, maxit=50)
    Uo, st, its, hist = orc.gmres(orc.spec(cfg), u0, tol=cfg.tol, restart=20, maxit=50)
    assert st == 0 and rep["converged"]
    assert rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9


@pytest.mark.parametrize("name,n,nt", [("c1", None, None), ("c2", 63, 64), ("c4", 15, 64), ("c2bdf2", 63, 64)])
def test_bicgstab_parity(orc, name, n, nt):
    cfg = synth.CONFIGS[name] if n is None else cfg_small(name, n, nt)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=6)
    u0 = synth.initial_condition(cfg)
    U, rep = plan.bicgstab_solve(T(u0), tol=cfg.tol, maxit=50)
    Uo, st, its, hist = orc.bicgstab(orc.spec(cfg), u0, tol=cfg.tol, maxit=50)
    assert st == 0 and rep["converged"]
    assert rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9


def test_bicgstab_slow_convergence_matches_oracle(orc):
    # alpha = 0.2 on a slowly decaying problem: several BiCGStab steps
    cfg = synth.Config("b", 1, 15, 0.05, 0.0, 0.5, 16, 0.2)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=6)
    u0 = np.random.default_rng(3).standard_normal(15)
    U, rep = plan.bicgstab_solve(T(u0), tol=1e-12, maxit=60)
    Uo, st, its, hist = orc.bicgstab(orc.spec(cfg), u0, tol=1e-12, maxit=60)
    assert rep["iterations"] == its and its >= 3
    h = np.array(rep["hist"])
    assert np.allclose(h[hist > 1e-9], hist[hist > 1e-9], rtol=1e-6)
    assert relmax(H(U), Uo) < 1e-9


def test_gmres_small_restart_matches_oracle(orc):
    cfg = synth.Config("g", 1, 15, 0.05, 0.0, 0.5, 16, 0.2)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=3)
    u0 = np.random.default_rng(3).standard_normal(15)
    U, rep = plan.gmres_solve(T(u0), tol=1e-12, restart=3, maxit=60)
    Uo, st, its, hist = orc.gmres(orc.spec(cfg), u0, tol=1e-12, restart=3, maxit=60)
    assert rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9


# ------------------------------------------------------------------------------------------
# argument validation (synchronous, before any launch)
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("kw,status", [({"alpha": 0.0}, 1), ({"nt": 12}, 1), ({"n": 10}, 1), ({"nt": 512}, 2),
                                       ({"a": -1.0}, 1), ({"dim": 4}, 1)])
def test_invalid_problems(kw, status):
    base = dict(dim=2, n=15, a=1.0, c=1.0, dt=0.1, nt=16, alpha=1e-2)
    base.update(kw)
    with pytest.raises(ExpdError) as ei:
        Plan(Problem(**base))
    assert ei.value.status == status


# ------------------------------------------------------------------------------------------
# the distributed schedule on one GPU: a real NCCL communicator of one rank,
# mode-slab K1, time-slab stage 3, all-to-alls (here local copies) and allreduces
# ------------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def comm1():
    from paper_2603_04350_b200 import Comm

    c = Comm(0, 1, 0)
    yield c
    c.close()


@pytest.mark.parametrize("name,n,nt", [("c1", None, None), ("c3", 63, 128), ("c5", 63, 256), ("c2", 63, 64),
                                       ("c5", 255, 16), ("c3if", 63, 128), ("c5if", 255, 16)])
def test_dist1_fixed_point_parity(orc, comm1, name, n, nt):
    cfg = synth.CONFIGS[name] if n is None else cfg_small(name, n, nt)
    plan = Plan(Problem.from_config(cfg), comm=comm1)
    u0 = synth.initial_condition(cfg)
    U, rep = plan.fixed_point_solve(T(u0), tol=cfg.tol, maxit=50)
    Uo, st, its, hist = orc.fixed_point(orc.spec(cfg), u0, tol=cfg.tol, maxit=50)
    assert st == 0 and rep["converged"] and rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9


@pytest.mark.parametrize("name,n,nt", [("c2", 63, 64), ("c4", 15, 64), ("c2bdf2", 63, 64)])
def test_dist1_bicgstab_parity(orc, comm1, name, n, nt):
    cfg = cfg_small(name, n, nt)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=6, comm=comm1)
    u0 = synth.initial_condition(cfg)
    U, rep = plan.bicgstab_solve(T(u0), tol=cfg.tol, maxit=50)
    Uo, st, its, hist = orc.bicgstab(orc.spec(cfg), u0, tol=cfg.tol, maxit=50)
    assert st == 0 and rep["converged"] and rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9


@pytest.mark.parametrize("name,n,nt", [("c2", 63, 64), ("c4", 15, 64), ("c2bdf2", 63, 64)])
def test_dist1_gmres_parity(orc, comm1, name, n, nt):
    cfg = cfg_small(name, n, nt)
    plan = Plan(Problem.from_config(cfg), krylov_vectors=21, comm=comm1)
    u0 = synth.initial_condition(cfg)
    U, rep = plan.gmres_solve(T(u0), tol=cfg.tol, restart=20, maxit=50)
    Uo, st, its, hist = orc.gmres(orc.spec(cfg), u0, tol=cfg.tol, restart=20, maxit=50)
    assert st == 0 and rep["converged"] and rep["iterations"] == its
    assert relmax(H(U), Uo) < 1e-9


@pytest.mark.parametrize("name,n,nt", [("c5", 31, 256), ("c3", 255, 8)])
def test_dist1_primitives_parity(orc, comm1, name, n, nt):
    cfg = cfg_small(name, n, nt)
    plan = Plan(Problem.from_config(cfg), comm=comm1)
    s = orc.spec(cfg)
    R = synth.random_spacetime(cfg)
    want, _ = orc.precond(s, R)
    assert relmax(H(plan.precond_apply(T(R))), want) < 1e-11
    u0 = synth.initial_condition(cfg)
    U = synth.random_spacetime(cfg, scale=0.5)
    Rg, rn2 = plan.residual(T(u0), T(U), norm=True)
    want, wn2 = orc.residual(s, u0, U)
    assert relmax(H(Rg), want) < 1e-11
    assert abs(rn2 - wn2) < 1e-11 * wn2


def test_dist1_matches_single_gpu_schedule(comm1):
    # same problem through both schedules: the same kernels on the same modes, so the
    # solutions agree to rounding (only the all-to-all copies and the stage-3 chunking differ)
    cfg = cfg_small("c5", 255, 16)
    u0 = T(synth.initial_condition(cfg))
    U1, r1 = Plan(Problem.from_config(cfg)).fixed_point_solve(u0, tol=cfg.tol, maxit=50)
    U2, r2 = Plan(Problem.from_config(cfg), comm=comm1).fixed_point_solve(u0, tol=cfg.tol, maxit=50)
    assert r1["iterations"] == r2["iterations"]
    assert relmax(H(U2), H(U1)) < 1e-13


def test_dist1_uneven_pipeline_chunks(tmp_path):
    """The pipelined exchange with chunks that do not divide the time slab (EXPD_DIST_CHUNKS
    = 3 over 8 slices: 3 + 3 + 2), in a fresh process (the setting is read once)."""
    import subprocess
    import sys

    code = """
import sys; sys.path.insert(0, '.')
import numpy as np, torch, synth, oracle
from paper_2603_04350_b200 import Comm, Plan, Problem
cfg = synth.CONFIGS['c5'].scaled(63, 8)
comm = Comm(0, 1, 0)
plan = Plan(Problem.from_config(cfg), comm=comm)
u0 = synth.initial_condition(cfg)
U, rep = plan.fixed_point_solve(torch.from_numpy(u0).cuda(), tol=cfg.tol, maxit=50)
Uo, st, its, _ = oracle.fixed_point(oracle.spec(cfg), u0, tol=cfg.tol, maxit=50)
err = np.abs(U.cpu().numpy() - Uo).max() / np.abs(Uo).max()
assert rep['converged'] and rep['iterations'] == its and err < 1e-9, (rep['iterations'], its, err)
print('ok', its, err)
"""
    import os

    env = dict(os.environ, EXPD_DIST_CHUNKS="3")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("name,n,nt", [("c1", None, None), ("c2", 63, 64), ("c5", 255, 16), ("c3if", 63, 128)])
def test_device_loop_matches_host_loop(orc, name, n, nt, monkeypatch):
    """The fixed-point / Picard solve's device-side loop (CUDA-graph WHILE node, one host sync)
    takes the same iterations, history and solution as the host-driven loop and the oracle."""
    cfg = synth.CONFIGS[name] if n is None else cfg_small(name, n, nt)
    u0 = synth.initial_condition(cfg)
    plan = Plan(Problem.from_config(cfg))
    Ud, rd = plan.fixed_point_solve(T(u0), tol=cfg.tol, maxit=50)
    Ud2, rd2 = plan.fixed_point_solve(T(u0), tol=cfg.tol, maxit=50)  # the graph is reused
    monkeypatch.setenv("EXPD_DEVICE_LOOP", "0")
    Uh, rh = plan.fixed_point_solve(T(u0), tol=cfg.tol, maxit=50)
    Uo, st, its, hist = orc.fixed_point(orc.spec(cfg), u0, tol=cfg.tol, maxit=50)
    assert rd["converged"] and rh["converged"] and rd["iterations"] == rh["iterations"] == its
    assert rd["sweeps"] == rh["sweeps"] == its + 1
    assert rd["hist"] == rh["hist"] == rd2["hist"]  # the same kernels in the same order: bitwise
    assert float((Ud - Uh).abs().max()) == 0.0 and float((Ud2 - Uh).abs().max()) == 0.0
    assert relmax(H(Ud), Uo) < 1e-9


def test_device_loop_not_converged_and_maxit(orc):
    cfg = cfg_small("c5", 63, 32)
    plan = Plan(Problem.from_config(cfg))
    u0 = T(synth.initial_condition(cfg))
    U, rep = plan.fixed_point_solve(u0, tol=1e-30, maxit=3)
    assert rep["status"] == "EXPD_ERR_NOT_CONVERGED" and not rep["converged"]
    assert rep["iterations"] == 3 and rep["sweeps"] == 4 and len(rep["hist"]) == 4
    U0, rep0 = plan.fixed_point_solve(u0, tol=1e-30, maxit=0)
    assert rep0["sweeps"] == 1 and len(rep0["hist"]) == 1


@pytest.mark.parametrize("env", [{"EXPD_LINE2": "1"}, {"EXPD_S3P": "1"}, {"EXPD_S3P": "1", "EXPD_S3P_K": "2"},
                                 {"EXPD_K1V": "2562"}])
def test_opt_in_variants_match_default(orc, env, monkeypatch):
    """The measured-and-kept-opt-in kernel variants (k_line2, the
    persistent stage 3 with rings of 4 and 2 slices, the previous K1 default) give the default
    path's Picard iterations and solution at n + 1 = 2048 (their launch size), and k_line2's
    stage 3 matches the oracle at sampled modes."""
    cfg = synth.CONFIGS["c5"].scaled(2047, 8)
    u0 = T(synth.initial_condition(cfg))
    plan = Plan(Problem.from_config(cfg))
    Ud, rd = plan.fixed_point_solve(u0, tol=1e-12, maxit=30)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    plan2 = Plan(Problem.from_config(cfg))
    Uv, rv = plan2.fixed_point_solve(u0, tol=1e-12, maxit=30)
    assert rd["converged"] and rv["converged"] and rv["iterations"] == rd["iterations"]
    assert relmax(H(Uv), H(Ud)) < 1e-12
    if "EXPD_LINE2" in env:
        s = orc.spec(cfg)
        uh = np.random.default_rng(57).standard_normal((1,) + cfg.shape) / np.sqrt(cfg.N)
        got = H(plan2.nonlin_hat(T(uh))).reshape(1, -1)
        idx = np.random.default_rng(58).integers(0, cfg.N, 16)
        want = orc.dst_sample(s, orc.nonlin(s, orc.dst(s, uh[0])), idx)
        assert np.abs(got[0][idx] - want).max() < 1e-12 * np.abs(got[0]).max()


@pytest.mark.parametrize("env", [{"EXPD_COLV": "13", "EXPD_ROWV": "3"}, {"EXPD_COLV": "11", "EXPD_ROWV": "1"},
                                 {"EXPD_COLV": "22"}, {"EXPD_COLTS": "0"}, {"EXPD_LINE_HY": "0"}])
def test_line_launch_variants_match_oracle(tmp_path, env):
    """The line kernels' launch variants read once per process (EXPD_COLV / EXPD_ROWV: the
    ping-pong buffers, one buffer per CTA, two column pairs per item; EXPD_COLTS=0: the
    strided-axis result compacted and stored in boxes of 256 rows instead of the transposed
    store; EXPD_LINE_HY=0: the in-place buffer schedule instead of the hybrid one), each in a
    fresh process:
    the c5 Picard solve at n + 1 = 2048 takes the oracle's iterations, and stage 3 matches the
    oracle at sampled modes."""
    import os
    import subprocess
    import sys

    code = """
import sys; sys.path.insert(0, '.')
import numpy as np, torch, synth, oracle
from paper_2603_04350_b200 import Plan, Problem
cfg = synth.CONFIGS['c5'].scaled(2047, 4)
s = oracle.spec(cfg)
plan = Plan(Problem.from_config(cfg))
uh = np.random.default_rng(57).standard_normal((1,) + cfg.shape) / np.sqrt(cfg.N)
got = plan.nonlin_hat(torch.from_numpy(uh).cuda()).cpu().numpy().reshape(1, -1)
idx = np.random.default_rng(58).integers(0, cfg.N, 16)
want = oracle.dst_sample(s, oracle.nonlin(s, oracle.dst(s, uh[0])), idx)
err = np.abs(got[0][idx] - want).max() / np.abs(got[0]).max()
assert err < 1e-12, err
small = synth.CONFIGS['c5'].scaled(255, 8)
p2 = Plan(Problem.from_config(small))
u0 = synth.initial_condition(small)
U, rep = p2.fixed_point_solve(torch.from_numpy(u0).cuda(), tol=small.tol, maxit=50)
Uo, st, its, _ = oracle.fixed_point(oracle.spec(small), u0, tol=small.tol, maxit=50)
e2 = np.abs(U.cpu().numpy() - Uo).max() / np.abs(Uo).max()
assert rep['converged'] and rep['iterations'] == its and e2 < 1e-9, (rep['iterations'], its, e2)
print('ok', err, e2)
"""
    full_env = dict(os.environ, **env)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=full_env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
