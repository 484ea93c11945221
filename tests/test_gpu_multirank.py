"""The distributed plan with 2 and 4 ranks on the GPU.

NCCL refuses two ranks on one device and this pool gives one GPU, so the ranks here are
processes sharing cuda:0 whose plans exchange through a HOST communicator
(expd_host_comm_create over torch.distributed gloo): the same mode-slab K1, time-slab stage 3,
pipelined all-to-all schedule (message lists, chunking, self pairing) and allreduces as on
NVLink, with every exchange staged through host memory.  No rank's kernel waits on another's
-- the hosts move the data between the launches.  Each rank returns its time slab; the
concatenation is compared with the oracle: the preconditioner apply and the residual at
1e-11, the solvers with identical iteration counts and solutions within 1e-9.

The shapes keep the solution well above round-off of u0 (at n = 31, nt = 8 the linear c2
problems decay to 1e-19 of u0 within one step, where a relative comparison means nothing).
The uneven mode splits are the point: n odd and P a power of two, so the x-line units never
divide evenly (31 lines over 2 ranks: 16 + 15), incl. the complex 2D case whose staging
buffers once overflowed on ranks with the short slab.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from test_dist_cpu import GlooTransport, _cfg, _init, _spawn  # noqa: E402

SOLVERS = {"fixed_point": {}, "gmres": {"restart": 20}, "bicgstab": {}}


def _worker(rank, P, port, name, n, nt, solvers, out_dir):
    _init(rank, P, port)
    try:
        from paper_2603_04350_b200 import HostComm, Plan, Problem

        torch.cuda.set_device(0)
        dev = torch.device("cuda:0")
        cfg = _cfg(name, n, nt)
        prob = Problem.from_config(cfg)
        comm = HostComm(rank, P, 0, GlooTransport())
        plan = Plan(prob, krylov_vectors=21, comm=comm)
        t0, ntl = plan.layout["t0"], plan.layout["nt_local"]

        def T(x):
            return torch.from_numpy(np.ascontiguousarray(x)).to(dev)

        out = {}
        R = synth.random_spacetime(cfg)
        out["S"] = plan.precond_apply(T(R[t0:t0 + ntl])).cpu().numpy()
        u0 = synth.initial_condition(cfg)
        U = synth.random_spacetime(cfg, scale=0.5)
        Rg, rn2 = plan.residual(T(u0), T(U[t0:t0 + ntl]), norm=True)
        out["R"], out["rn2"] = Rg.cpu().numpy(), np.array(rn2)
        for sv in solvers:
            Us, rep = getattr(plan, sv + "_solve")(T(u0), tol=cfg.tol, maxit=50, **SOLVERS[sv])
            out["U_" + sv] = Us.cpu().numpy()
            out["its_" + sv] = np.array([rep["iterations"], int(rep["converged"])])
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
        del plan
        comm.close()
    finally:
        dist.destroy_process_group()


def relmax(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


@pytest.mark.parametrize("P,name,n,nt,solvers", [
    (2, "c7se", 31, 8, ("fixed_point", "gmres", "bicgstab")),  # complex 2D, 16 + 15 x-lines
    (2, "c5", 63, 8, ("fixed_point",)),                         # ETD2 Picard: stage 3 on time slabs
    (2, "c5", 63, 256, ("fixed_point",)),                       # Nt = 256: the warp-per-pair K1 on mode slabs
    (2, "c2bdf2", 63, 64, ("fixed_point", "gmres")),            # exponential BDF2 (NEXT-2)
    (2, "c2", 63, 64, ("bicgstab",)),                           # real BiCGStab (NEXT-4)
    (2, "c5if", 31, 8, ("fixed_point",)),                       # IMEX-type iteration (NEXT-1)
    (4, "c5", 31, 8, ("fixed_point",)),                         # 4 ranks: 8 + 8 + 8 + 7 lines
    (4, "c4", 15, 64, ("gmres",)),                              # 3D GMRES over 4 mode slabs
    (2, "c1", None, None, ("fixed_point", "gmres")),            # 1D: mode pairs, not x-lines
])
def test_multirank_parity(orc, tmp_path, P, name, n, nt, solvers):
    _spawn(_worker, P, name, n, nt, solvers, str(tmp_path))
    _check(orc, tmp_path, P, name, n, nt, solvers)


@pytest.mark.parametrize("chunks", ["3", "1", "64"])
def test_multirank_pipeline_chunks(orc, tmp_path, monkeypatch, chunks):
    """The pipelined exchange of stage 3 with key ranges that do not divide the time slab
    (3 over 8 slices: 3 + 3 + 2), one range, and more ranges than slices (read by the
    spawned ranks from the environment)."""
    monkeypatch.setenv("EXPD_DIST_CHUNKS", chunks)
    _spawn(_worker, 2, "c5", 31, 16, ("fixed_point",), str(tmp_path))
    _check(orc, tmp_path, 2, "c5", 31, 16, ("fixed_point",))


def _check(orc, tmp_path, P, name, n, nt, solvers):
    cfg = _cfg(name, n, nt)
    s = orc.spec(cfg)
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(P)]
    cat = lambda key: np.concatenate([g[key] for g in got])  # noqa: E731
    cx = cfg.is_complex
    R = synth.random_spacetime(cfg)
    want = orc.cplx_precond(s, R) if cx else orc.precond(s, R)[0]
    assert relmax(cat("S"), want) < 1e-11
    u0 = synth.initial_condition(cfg)
    U = synth.random_spacetime(cfg, scale=0.5)
    want, wn2 = orc.cplx_residual(s, u0, U) if cx else orc.residual(s, u0, U)
    assert relmax(cat("R"), want) < 1e-11
    for g in got:  # the allreduced norm: the same bits on every rank
        assert float(g["rn2"]) == float(got[0]["rn2"]) and abs(float(g["rn2"]) - wn2) < 1e-11 * wn2
    for sv in solvers:
        kw = SOLVERS[sv]
        ref = getattr(orc, ("cplx_" if cx else "") + sv)
        Uo, st, its, _ = ref(s, u0, tol=cfg.tol, maxit=50, **kw)
        for g in got:
            assert g["its_" + sv][1] == 1 and g["its_" + sv][0] == its, sv
        assert st == 0 and relmax(cat("U_" + sv), Uo) < 1e-9, sv


def _peer_worker(rank, P, port, name, n, nt, out_dir):
    _init(rank, P, port)
    try:
        from paper_2603_04350_b200 import HostComm, Plan, Problem

        torch.cuda.set_device(0)
        dev = torch.device("cuda:0")
        cfg = _cfg(name, n, nt)
        comm = HostComm(rank, P, 0, GlooTransport())
        u0 = torch.from_numpy(np.ascontiguousarray(synth.initial_condition(cfg))).to(dev)
        res = {}
        for peer in (False, True):
            plan = Plan(Problem.from_config(cfg), comm=comm)
            if peer:
                plan.enable_peer_stores()
            t0, ntl = plan.layout["t0"], plan.layout["nt_local"]
            U = torch.from_numpy(np.ascontiguousarray(synth.random_spacetime(cfg, scale=0.5)[t0:t0 + ntl])).to(dev)
            R, rn2 = plan.residual(u0, U, norm=True)
            Us, rep = plan.fixed_point_solve(u0, tol=cfg.tol, maxit=50)
            res[peer] = (R.cpu().numpy(), rn2, Us.cpu().numpy(), rep["iterations"], rep["hist"])
            del plan
        assert np.array_equal(res[False][0], res[True][0]) and res[False][1] == res[True][1]
        assert np.array_equal(res[False][2], res[True][2]) and res[False][3] == res[True][3]
        assert res[False][4] == res[True][4]
        # the stores really go through the registered slabs: peers registered one x-line off
        # (a plan's own slab stays right) give a different solution
        import ctypes as C

        differs = []
        for which in (0, 1):  # 0: the N-hat stores one x-line off, 1: the U-hat loads
            plan = Plan(Problem.from_config(cfg), comm=comm)
            h = (C.c_ubyte * 64)()
            offn, offu = C.c_long(), C.c_long()
            plan._check(plan.lib.expd_plan_slab_ipc_handle(plan.handle, h, C.byref(offn), C.byref(offu)))
            allh = [None] * P
            dist.all_gather_object(allh, (bytes(h), offn.value, offu.value))
            line = 8 * (cfg.n + 1)
            for q, (hb, on, ou) in enumerate(allh):
                if q != rank:
                    on, ou = (on + line, ou) if which == 0 else (on, ou + line)
                plan._check(plan.lib.expd_plan_set_peer_slabs(plan.handle, q, (C.c_ubyte * 64)(*hb), on, ou))
            plan._check(plan.lib.expd_plan_enable_peer_stores(plan.handle, 1))
            Ub, repb = plan.fixed_point_solve(u0, tol=cfg.tol, maxit=50)
            differs.append(not np.array_equal(Ub.cpu().numpy(), res[True][2]))
            del plan
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), U=res[True][2], its=np.array([res[True][3]]),
                 sabotage_differs=np.array(differs))
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P,name,n,nt", [(2, "c5", 255, 8), (4, "c5", 255, 8), (2, "c5if", 255, 8),
                                         (2, "c3", 255, 16)])
def test_multirank_peer_stores(orc, tmp_path, P, name, n, nt):
    """Stage 3 with peer access (each rank's x-IDST rows loaded straight from the owners' U-hat
    slabs and its x-DST rows stored straight into the owners' N-hat slabs, through CUDA IPC --
    here other processes on the same GPU): the residual, the
    iterations, the history and the solution are bitwise those of the all-to-all schedule,
    and the solution matches the oracle (255 x-lines over 2 / 4 ranks: 128 + 127, 64 x 3 + 63)."""
    _spawn(_peer_worker, P, name, n, nt, str(tmp_path))
    cfg = _cfg(name, n, nt)
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(P)]
    U = np.concatenate([g["U"] for g in got])
    Uo, st, its, _ = orc.fixed_point(orc.spec(cfg), synth.initial_condition(cfg), tol=cfg.tol, maxit=50)
    assert st == 0 and all(int(g["its"][0]) == its for g in got)
    assert relmax(U, Uo) < 1e-9
    assert any(bool(g["sabotage_differs"][0]) for g in got) and any(bool(g["sabotage_differs"][1]) for g in got)
