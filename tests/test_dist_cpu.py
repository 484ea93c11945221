"""Multi-GPU host logic on CPU: the mode-slab /
time-slab partition and the all-to-all message schedules that libexpd.so executes with NCCL,
checked here as data and executed by the library's own all-to-all routine (the one the GPU
sweep runs with NCCL) through a host transport over torch.distributed (gloo, world size 2
and 4).

The last test runs the whole distributed Picard / fixed-point schedule of one sweep --
all-to-all U-hat to time slabs, stage 3 on the local slices, all-to-all N-hat back shifted
one slice, the time-local residual + alpha-circulant preconditioner + update on the mode
slab, allreduce of ||r||^2 -- with the oracle's per-slice and per-mode functions as the local
compute and gloo as the network, and compares the result with the single-process oracle
solve: the decomposition (not the kernels) is what is pinned here.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2603_04350_b200 import Problem, a2a_schedule, layout
from paper_2603_04350_b200.expd import a2a_execute_host

CASES = [("c1", None, None), ("c2", 15, 8), ("c3", 31, 16), ("c4", 7, 8), ("c5", 15, 16), ("c5", 2047, 256),
         ("c4", 255, 64)]


def _cfg(name, n, nt):
    return synth.CONFIGS[name] if n is None else synth.CONFIGS[name].scaled(n, nt)


@pytest.mark.parametrize("name,n,nt", CASES)
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_layout_partitions(name, n, nt, P):
    cfg = _cfg(name, n, nt)
    prob = Problem.from_config(cfg)
    if cfg.nt % P:
        pytest.skip("nt % P != 0")
    L = [layout(prob, r, P) for r in range(P)]
    M = cfg.n + 1
    npad = L[0]["npad"]
    assert npad == cfg.n ** (cfg.dim - 1) * M
    unit = M if cfg.dim >= 2 else 2
    off = 0
    for r, l in enumerate(L):
        assert l["mode_off"] == off and l["mode_len"] % unit == 0 and l["mode_len"] > 0
        off += l["mode_len"]
        assert l["t0"] == r * cfg.nt // P and l["nt_local"] == cfg.nt // P
    assert off == npad
    lens = [l["mode_len"] for l in L]
    assert max(lens) - min(lens) <= unit  # balanced to one partition unit


@pytest.mark.parametrize("name,n,nt", CASES[:5])
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("direction,shift", [(0, 0), (1, 0), (1, 1)])
def test_schedules_match_and_cover(name, n, nt, P, direction, shift):
    cfg = _cfg(name, n, nt)
    prob = Problem.from_config(cfg)
    if cfg.nt % P:
        pytest.skip("nt % P != 0")
    S = [a2a_schedule(prob, r, P, direction, shift) for r in range(P)]
    L = [layout(prob, r, P) for r in range(P)]
    for r in range(P):
        for q in range(P):
            sent = S[r][0][S[r][0][:, 0] == q][:, 3]
            got = S[q][1][S[q][1][:, 0] == r][:, 3]
            assert list(sent) == list(got), (r, q)
    for q in range(P):
        recv = S[q][1]
        if direction == 0:
            size = L[q]["nt_local"] * L[q]["npad"]
        else:
            size = (cfg.nt + shift) * L[q]["mode_len"]
        cover = np.zeros(size, dtype=np.int64)
        for peer, _, dst, cnt in recv:
            cover[dst:dst + cnt] += 1
        if direction == 0:
            assert (cover == 1).all()
        else:
            lo = shift * L[q]["mode_len"]
            assert (cover[:lo] == 0).all() and (cover[lo:] == 1).all()


# ------------------------------------------------------------------------------------------
# gloo execution
# ------------------------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_schedule(sends, recvs, src: torch.Tensor, dst: torch.Tensor, rank: int):
    """Execute the library's message list with torch.distributed point-to-point calls
    (tag = position of the message in its (sender, receiver) stream)."""
    reqs, bufs = [], []
    tags = {}
    self_src = [m for m in sends if m[0] == rank]
    self_dst = [m for m in recvs if m[0] == rank]
    for (_, so, _, c), (_, _, do, c2) in zip(self_src, self_dst):
        assert c == c2
        dst[do:do + c] = src[so:so + c]
    for peer, so, _, c in sends:
        if peer == rank:
            continue
        t = tags.get(("s", peer), 0)
        tags[("s", peer)] = t + 1
        reqs.append(dist.isend(src[so:so + c].clone(), dst=int(peer), tag=t))
    for peer, _, do, c in recvs:
        if peer == rank:
            continue
        t = tags.get(("r", peer), 0)
        tags[("r", peer)] = t + 1
        b = torch.empty(int(c), dtype=src.dtype)
        bufs.append((b, do, c))
        reqs.append(dist.irecv(b, src=int(peer), tag=t))
    for r in reqs:
        r.wait()
    for b, do, c in bufs:
        dst[do:do + c] = b


class GlooTransport:
    """expd_transport over torch.distributed (gloo): isend / irecv per message, tagged by the
    message's position in its (sender, receiver) stream within the chunk; group_end waits
    for every request and copies the received buffers into the library's destination views."""

    def __init__(self):
        self.reqs, self.pending, self.tags = [], [], {}

    def group_start(self):
        self.reqs, self.pending, self.tags = [], [], {}

    def _tag(self, kind, peer):
        t = self.tags.get((kind, peer), 0)
        self.tags[(kind, peer)] = t + 1
        return t

    def send(self, view, peer):
        self.reqs.append(dist.isend(torch.from_numpy(view.copy()), dst=peer, tag=self._tag("s", peer)))

    def recv(self, view, peer):
        b = torch.empty(len(view), dtype=torch.float64)
        self.reqs.append(dist.irecv(b, src=peer, tag=self._tag("r", peer)))
        self.pending.append((view, b))

    def group_end(self):
        for r in self.reqs:
            r.wait()
        for v, b in self.pending:
            v[:] = b.numpy()


def lib_a2a(prob, rank, P, direction, shift, src, dst, s_lo=0, s_hi=1 << 30):
    """The library's all-to-all (expd_a2a_execute_host) on torch / numpy float64 buffers."""
    tr = GlooTransport()
    s = np.ascontiguousarray(src.numpy() if isinstance(src, torch.Tensor) else src)
    d = dst.numpy() if isinstance(dst, torch.Tensor) else dst
    assert d.flags.c_contiguous
    a2a_execute_host(prob, rank, P, direction, shift, s, d, tr.send, tr.recv, tr.group_start, tr.group_end,
                     s_lo=s_lo, s_hi=s_hi)


def _spawn(fn, P, *args):
    port = _free_port()
    mp.spawn(fn, args=(P, port) + args, nprocs=P, join=True)


def _init(rank, P, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)


def _a2a_worker(rank, P, port, name, n, nt):
    _init(rank, P, port)
    try:
        cfg = _cfg(name, n, nt)
        prob = Problem.from_config(cfg)
        L = layout(prob, rank, P)
        npad, off, ln, t0, ntl = L["npad"], L["mode_off"], L["mode_len"], L["t0"], L["nt_local"]
        G = torch.from_numpy(np.random.default_rng(7).standard_normal((cfg.nt, npad)))
        # mode slab -> time slab
        mode = G[:, off:off + ln].contiguous().reshape(-1)
        time = torch.full((ntl * npad,), float("nan"), dtype=torch.float64)
        lib_a2a(prob, rank, P, 0, 0, mode, time)
        assert torch.equal(time.reshape(ntl, npad), G[t0:t0 + ntl])
        # time slab -> mode slab, shifted one slice (the N-hat exchange)
        back = torch.zeros(((cfg.nt + 1) * ln,), dtype=torch.float64)
        lib_a2a(prob, rank, P, 1, 1, time, back)
        assert torch.equal(back.reshape(cfg.nt + 1, ln)[1:], G[:, off:off + ln])
        # the test-side executor of the message lists agrees with the library's
        time2 = torch.full((ntl * npad,), float("nan"), dtype=torch.float64)
        s, r = a2a_schedule(prob, rank, P, 0, 0)
        run_schedule(s, r, mode, time2, rank)
        assert torch.equal(time2, time)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P,name,n,nt", [(2, "c3", 31, 16), (4, "c5", 15, 16), (2, "c4", 7, 8), (2, "c1", None, None)])
def test_a2a_gloo(P, name, n, nt):
    _spawn(_a2a_worker, P, name, n, nt)


# ------------------------------------------------------------------------------------------
# the distributed sweep, oracle compute + gloo network
# ------------------------------------------------------------------------------------------
def _pad(x, cfg):
    """[.., n^dim] -> padded spectral slices [.., n^{dim-1} (n+1)] (pad entry 0)."""
    n = cfg.n
    lead = x.shape[:-cfg.dim]
    rows = x.reshape(lead + (-1, n))
    out = np.zeros(lead + (rows.shape[-2], n + 1))
    out[..., :n] = rows
    return out.reshape(lead + (-1,))


def _unpad(x, cfg):
    n = cfg.n
    lead = x.shape[:-1]
    return x.reshape(lead + (-1, n + 1))[..., :n].reshape(lead + (n,) * cfg.dim)


def _dist_picard_worker(rank, P, port, name, n, nt, out_dir):
    import oracle

    _init(rank, P, port)
    try:
        cfg = _cfg(name, n, nt)
        prob = Problem.from_config(cfg)
        s = oracle.spec(cfg)
        L = layout(prob, rank, P)
        npad, off, ln, t0, ntl = L["npad"], L["mode_off"], L["mode_len"], L["t0"], L["nt_local"]
        M = cfg.n + 1
        nl = len(cfg.q) > 0
        u0 = synth.initial_condition(cfg)
        u0h = _pad(oracle.dst(s, u0)[None], cfg)[0]
        modes = [e for e in range(off, off + ln) if e % M != M - 1]  # this rank's real modes
        J = {e: (e // M) * cfg.n + e % M for e in modes}
        Uh = np.zeros((cfg.nt, ln))
        Nh = np.zeros((cfg.nt + 1, ln))
        if nl:
            Nh[0] = _pad(oracle.dst(s, oracle.nonlin(s, u0))[None], cfg)[0][off:off + ln]
        hist, r0 = [], None
        for k in range(60):
            if nl:  # stage 3 on the time slab
                UT = np.zeros(ntl * npad)
                lib_a2a(prob, rank, P, 0, 0, Uh.reshape(-1), UT)
                UT = UT.reshape(ntl, npad)
                NT = np.zeros((ntl, npad))
                for i in range(ntl):
                    uh = _unpad(UT[i], cfg)
                    NT[i] = _pad(oracle.dst(s, oracle.nonlin(s, oracle.dst(s, uh)))[None], cfg)[0]
                nh = Nh.reshape(-1).copy()
                lib_a2a(prob, rank, P, 1, 1, NT.reshape(-1), nh)
                Nh = nh.reshape(cfg.nt + 1, ln)
            rn2 = 0.0
            for e in modes:  # K1 on the mode slab: residual, ||r||^2, preconditioner, update
                c = e - off
                nh = None
                if nl:  # ETD: N-hat_0..N-hat_{nt-1}; IF / IMEX (scheme 2): N-hat of u_1..u_nt
                    nh = Nh[1: cfg.nt + 1, c] if cfg.scheme == 2 else Nh[: cfg.nt, c]
                r = oracle.mode_residual(s, J[e], Uh[:, c], u0h[e], nh)
                rn2 += float(np.dot(r, r))
                Uh[:, c] += oracle.mode_precond(s, J[e], r)
            t = torch.tensor([rn2], dtype=torch.float64)
            dist.all_reduce(t)
            rn = float(np.sqrt(t.item()))
            r0 = rn if r0 is None else r0
            hist.append(rn / r0)
            if hist[-1] < cfg.tol:
                break
        UT = np.zeros(ntl * npad)
        lib_a2a(prob, rank, P, 0, 0, Uh.reshape(-1), UT)
        U = np.stack([oracle.dst(s, _unpad(x, cfg)) for x in UT.reshape(ntl, npad)])
        np.save(os.path.join(out_dir, f"U{rank}.npy"), U)
        np.save(os.path.join(out_dir, f"hist{rank}.npy"), np.array(hist))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P,name,n,nt", [(2, "c3", 15, 8), (2, "c5", 15, 8), (2, "c2", 15, 8), (4, "c5", 7, 8),
                                         (2, "c5if", 15, 8)])
def test_distributed_sweep_matches_oracle(tmp_path, P, name, n, nt):
    import oracle

    _spawn(_dist_picard_worker, P, name, n, nt, str(tmp_path))
    cfg = _cfg(name, n, nt)
    s = oracle.spec(cfg)
    Uo, st, its, hist_o = oracle.fixed_point(s, synth.initial_condition(cfg), tol=cfg.tol, maxit=60)
    U = np.concatenate([np.load(tmp_path / f"U{r}.npy") for r in range(P)])
    hists = [np.load(tmp_path / f"hist{r}.npy") for r in range(P)]
    for h in hists[1:]:
        assert np.array_equal(h, hists[0])  # every rank takes the same decisions
    assert st == 0 and len(hists[0]) - 1 == its  # identical iteration count (R8)
    assert np.abs(U - Uo).max() <= 1e-12 * np.abs(Uo).max()


# ------------------------------------------------------------------------------------------
# the pipelined exchange: chunks of slice keys (expd_api.cu stage3_dist)
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,n,nt", CASES[:5])
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("direction,shift", [(0, 0), (1, 1)])
def test_keyed_chunks_are_symmetric(name, n, nt, P, direction, shift):
    """Every slice-key chunk is a complete all-to-all by itself: what r sends q with key i
    is what q posts to receive from r with key i, in the same order."""
    cfg = _cfg(name, n, nt)
    prob = Problem.from_config(cfg)
    if cfg.nt % P:
        pytest.skip("nt % P != 0")
    S = [a2a_schedule(prob, r, P, direction, shift, keyed=True) for r in range(P)]
    ntl = cfg.nt // P
    for r in range(P):
        assert np.array_equal(S[r][0][:, :4], a2a_schedule(prob, r, P, direction, shift)[0])
        assert set(S[r][0][:, 4]) == set(range(ntl)) == set(S[r][1][:, 4])
        for q in range(P):
            for key in range(ntl):
                sent = S[r][0][(S[r][0][:, 0] == q) & (S[r][0][:, 4] == key)][:, 3]
                got = S[q][1][(S[q][1][:, 0] == r) & (S[q][1][:, 4] == key)][:, 3]
                assert list(sent) == list(got), (r, q, key)


def _chunked_worker(rank, P, port, name, n, nt, k):
    _init(rank, P, port)
    try:
        cfg = _cfg(name, n, nt)
        prob = Problem.from_config(cfg)
        L = layout(prob, rank, P)
        npad, off, ln, t0, ntl = L["npad"], L["mode_off"], L["mode_len"], L["t0"], L["nt_local"]
        G = torch.from_numpy(np.random.default_rng(7).standard_normal((cfg.nt, npad)))
        mode = G[:, off:off + ln].contiguous().reshape(-1)
        time = torch.full((ntl * npad,), float("nan"), dtype=torch.float64)
        back = torch.zeros(((cfg.nt + 1) * ln,), dtype=torch.float64)
        s0, r0 = a2a_schedule(prob, rank, P, 0, 0, keyed=True)
        s1, r1 = a2a_schedule(prob, rank, P, 1, 1, keyed=True)
        chunks = [(lo, min(lo + k, ntl)) for lo in range(0, ntl, k)]
        sel = lambda m, lo, hi: m[(m[:, 4] >= lo) & (m[:, 4] < hi)][:, :4]  # noqa: E731
        for lo, hi in chunks:  # every mode -> time chunk first (as posted on the comm stream)
            run_schedule(sel(s0, lo, hi), sel(r0, lo, hi), mode, time, rank)
        assert torch.equal(time.reshape(ntl, npad), G[t0:t0 + ntl])
        for lo, hi in chunks:  # then chunk by chunk back, after "stage 3" of the chunk
            run_schedule(sel(s1, lo, hi), sel(r1, lo, hi), time, back, rank)
        assert torch.equal(back.reshape(cfg.nt + 1, ln)[1:], G[:, off:off + ln])
        # the library's chunked execution (slice-key ranges, expd_api.cu stage3_dist's order)
        time2 = torch.full((ntl * npad,), float("nan"), dtype=torch.float64)
        back2 = torch.zeros(((cfg.nt + 1) * ln,), dtype=torch.float64)
        for lo, hi in chunks:
            lib_a2a(prob, rank, P, 0, 0, mode, time2, lo, hi)
        assert torch.equal(time2, time)
        for lo, hi in chunks:
            lib_a2a(prob, rank, P, 1, 1, time2, back2, lo, hi)
        assert torch.equal(back2, back)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P,name,n,nt,k", [(2, "c3", 31, 16, 3), (4, "c5", 15, 16, 1), (2, "c4", 7, 8, 2)])
def test_chunked_a2a_gloo(P, name, n, nt, k):
    _spawn(_chunked_worker, P, name, n, nt, k)


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("dim,n,nt", [(1, 15, 8), (2, 15, 8), (3, 7, 8)])
def test_complex_layout_is_the_real_one_doubled(P, dim, n, nt):
    """A complex problem partitions the interleaved (re, im) spectral slice: the same padded
    x-lines per rank as the real problem (dim >= 2), every offset and length doubled."""
    base = dict(dim=dim, n=n, a=1.0, c=0.0, dt=0.01, nt=nt, alpha=1e-2)
    real = Problem(**base)
    cplx = Problem(**{**base, "a": 0.0, "a_im": 1.0, "c_im": 2.0})
    for r in range(P):
        lr, lc = layout(real, r, P), layout(cplx, r, P)
        assert lc["npad"] == 2 * lr["npad"] and lc["nt_local"] == lr["nt_local"]
        assert lc["mode_len"] % 2 == 0 and lc["mode_off"] % 2 == 0
        if dim >= 2:
            assert lc["mode_off"] == 2 * lr["mode_off"] and lc["mode_len"] == 2 * lr["mode_len"]
    off = 0
    for r in range(P):
        lc = layout(cplx, r, P)
        assert lc["mode_off"] == off
        off += lc["mode_len"]
    assert off == 2 * layout(real, 0, P)["npad"]


# ------------------------------------------------------------------------------------------
# the host communicator (expd_host_comm_create): host-only lifecycle and argument checks;
# tests/test_gpu_multirank.py runs distributed plans through it on the GPU
# ------------------------------------------------------------------------------------------
def test_host_comm_lifecycle():
    import ctypes as C

    from paper_2603_04350_b200 import ExpdError, HostComm
    from paper_2603_04350_b200.expd import _make_transport, load_library

    tr = GlooTransport()
    c = HostComm(1, 2, 0, tr)
    assert c.ptr
    lib = load_library()
    lib.expd_nccl_comm_destroy(c.ptr)  # not an NCCL communicator: ignored
    c.close()
    c.close()  # idempotent
    with pytest.raises(ExpdError):
        HostComm(2, 2, 0, tr)  # rank out of range
    t, cb = _make_transport(tr.send, tr.recv)
    h = C.c_void_p()
    assert lib.expd_host_comm_create(C.byref(t), 0, 0, C.byref(h)) == 1  # nranks < 1
    assert lib.expd_host_comm_create(None, 0, 1, C.byref(h)) == 1
