"""S-lit against S-spec, measured: the preconditioner apply s = Q_alpha^{-1} r on physical slices
in the paper's literal order (Steps (a)-(c)) next to the library's S-spec
apply (DST -> K1 -> IDST, `expd_precond_apply`), at c3 and c5's full sizes on one B200.

S-lit here ("S-lit as a measured comparison"):
  (a) Gamma_alpha scaling and the time DFT of every spatial point      torch.fft.rfft (cuFFT)
  (b) per frequency k, the spatial solve (I - lambda_k A)^{-1}:
      planar split, V (the library's DST-I line kernels, expd_dst), divide by 1 - lambda_k E_J,
      V again (V = V^{-1}), interleave                                   expd_dst + torch
  (c) inverse time DFT and Gamma_alpha^{-1}                              torch.fft.irfft
with lambda_k = alpha^{1/Nt} e^{-2 pi i k / Nt} (Gamma C_alpha Gamma^{-1} = alpha^{1/Nt} Z, Z the
cyclic shift) and E_J = exp(dt (a mu_J - c)).  Real r -> Hermitian spectrum,
so only k = 0..Nt/2 is solved.  This is a measurement tool, not the product path: the time
DFT is cuFFT's and the pointwise steps are torch's, the spatial transforms are ours.

Usage: python tools/slit_compare.py [c3 c5 ...] > gpurun_out/slit.json
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def mode_E(cfg, device=None) -> torch.Tensor:
    """E_J = exp(dt (a mu_J - c)), mu_J = sum over axes of -(4/h^2) sin^2(j pi h / 2), x fastest."""
    n, h = cfg.n, 1.0 / (cfg.n + 1)
    j = np.arange(1, n + 1, dtype=np.float64)
    lam = -4.0 / h ** 2 * np.sin(np.pi * j * h / 2) ** 2
    mu = np.zeros((n,) * cfg.dim)
    for ax in range(cfg.dim):
        shape = [1] * cfg.dim
        shape[cfg.dim - 1 - ax] = n  # axis 0 of the J index (x) is the last array axis
        mu = mu + lam.reshape(shape)
    return torch.from_numpy(np.exp(cfg.dt * (cfg.a * mu - cfg.c))).to(device)


def slit_apply(cfg, R: torch.Tensor, E: torch.Tensor, dst, timer=None) -> torch.Tensor:
    """Steps (a)-(c) literally; `dst` applies V to a stack of real slices; `timer(name)` marks
    the end of each step when given."""
    mark = timer or (lambda name: None)
    nt, K = cfg.nt, cfg.nt // 2 + 1
    g = torch.tensor([cfg.alpha ** (m / nt) for m in range(nt)], dtype=torch.float64, device=R.device)
    gs = g.reshape((nt,) + (1,) * cfg.dim)
    Y = torch.fft.rfft(R * gs, dim=0)  # (a)
    mark("a_time_dft")
    P = torch.view_as_real(Y).movedim(-1, 1).contiguous()  # (K, 2, n..n) planar
    del Y
    mark("b_split")
    P = dst(P)
    mark("b_dst")
    k = torch.arange(K, dtype=torch.float64, device=R.device)
    lam = cfg.alpha ** (1.0 / nt) * torch.exp(torch.complex(torch.zeros_like(k), -2 * math.pi * k / nt))
    D = 1 - lam.reshape((K,) + (1,) * cfg.dim) * E
    Z = torch.complex(P[:, 0], P[:, 1]) / D
    del D
    P = torch.stack((Z.real, Z.imag), 1)
    del Z
    mark("b_divide")
    P = dst(P)
    mark("b_idst")
    Y = torch.complex(P[:, 0], P[:, 1])
    del P
    mark("b_merge")
    S = torch.fft.irfft(Y, n=nt, dim=0) / gs  # (c)
    mark("c_inverse_dft")
    return S


def main(names):
    import synth
    from paper_2603_04350_b200 import Plan, Problem

    dev = torch.device("cuda:0")
    out = {}
    for name in names:
        cfg = synth.CONFIGS[name]
        plan = Plan(Problem.from_config(cfg))
        R = torch.from_numpy(synth.random_spacetime(cfg)).to(dev)
        E = mode_E(cfg, dev)
        S_spec = plan.precond_apply(R)
        torch.cuda.synchronize()

        def run_lit(times=None):
            evs = []

            def timer(label):
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                evs.append((label, ev))

            start = torch.cuda.Event(enable_timing=True)
            start.record()
            S = slit_apply(cfg, R, E, plan.dst, timer)
            torch.cuda.synchronize()
            if times is not None:
                prev = start
                for label, ev in evs:
                    times.setdefault(label, []).append(prev.elapsed_time(ev))
                    prev = ev
                times.setdefault("total", []).append(start.elapsed_time(evs[-1][1]))
            return S

        S_lit = run_lit()
        err = float((S_lit - S_spec).abs().max() / S_spec.abs().max())
        del S_lit
        torch.cuda.empty_cache()
        lit = {}
        for _ in range(5):
            run_lit(lit)
        spec = []
        Sbuf = torch.empty_like(R)
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            plan.precond_apply(R, Sbuf)
            b.record()
            torch.cuda.synchronize()
            spec.append(a.elapsed_time(b))
        med = lambda v: float(np.median(v))  # noqa: E731
        dofs = cfg.nt * cfg.N
        out[name] = {
            "shape": [cfg.nt] + [cfg.n] * cfg.dim,
            "rel_max_diff_lit_vs_spec": err,
            "s_lit_ms": {k: med(v) for k, v in lit.items()},
            "s_spec_precond_apply_ms": med(spec),
            "s_lit_over_s_spec": med(lit["total"]) / med(spec),
            "dofs": dofs,
            "note": "physical in / physical out preconditioner apply; inside the sweep S-spec never "
                    "leaves the DST basis, so its preconditioner is only K1 (fused with the residual)",
        }
        del R, E, S_spec, Sbuf, plan
        torch.cuda.empty_cache()
        print(json.dumps({name: out[name]}), file=sys.stderr)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3", "c5"])
