"""NEXT-3 analysis harness (oracle/analysis.py) against the oracle's solves and closed forms."""
from __future__ import annotations

import math

import numpy as np
import pytest

import synth
from oracle import analysis


@pytest.mark.parametrize("name,n,nt", [("c1", None, None), ("c2", 15, 16), ("c4", 7, 8), ("c2", 31, 64)])
def test_exact_history_predicts_fixed_point_count(orc, name, n, nt):
    cfg = synth.CONFIGS[name] if n is None else synth.CONFIGS[name].scaled(n, nt)
    s = orc.spec(cfg)
    u0 = synth.initial_condition(cfg)
    _, st, its, hist = orc.fixed_point(s, u0, tol=cfg.tol, maxit=40)
    assert st == 0
    assert analysis.fp_iterations_exact(s, u0, cfg.tol) == its
    pred = analysis.fp_history_exact(s, u0, len(hist) - 1)
    big = hist > 1e-12
    assert np.allclose(pred[big], hist[big], rtol=1e-8)
    assert its <= analysis.fp_iterations_bound(s, cfg.tol)  # Thm 2.1 bounds the count


def test_bounds_cover_the_solvers(orc):
    # slow case (alpha = 0.2, weak diffusion): several iterations, still within the bounds
    cfg = synth.Config("b", 1, 15, 0.05, 0.0, 0.5, 16, 0.2)
    s = orc.spec(cfg)
    u0 = np.random.default_rng(3).standard_normal(15)
    _, st, its, _ = orc.fixed_point(s, u0, tol=1e-12, maxit=60)
    assert st == 0 and 3 <= its <= analysis.fp_iterations_bound(s, 1e-12)
    _, st, its_g, _ = orc.gmres(s, u0, tol=1e-12, restart=50, maxit=60)
    assert st == 0 and its_g <= analysis.gmres_iterations_bound(s, 1e-12)


def test_minmax_objective_closed_form_and_monotone(orc):
    """The max over omega of (minmax) sits at omega = 0: alpha e^{-cT} / (1 - alpha e^{-cT});
    increasing in alpha, so the minimiser runs to the lower end (reading R19)."""
    s = orc.spec(synth.CONFIGS["c2"])
    for al in (1e-4, 1e-3, 0.1, 0.5):
        e = al * math.exp(-s.c * s.T)
        assert abs(analysis.minmax_objective(al, s) - e / (1 - e)) < 1e-15
    vals = [analysis.minmax_objective(a, s) for a in np.geomspace(1e-8, 0.9, 30)]
    assert all(b > a for a, b in zip(vals, vals[1:]))
    assert analysis.alpha_minmax(s, lo=1e-10) < 1e-9


def test_config_alphas_satisfy_the_theory(orc):
    """Every config's alpha: contraction < 1, Elman's condition (R12), and the
    round-off floor eps cond(Gamma_alpha) below the config tolerance."""
    for cfg in synth.CONFIGS.values():
        r = analysis.report(cfg)
        assert r["psi_max"] < 1.0
        assert r["elman_applies"], cfg.name
        assert r["roundoff_floor"] < cfg.tol, cfg.name
        assert r["minmax_objective_increasing"]
