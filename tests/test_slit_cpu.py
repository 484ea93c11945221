"""The S-lit comparison arm (tools/slit_compare.py: the paper's literal Steps (a)-(c) with
cuFFT / torch for the time DFT and the library's DST for V) computes Q_alpha^{-1}: checked on
CPU against the oracle's preconditioner, with scipy's orthonormal DST-I standing in for V."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest
import torch

import synth

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import slit_compare  # noqa: E402

sfft = pytest.importorskip("scipy.fft")


def _dst(P: torch.Tensor) -> torch.Tensor:
    x = P.numpy()
    axes = tuple(range(2, x.ndim))  # the spatial axes of (K, 2, n..n)
    return torch.from_numpy(sfft.dstn(x, type=1, axes=axes, norm="ortho"))


@pytest.mark.parametrize("name,n,nt", [("c2", 15, 16), ("c3", 15, 8), ("c5", 31, 8), ("c1", 31, 32)])
def test_slit_arm_equals_oracle_precond(orc, name, n, nt):
    cfg = synth.CONFIGS[name].scaled(n, nt)
    R = synth.random_spacetime(cfg, seed=5)
    want, leak = orc.precond(orc.spec(cfg), R)
    got = slit_compare.slit_apply(cfg, torch.from_numpy(R), slit_compare.mode_E(cfg), _dst).numpy()
    assert np.abs(got - want).max() < 1e-11 * np.abs(want).max()


def test_mode_table_matches_oracle(orc):
    cfg = synth.CONFIGS["c3"].scaled(9, 4)
    mu, E, f1, f2 = orc.mode_tables(orc.spec(cfg))
    assert np.abs(slit_compare.mode_E(cfg).numpy() - E).max() < 1e-14 * np.abs(E).max()
