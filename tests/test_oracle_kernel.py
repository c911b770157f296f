"""Pins of the oracle's pair kernel and direct sum (Eqs. 1-3) against
values the paper and the mathematics fix -- not against the oracle itself.

* Eq. 2 cutoff vs scipy.special.erf and the golden g(1) (reading Z23).
* Eq. 1 single blob closed form (golden, reading Z1).
* Eq. 3 = central finite difference of Eq. 1 along alpha_i (Z3).
* Lamb-Oseen line vortex closed form (free-space direct sum).
* Taylor-Green closed form (periodic direct sum over 27^3 boxes, Z14/Z26).
* Linearity, antisymmetry, additivity, self-pair zero (Z7).
"""
import json
import os

import numpy as np
import pytest
from scipy.special import erf

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_cutoff_matches_scipy_and_golden(oracle_mod):
    rho = np.concatenate([np.linspace(0, 6, 601), [1e-3, 0.05, 10.0, 30.0]])
    ref = erf(rho) - 2.0 / np.sqrt(np.pi) * rho * np.exp(-rho ** 2)
    got = np.array([oracle_mod.cutoff_g(r) for r in rho])
    assert np.max(np.abs(got - ref)) < 1e-15
    assert oracle_mod.cutoff_g(0.0) == 0.0
    g1 = GOLD["cutoff_g_rho1"]
    assert abs(oracle_mod.cutoff_g(g1["rho"]) - g1["g"]) < 1e-13
    assert np.all(np.diff(got[:601]) >= 0)          # monotone
    assert abs(oracle_mod.cutoff_g(10.0) - 1.0) < 1e-15


def test_single_blob_golden(oracle_mod):
    b = GOLD["single_blob"]
    u, s = oracle_mod.direct([b["target"]], [[0, 0, 0]], [b["source"]], [b["alpha"]], [b["sigma"]])
    assert np.allclose(u[0], b["u"], rtol=0, atol=1e-15)
    assert np.allclose(s[0], 0.0, atol=1e-15)       # alpha_i = 0 => no stretching


def test_self_pair_and_empty(oracle_mod):
    x = [[0.1, 0.2, 0.3]]
    a = [[0.3, -0.2, 0.5]]
    u, s = oracle_mod.direct(x, a, x, a, [0.1])
    assert np.all(u == 0) and np.all(s == 0)        # reading Z7
    u, s = oracle_mod.direct(x, a, np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0))
    assert np.all(u == 0) and np.all(s == 0)


def test_stretching_is_directional_derivative_of_velocity(oracle_mod):
    """Eq. 3 equals (alpha_i . grad) u, checked by central differences of
    Eq. 1 along alpha_i with step 1e-5 sigma."""
    rng = np.random.default_rng(1106)
    ns = 60
    xs = rng.random((ns, 3))
    as_ = rng.standard_normal((ns, 3))
    sig = 0.05 + 0.1 * rng.random(ns)
    xt = rng.random((20, 3)) + 0.013
    at = rng.standard_normal((20, 3))
    _, s = oracle_mod.direct(xt, at, xs, as_, sig)
    h = 1e-5 * sig.min()
    fd = np.zeros_like(s)
    for i in range(len(xt)):
        dirn = at[i]
        up, _ = oracle_mod.direct(xt[i:i + 1] + h * dirn, at[i:i + 1], xs, as_, sig)
        um, _ = oracle_mod.direct(xt[i:i + 1] - h * dirn, at[i:i + 1], xs, as_, sig)
        fd[i] = (up[0] - um[0]) / (2 * h)
    assert np.linalg.norm(fd - s) / np.linalg.norm(s) < 1e-6


def test_lamb_oseen_line_vortex(oracle_mod):
    """A line of Gaussian blobs along z (spacing h <= sigma, strength Gamma h,
    half-length Lambda) has u_theta = Gamma/(2 pi r)(1 - e^{-r^2/2 sigma^2})
    * Lambda/sqrt(r^2 + Lambda^2)."""
    sigma, gamma, lam = 1.0, 2.5, 2000.0
    for h in (0.5, 1.0):
        z = np.arange(-lam, lam + 1e-9, h)
        xs = np.stack([np.zeros_like(z), np.zeros_like(z), z], -1)
        as_ = np.tile([0.0, 0.0, gamma * h], (len(z), 1))
        r = np.array([0.3, 0.7, 1.0, 1.5, 2.5, 4.0, 7.0])
        phi = np.linspace(0.1, 2 * np.pi, len(r))
        xt = np.stack([r * np.cos(phi), r * np.sin(phi), np.zeros_like(r)], -1)
        u, _ = oracle_mod.direct(xt, np.zeros_like(xt), xs, as_, np.full(len(z), sigma))
        ut = gamma / (2 * np.pi * r) * (1 - np.exp(-r ** 2 / (2 * sigma ** 2))) * lam / np.sqrt(r ** 2 + lam ** 2)
        etheta = np.stack([-np.sin(phi), np.cos(phi), np.zeros_like(phi)], -1)
        assert np.max(np.abs(u - ut[:, None] * etheta)) / ut.max() < 1e-6


def _tg_closed_form(x, alpha, sigma):
    X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
    damp = np.exp(-1.5 * sigma ** 2)
    u = np.stack([np.sin(X) * np.cos(Y) * np.cos(Z), -np.cos(X) * np.sin(Y) * np.cos(Z), 0 * X], -1)
    J = np.zeros((len(X), 3, 3))     # J[a, d] = d u_a / d x_d
    J[:, 0, 0] = np.cos(X) * np.cos(Y) * np.cos(Z)
    J[:, 0, 1] = -np.sin(X) * np.sin(Y) * np.cos(Z)
    J[:, 0, 2] = -np.sin(X) * np.cos(Y) * np.sin(Z)
    J[:, 1, 0] = np.sin(X) * np.sin(Y) * np.cos(Z)
    J[:, 1, 1] = -np.cos(X) * np.cos(Y) * np.cos(Z)
    J[:, 1, 2] = np.cos(X) * np.sin(Y) * np.sin(Z)
    s = np.einsum("nad,nd->na", J, alpha)
    return damp * u, damp * s


def test_taylor_green_periodic_direct_sum_closed_form(oracle_mod):
    """Periodic direct sum over 27^3 image boxes (k = 3, Z14) of the TG
    lattice equals the Gaussian-smoothed TG field e^{-3 sigma^2/2} u_TG and
    its stretching (Z26; closed form of the |k|^2 = 3 mode)."""
    x, a, s = synth.taylor_green(6)
    u, st = oracle_mod.direct(x, a, x, a, s, images=3)
    uc, sc = _tg_closed_form(x.astype(np.float64), a.astype(np.float64), float(s[0]))
    assert oracle_mod.rel_l2(u, uc) < 3e-6
    assert oracle_mod.rel_l2(st, sc) < 3e-6
    # zero mean velocity of a periodic TG field with sum(alpha) = 0 (invariant)
    assert abs(a.astype(np.float64).sum(0)).max() < 1e-7
    assert np.abs(u.mean(0)).max() < 1e-10


def test_linearity_antisymmetry_additivity(oracle_mod):
    rng = np.random.default_rng(5273)
    xs = rng.random((40, 3)); as_ = rng.standard_normal((40, 3)); sig = np.full(40, 0.2)
    xt = rng.random((15, 3)); at = rng.standard_normal((15, 3))
    u, s = oracle_mod.direct(xt, at, xs, as_, sig)
    u2, s2 = oracle_mod.direct(xt, 3 * at, xs, 3 * as_, sig)
    assert np.allclose(u2, 3 * u, rtol=1e-13, atol=0)     # u linear in alpha_j
    assert np.allclose(s2, 9 * s, rtol=1e-13, atol=0)     # s bilinear in alpha_i, alpha_j
    ua, sa = oracle_mod.direct(xt, at, xs[:25], as_[:25], sig[:25])
    ub, sb = oracle_mod.direct(xt, at, xs[25:], as_[25:], sig[25:])
    assert np.allclose(ua + ub, u, rtol=1e-13, atol=1e-15)   # additivity
    assert np.allclose(sa + sb, s, rtol=1e-13, atol=1e-15)
    # antisymmetry of the pair velocity: swapping i and j with equal alpha
    p = rng.random((2, 3)); al = rng.standard_normal(3)
    uij, _ = oracle_mod.direct(p[:1], [al], p[1:], [al], [0.3])
    uji, _ = oracle_mod.direct(p[1:], [al], p[:1], [al], [0.3])
    assert np.allclose(uij, -uji, rtol=1e-14, atol=1e-16)


def test_flop_model_golden():
    """Table 1 totals and the corrected sustained-performance formula (Z21)."""
    t = GOLD["table1_breakdown"]
    assert sum(t["biot_savart"].values()) == GOLD["table1_flops_per_pair"]["biot_savart"]
    assert sum(t["stretching"].values()) == GOLD["table1_flops_per_pair"]["stretching"]
    f = GOLD["flop_formula"]
    v = (f["processes"] * f["targets_per_process"] * f["source_cells_per_target"] *
         f["particles_per_cell"] * f["flops_per_interaction"] / f["wall_clock_s"])
    assert abs(v / f["result_flops"] - 1) < f["rel_tol"]
