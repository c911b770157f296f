"""Pins of the oracle's spherical-harmonic expansions (P:109 Cheng et al. basis,
SURVEY 8c-2 items 8-16) against library routines and closed forms.

* R_n^m, I_n^m vs scipy.special.lpmv (Condon-Shortley P_n^m): R = r^n P e^{im phi}
  /(n+m)!, I = (n-m)! P e^{im phi} / r^{n+1}.
* Addition theorem for 1/|x - y| (exact series, checked to 1e-13).
* M2M and L2L are exact; P2M of a centred particle has only n = 0.
* M2L + L2P potential, gradient and Hessian vs the direct point-source sums,
  with error decreasing monotonically in p.
"""
import math

import numpy as np
import pytest
from scipy.special import lpmv


def _nm(P):
    return [(n, m) for n in range(P) for m in range(n + 1)]


def _sph(x):
    r = np.linalg.norm(x)
    return r, x[2] / r, math.atan2(x[1], x[0])


@pytest.mark.parametrize("x", [[0.3, -0.4, 0.5], [-1.2, 0.7, -0.1], [0.05, 0.02, 1.3]])
def test_harmonics_match_legendre(oracle_mod, x):
    P = 12
    R = oracle_mod.regular(x, P)
    I = oracle_mod.irregular(x, P)
    r, ct, ph = _sph(np.array(x))
    for k, (n, m) in enumerate(_nm(P)):
        pl = lpmv(m, n, ct)
        rref = r ** n * pl * np.exp(1j * m * ph) / math.factorial(n + m)
        iref = math.factorial(n - m) * pl * np.exp(1j * m * ph) / r ** (n + 1)
        assert abs(R[k] - rref) <= 1e-12 * max(1.0, abs(rref))
        assert abs(I[k] - iref) <= 1e-12 * max(1.0, abs(iref))


def _full(C, P):
    """dict (n, m) -> value over all m in [-n, n] via C_n^{-m} = (-1)^m conj."""
    out = {}
    k = 0
    for n in range(P):
        for m in range(n + 1):
            out[(n, m)] = C[k]
            out[(n, -m)] = (-1) ** m * np.conj(C[k])
            k += 1
    return out


def test_addition_theorem_inverse_distance(oracle_mod):
    P = 45
    x = np.array([0.9, -0.5, 0.7]); y = np.array([0.1, 0.2, -0.15])
    R = _full(oracle_mod.regular(y, P), P)
    I = _full(oracle_mod.irregular(x, P), P)
    s = sum(np.conj(R[(n, m)]) * I[(n, m)] for n in range(P) for m in range(-n, n + 1))
    assert abs(s.imag) < 1e-13
    assert abs(s.real - 1 / np.linalg.norm(x - y)) < 1e-13


def test_p2m_centred_particle_and_symmetric_pair(oracle_mod):
    P = 10
    M = oracle_mod.p2m(P, [[0.5, 0.5, 0.5]], [2.0], [0.5, 0.5, 0.5])
    assert M[0] == 2.0 and np.all(M[1:] == 0)
    M = oracle_mod.p2m(P, [[0.1, 0, 0], [-0.1, 0, 0]], [1.0, -1.0], [0, 0, 0])
    assert abs(M[0]) < 1e-16 and abs(M[2]) > 0.01        # n = 1, m = 1 dipole


def test_m2m_is_exact(oracle_mod):
    rng = np.random.default_rng(1106)
    P = 10
    x = rng.random((30, 3)) * 0.5
    q = rng.standard_normal(30)
    cc = np.array([0.25, 0.25, 0.25]); cp = np.array([0.5, 0.5, 0.5]); cp2 = np.array([1.1, -0.3, 0.2])
    Mc = oracle_mod.p2m(P, x, q, cc)
    Mp = oracle_mod.m2m(P, Mc, cc - cp)
    ref = oracle_mod.p2m(P, x, q, cp)
    assert np.max(np.abs(Mp - ref)) < 1e-12 * np.max(np.abs(ref))
    # composition: two shifts == one shift
    Mp2 = oracle_mod.m2m(P, Mp, cp - cp2)
    assert np.max(np.abs(Mp2 - oracle_mod.m2m(P, Mc, cc - cp2))) < 1e-12 * np.max(np.abs(Mp2))


def _direct_phi_derivs(xt, xs, q):
    d = xt[None, :] - xs
    r = np.linalg.norm(d, axis=1)
    phi = np.sum(q / r)
    grad = -np.sum((q / r ** 3)[:, None] * d, axis=0)
    H = np.zeros((3, 3))
    for a in range(3):
        for b in range(3):
            H[a, b] = np.sum(q * (3 * d[:, a] * d[:, b] / r ** 5 - (a == b) / r ** 3))
    return phi, grad, H


def _hess6(H):
    return np.array([H[0, 0], H[1, 1], H[2, 2], H[0, 1], H[0, 2], H[1, 2]])


def test_m2l_l2p_derivatives_converge_to_direct(oracle_mod):
    """Cluster of radius 0.5 around cs, local expansion about ct at distance 3:
    potential, gradient and Hessian at a point 0.4 from ct approach the
    direct point-source values monotonically as p grows."""
    rng = np.random.default_rng(5273)
    cs = np.array([0.0, 0.0, 0.0]); ct = np.array([2.0, 1.5, -1.3])
    xs = cs + (rng.random((40, 3)) - 0.5) * 0.55
    q = rng.standard_normal(40)
    pt = ct + np.array([0.2, -0.25, 0.2])
    phi0, g0, H0 = _direct_phi_derivs(pt, xs, q)
    errs = []
    for P in (4, 6, 8, 10, 12, 14):
        M = oracle_mod.p2m(P, xs, q, cs)
        L = oracle_mod.m2l(P, M, ct - cs)
        phi, g, h = oracle_mod.l2p_derivs(P, L, pt - ct)
        e = max(abs(phi - phi0) / abs(phi0), np.linalg.norm(g - g0) / np.linalg.norm(g0),
                np.linalg.norm(h - _hess6(H0)) / np.linalg.norm(_hess6(H0)))
        errs.append(e)
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-6


def test_l2l_is_exact_and_m2p(oracle_mod):
    rng = np.random.default_rng(7)
    P = 10
    cs = np.zeros(3); ct = np.array([3.0, 0.5, 0.2])
    xs = (rng.random((20, 3)) - 0.5) * 0.6
    q = rng.standard_normal(20)
    M = oracle_mod.p2m(P, xs, q, cs)
    # multipole potential converges to the direct potential far away
    far = np.array([5.0, -4.0, 3.0])
    assert abs(oracle_mod.m2p(P, M, far - cs) - np.sum(q / np.linalg.norm(far - xs, axis=1))) < 1e-12
    L = oracle_mod.m2l(P, M, ct - cs)
    cc = ct + np.array([0.15, -0.1, 0.12])
    Lc = oracle_mod.l2l(P, L, cc - ct)
    for _ in range(5):
        y = ct + (rng.random(3) - 0.5) * 0.5
        a = oracle_mod.l2p_derivs(P, L, y - ct)
        b = oracle_mod.l2p_derivs(P, Lc, y - cc)
        assert abs(a[0] - b[0]) < 1e-12 * abs(a[0])
        assert np.allclose(a[1], b[1], rtol=1e-11, atol=1e-14)
        assert np.allclose(a[2], b[2], rtol=1e-10, atol=1e-13)
