"""Pins of the NEXT-4 oracle (RBF reinitialisation; oracle.zeta,
gauss_field, rbf_reinit) against things other than itself: the radial mass of
zeta is g of Eq. 2 (quadrature vs the C oracle's cutoff), the identity fixed
point (sites = particles, same core: A beta = A alpha), the Taylor-Green closed
form (a lattice Fourier mode is an eigenvector: beta = e^{3(s0^2 - s^2)/2} alpha)
and conservation of total strength (lattice sums of a Gaussian = 1/h^3).
The closed form neglects the lattice aliases of the Gaussian symbol
(~e^{-2 pi^2 s0^2 / h^2}) and the image truncation; both are below 2e-6 for
s0 in [h, 1.2 h] (0.8 h: 2e-4, 1.5 h: 3e-4 through the conditioning of A,
which grows like e^{3 pi^2 s0^2 / (2 h^2)} -- DESIGN.md reading R2)."""
import numpy as np
import pytest
from scipy import integrate

import oracle
import synth


@pytest.mark.parametrize("s", [0.3, 1.0, 2.5])
def test_zeta_radial_mass_is_eq2_cutoff(s):
    for r in (0.1 * s, 0.7 * s, 1.0 * s, 2.0 * s, 4.0 * s):
        m, _ = integrate.quad(lambda t: 4 * np.pi * t * t * float(oracle.zeta(t * t, s)), 0.0, r, epsabs=1e-14,
                              epsrel=1e-13)
        assert abs(m - oracle.cutoff_g(r / (np.sqrt(2.0) * s))) < 1e-11
    tot, _ = integrate.quad(lambda t: 4 * np.pi * t * t * float(oracle.zeta(t * t, s)), 0.0, 40 * s)
    assert abs(tot - 1.0) < 1e-10


def test_identity_fixed_point_random_strengths():
    x, _a, s = synth.jittered_lattice(6)
    a = np.random.default_rng(7).standard_normal(x.shape)
    beta = oracle.rbf_reinit(x, a, s, x, float(s[0]), images=1)
    assert np.abs(beta - a).max() / np.abs(a).max() < 1e-9


@pytest.mark.parametrize("f0", [1.0, 1.1, 1.2])
def test_taylor_green_closed_form(f0):
    n = 8
    x, a, s = synth.taylor_green(n)
    h = 2 * np.pi / n
    beta = oracle.rbf_reinit(x, a, s, x, f0 * h, images=1)
    want = np.exp(1.5 * ((f0 * h) ** 2 - h ** 2)) * a.astype(np.float64)
    assert np.linalg.norm(beta - want) / np.linalg.norm(want) < 5e-6


def test_total_strength_conserved():
    rng = np.random.default_rng(11)
    n = 8
    h = 2 * np.pi / n
    x = (-np.pi + 2 * np.pi * rng.random((300, 3)))
    a = rng.standard_normal((300, 3)) * h ** 3
    s = np.full(300, h)
    y, _ya, _ys = synth.taylor_green(n)
    beta = oracle.rbf_reinit(x, a, s, y, h, images=1)
    assert np.abs(beta.sum(0) - a.sum(0)).max() < 1e-6 * np.abs(a).sum()
