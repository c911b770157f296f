"""Pins of the oracle's NEXT-1 time step (Eq. 4): a lone
particle does not move and keeps its strength while sigma^2 grows by exactly
2 nu dt; sigma is untouched at nu = 0; the midpoint RK2 is second
order (error ratio ~4 per halving of dt on a co-rotating vortex pair)."""
import numpy as np


def test_single_particle_and_core_spreading(oracle_mod):
    x = np.array([[0.1, 0.2, 0.3]]); a = np.array([[0.0, 0.4, 1.0]]); s = np.array([0.3])
    x1, a1, s1 = oracle_mod.rk2_step(x, a, s, dt=0.1, nu=0.05)
    assert np.array_equal(x1, x) and np.array_equal(a1, a)
    assert abs(s1[0] ** 2 - (0.3 ** 2 + 2 * 0.05 * 0.1)) < 1e-15
    x2, a2, s2 = oracle_mod.rk2_step(np.random.default_rng(1).random((20, 3)), np.ones((20, 3)) * 1e-2,
                                     np.full(20, 0.2), dt=0.01, nu=0.0)
    assert np.all(s2 == 0.2)


def test_rk2_is_second_order(oracle_mod):
    # two parallel vortex blobs separated along x co-rotate
    x0 = np.array([[-0.5, 0.0, 0.0], [0.5, 0.0, 0.0]])
    a0 = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 1.0]])
    s0 = np.array([0.2, 0.2])
    T = 0.4

    def run(nsteps):
        x, a, s = x0.copy(), a0.copy(), s0.copy()
        for _ in range(nsteps):
            x, a, s = oracle_mod.rk2_step(x, a, s, T / nsteps)
        return x

    ref = run(512)
    e = [np.linalg.norm(run(m) - ref) for m in (8, 16, 32)]
    assert 3.0 < e[0] / e[1] < 5.0 and 3.0 < e[1] / e[2] < 5.0, e
