"""GPU parity of NEXT-1, the vortex time step around evaluate (fmm_step):
midpoint RK2 of P:69 with sigma^2 += 2 nu dt (Eq. 4) against the oracle's RK2
on the c-1 direct sum."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def test_single_particle_core_spreading_exact():
    import paper_1106_5273_b200 as P
    f = P.FMM(images=0)
    x = np.array([[0.1, 0.2, 0.3]], np.float32)
    a = np.array([[0.0, 0.4, 1.0]], np.float32)
    s = np.array([0.3], np.float32)
    f.step(x, a, s, dt=0.1, nu=0.05)
    assert np.array_equal(x, [[0.1, 0.2, 0.3]]) or np.allclose(x, [[0.1, 0.2, 0.3]], atol=0)
    assert np.array_equal(a, np.array([[0.0, 0.4, 1.0]], np.float32))
    assert s[0] == np.float32(np.sqrt(0.3 ** 2 + 2 * 0.05 * 0.1)) or abs(s[0] ** 2 - 0.1) < 1e-7
    f.close()


@pytest.mark.parametrize("images", [0, 1])
def test_rk2_step_vs_oracle(oracle_mod, images):
    """Free space with a root leaf (exact P2P) and a periodic Taylor-Green
    lattice (FMM); both well resolved (sigma >= spacing) so the step is not
    dominated by close encounters."""
    import paper_1106_5273_b200 as P
    if images == 0:
        x, a, s = synth.random_cloud(60, seed=1106, sigma=0.2)
        x = (x * np.float32(0.2)).astype(np.float32)
        a = (a * np.float32(50.0)).astype(np.float32)
    else:
        x, a, s = synth.taylor_green(8)
    xg, ag, sg = x.copy(), a.copy(), s.copy()
    f = P.FMM(images=images, ncrit=64 if images == 0 else 16)
    dt, nu = 0.02, 0.01
    f.step(xg, ag, sg, dt=dt, nu=nu)
    xo, ao, so = oracle_mod.rk2_step(x, a, s, dt, nu, images=images)
    dx = np.linalg.norm(xg - xo) / np.linalg.norm(xo - x)       # relative to the displacement
    da = np.linalg.norm(ag - ao) / np.linalg.norm(ao - a)       # relative to the strength change
    assert dx <= 1e-3 and da <= 1e-3, (dx, da)
    assert np.allclose(sg ** 2, so ** 2, rtol=1e-6)
    f.close()
