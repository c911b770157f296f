"""End-to-end pins of the oracle FMM (c-2) against the direct sum (c-1) and
closed forms.

* Free space, random cloud: rel-L2 <= 1e-3 at p = 10 (BASELINE.json bar),
  error decreasing monotonically in p.
* Periodic k = 1 vs the explicit 27-image direct sum; k = 2 vs the
  explicit 9^3-image direct sum (periodic far-field layer, Z14).
* C1 Taylor-Green 16^3, k = 3: vs the closed form (Z26).
* Invariants: root monopole = sum(alpha); translation invariance
  within FMM error; leaf-first traversal gives the same field.
"""
import numpy as np
import pytest

import synth
from test_oracle_kernel import _tg_closed_form


def test_free_space_random_vs_direct_and_p_convergence(oracle_mod):
    x, a, s = synth.random_cloud(2000, seed=1106, sigma=0.1)  # Z5
    u0, s0 = oracle_mod.direct(x, a, x, a, s, images=0)
    eu, es = [], []
    for p in (4, 6, 8, 10, 12):
        r = oracle_mod.OracleFMM(x, a, s, order=p, theta=(1, 2), ncrit=32, images=0).evaluate()
        eu.append(oracle_mod.rel_l2(r["u"], u0))
        es.append(oracle_mod.rel_l2(r["s"], s0))
    assert all(b < c for c, b in zip(eu, eu[1:])), eu
    assert all(b < c for c, b in zip(es, es[1:])), es
    assert eu[3] < 1e-3 and es[3] < 1e-3


@pytest.mark.parametrize("traversal", [0, 1])
def test_periodic_k1_vs_explicit_images(oracle_mod, traversal):
    x, a, s = synth.random_cloud(600, seed=5273, sigma=0.05)  # Z5: sigma << M2L separation
    u0, s0 = oracle_mod.direct(x, a, x, a, s, images=1)
    r = oracle_mod.OracleFMM(x, a, s, order=10, ncrit=16, images=1, traversal=traversal).evaluate()
    assert oracle_mod.rel_l2(r["u"], u0) < 1e-3
    assert oracle_mod.rel_l2(r["s"], s0) < 1e-3


def test_periodic_k2_far_layer_vs_explicit_images(oracle_mod):
    x, a, s = synth.random_cloud(300, seed=1106, sigma=0.05)  # Z5
    a = a - a.mean(0)            # sum alpha = 0 as for a periodic vorticity field
    u0, s0 = oracle_mod.direct(x, a, x, a, s, images=2)
    r = oracle_mod.OracleFMM(x, a, s, order=12, ncrit=8, images=2).evaluate()
    assert oracle_mod.rel_l2(r["u"], u0) < 1e-4
    assert oracle_mod.rel_l2(r["s"], s0) < 1e-3
    # and the far layer matters: dropping it (k = 1) is visibly worse
    r1 = oracle_mod.OracleFMM(x, a, s, order=12, ncrit=8, images=1).evaluate()
    assert oracle_mod.rel_l2(r1["u"], u0) > 3 * oracle_mod.rel_l2(r["u"], u0)


def test_c1_taylor_green_closed_form(oracle_mod):
    x, a, s = synth.taylor_green(16)
    f = oracle_mod.OracleFMM(x, a, s, order=10, theta=(1, 2), ncrit=64, images=3)
    r = f.evaluate()
    uc, sc = _tg_closed_form(x.astype(np.float64), a.astype(np.float64), float(s[0]))
    assert oracle_mod.rel_l2(r["u"], uc) < 1e-4
    assert oracle_mod.rel_l2(r["s"], sc) < 1e-3
    M = f.multipoles()
    assert np.allclose(M[0, :, 0].real, a.astype(np.float64).sum(0), atol=1e-12)   # root monopole
    assert np.abs(r["u"].mean(0)).max() < 1e-8


def test_translation_invariance_free_space(oracle_mod):
    x, a, s = synth.random_cloud(1200, seed=7, sigma=0.1)
    r1 = oracle_mod.OracleFMM(x, a, s, order=10, ncrit=32, images=0).evaluate()
    shift = np.array([0.37, -1.21, 2.05], dtype=np.float32)
    r2 = oracle_mod.OracleFMM(x + shift, a, s, order=10, ncrit=32, images=0).evaluate()
    assert oracle_mod.rel_l2(r2["u"], r1["u"]) < 1e-3
    assert oracle_mod.rel_l2(r2["s"], r1["s"]) < 1e-3
