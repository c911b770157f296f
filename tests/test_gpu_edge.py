"""GPU parity on edge cases and adaptive trees (CUDA path through the C ABI vs
the CPU oracle): a single particle, a root leaf, coincident particles (Z7),
a clustered distribution (deep adaptive tree, lists mixing levels), variable
per-particle sigma (Z4), particles outside the periodic cell (a1 wrap),
a leaf forced to level 21 (more than ncrit coincident keys)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _both(oracle_mod, x, a, s, **cfg):
    from gpu_util import GpuRun
    g = GpuRun(x, a, s, **cfg)
    o = oracle_mod.OracleFMM(x, a, s, order=cfg.get("order", 10), theta=cfg.get("theta", (1, 2)),
                             ncrit=cfg.get("ncrit", 64), images=cfg.get("images", 3),
                             traversal=cfg.get("traversal", 0))
    return g, o


def _check_structure(g, o):
    kg, pg = g.keys()
    ko, po = o.keys()
    assert np.array_equal(kg, ko) and np.array_equal(pg, po)
    assert np.array_equal(g.cells(), o.cells())
    p2p, m2l = g.lists()
    assert np.array_equal(p2p, o.p2p_list()) and np.array_equal(m2l, o.m2l_list())


def _check_fields(oracle_mod, g, o, near_tol=1e-5, tol=1e-5):
    un, sn = g.evaluate(parts=1)
    u, s = g.evaluate()
    r = o.evaluate()
    if np.linalg.norm(r["u_near"]) > 0:
        assert oracle_mod.rel_l2(un, r["u_near"]) <= near_tol
    if np.linalg.norm(r["s_near"]) > 0:
        assert oracle_mod.rel_l2(sn, r["s_near"]) <= near_tol
    if np.linalg.norm(r["u"]) > 0:
        assert oracle_mod.rel_l2(u, r["u"]) <= tol
        assert oracle_mod.rel_l2(s, r["s"]) <= tol
    return u, s, r


@pytest.mark.parametrize("images", [0, 3])
def test_single_particle(oracle_mod, images):
    x = np.array([[0.3, -0.2, 1.1]], np.float32)
    a = np.array([[0.1, 0.2, -0.3]], np.float32)
    s = np.array([0.2], np.float32)
    g, o = _both(oracle_mod, x, a, s, images=images)
    _check_structure(g, o)
    u, st = g.evaluate()
    r = o.evaluate()
    assert np.allclose(u, r["u"], atol=1e-9) and np.allclose(st, r["s"], atol=1e-9)
    g.close()


def test_root_leaf_all_p2p(oracle_mod):
    x, a, s = synth.random_cloud(50, seed=1106, sigma=0.3)
    g, o = _both(oracle_mod, x, a, s, images=1, ncrit=64)
    _check_structure(g, o)
    assert len(o.m2l_list()) == 0
    _check_fields(oracle_mod, g, o)
    g.close()


def test_coincident_particles_contribute_nothing_to_each_other(oracle_mod):
    x, a, s = synth.random_cloud(400, seed=5273, sigma=0.1)
    x[1] = x[0]
    x[7] = x[0]
    x[200] = x[100]
    g, o = _both(oracle_mod, x, a, s, images=1, ncrit=16)
    _check_structure(g, o)
    _check_fields(oracle_mod, g, o)
    g.close()


def test_clustered_adaptive_tree(oracle_mod):
    """A dense Gaussian cluster inside a sparse background: a deep adaptive
    tree whose lists pair cells several levels apart."""
    rng = np.random.default_rng(1106)
    bg = -np.pi + 2 * np.pi * rng.random((1500, 3))
    cl = 0.6 + 0.05 * rng.standard_normal((2500, 3))
    x = np.concatenate([bg, cl]).astype(np.float32)
    a = (rng.standard_normal((4000, 3)) * 1e-3).astype(np.float32)
    s = np.full(4000, 0.004, np.float32)
    g, o = _both(oracle_mod, x, a, s, images=0, ncrit=16)
    _check_structure(g, o)
    cells = o.cells()
    m2l = o.m2l_list()
    assert cells[:, 0].max() >= 7
    assert np.abs(cells[m2l[:, 0], 0] - cells[m2l[:, 1], 0]).max() >= 1
    u, st, r = _check_fields(oracle_mod, g, o)
    idx = rng.choice(4000, 300, replace=False)
    u0, s0 = oracle_mod.direct(x[idx], a[idx], x, a, s, images=0)
    assert oracle_mod.rel_l2(u[idx], u0) <= 1e-3 and oracle_mod.rel_l2(st[idx], s0) <= 1e-3
    g.close()


def test_variable_sigma(oracle_mod):
    x, a, s = synth.random_cloud(3000, seed=7, sigma=0.05)
    s = (0.02 + 0.06 * np.random.default_rng(7).random(3000)).astype(np.float32)
    g, o = _both(oracle_mod, x, a, s, images=1, ncrit=32)
    _check_structure(g, o)
    _check_fields(oracle_mod, g, o)
    g.close()


def test_positions_outside_cell_are_wrapped(oracle_mod):
    x, a, s = synth.taylor_green(12)
    xs = x.copy()
    xs[::7, 0] += np.float32(2 * np.pi)
    xs[::5, 2] -= np.float32(2 * np.pi)
    g, o = _both(oracle_mod, xs, a, s, images=3, ncrit=32)
    _check_structure(g, o)
    assert np.array_equal(o.positions(), oracle_mod.OracleFMM(xs, a, s, images=3).positions())
    _check_fields(oracle_mod, g, o)
    g.close()


def test_level21_leaf_with_more_than_ncrit(oracle_mod):
    x, a, s = synth.random_cloud(200, seed=3, sigma=0.05)
    x[:40] = x[0] + np.float32(1e-7) * np.arange(40, dtype=np.float32)[:, None]
    g, o = _both(oracle_mod, x, a, s, images=1, ncrit=8)
    _check_structure(g, o)
    cells = o.cells()
    assert cells[:, 0].max() == 21 and cells[cells[:, 0] == 21, 5].max() > 8
    _check_fields(oracle_mod, g, o, near_tol=1e-4, tol=1e-4)
    g.close()
