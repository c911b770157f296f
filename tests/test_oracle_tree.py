"""Pins of the oracle's Morton keys, octree and dual tree traversal.

* Keys: min corner -> 0; level-1 octant (x > mid) -> 1; every
  level's octant digit equals the octant found by recursive midpoint
  comparisons (geometric construction).
* Tree: 8 octant centres with ncrit = 1 -> 8 leaves; children
  partition parents; leaves partition particles; bounds contain particles;
  leaf iff count <= ncrit; permutation is a bijection.
* Traversal (Alg. 1-2): the counting kernel covers every target
  exactly N * 27^k times in both traversal orders; every M2L
  pair satisfies the MAC (checked in floating point); theta -> 0 gives an
  all-P2P list.
"""
import numpy as np
import pytest

import synth


def _fmm(oracle_mod, x, a, s, **kw):
    return oracle_mod.OracleFMM(x, a, s, **kw)


def test_key_conventions(oracle_mod):
    x = np.array([[-np.pi, -np.pi, -np.pi], [1.0, -1.0, -1.0], [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]])
    f = _fmm(oracle_mod, x, np.zeros_like(x), np.ones(4), images=1, ncrit=1)
    keys, perm = f.keys()
    k = dict(zip(perm, keys))
    assert k[0] == 0
    assert int(k[1]) >> 60 == 1 and int(k[2]) >> 60 == 2 and int(k[3]) >> 60 == 4


def test_keys_match_recursive_midpoint_octants(oracle_mod):
    x, a, s = synth.random_cloud(3000, seed=1106)
    f = _fmm(oracle_mod, x, a, s, images=1)
    lo, L = f.box()
    keys, perm = f.keys()
    xs = f.positions()[perm]
    for i in range(0, 3000, 37):
        p = xs[i]
        clo = np.array(lo, dtype=np.float64)
        side = L
        for lev in range(1, 22):
            side = side / 2
            mid = clo + side
            bits = (p >= mid).astype(int)
            digit = (int(keys[i]) >> (3 * (21 - lev))) & 7
            assert digit == bits[0] | (bits[1] << 1) | (bits[2] << 2)
            clo = clo + bits * side
    assert np.all(np.diff(keys.astype(np.float64)) >= 0)
    assert np.array_equal(np.sort(perm), np.arange(3000))


def test_eight_octant_centres(oracle_mod):
    c = np.array([[(i & 1) * 2 - 1, ((i >> 1) & 1) * 2 - 1, ((i >> 2) & 1) * 2 - 1] for i in range(8)]) * np.pi / 2
    f = _fmm(oracle_mod, c, np.zeros((8, 3)), np.ones(8), images=1, ncrit=1)
    cells = f.cells()
    assert len(cells) == 9
    assert cells[0, 9] == 0 and np.all(cells[1:, 0] == 1) and np.all(cells[1:, 9] == 1)


@pytest.mark.parametrize("gen,ncrit", [("tg", 64), ("rand", 32), ("jit", 16)])
def test_tree_invariants(oracle_mod, gen, ncrit):
    if gen == "tg":
        x, a, s = synth.taylor_green(12)
    elif gen == "rand":
        x, a, s = synth.random_cloud(5000, seed=5273)
    else:
        x, a, s = synth.jittered_lattice(10)
    f = _fmm(oracle_mod, x, a, s, images=1, ncrit=ncrit)
    cells = f.cells()
    lo, L = f.box()
    keys, perm = f.keys()
    xs = f.positions()[perm]
    n = len(x)
    covered = np.zeros(n, dtype=int)
    for c, (lev, qx, qy, qz, b, cnt, par, cb, nch, leaf) in enumerate(cells):
        side = L / 2 ** lev
        pts = xs[b:b + cnt]
        q = np.array([qx, qy, qz])
        assert np.all(pts >= lo + q * side - 1e-12) and np.all(pts <= lo + (q + 1) * side + 1e-12)
        assert bool(leaf) == (cnt <= ncrit or lev == 21)
        if leaf:
            covered[b:b + cnt] += 1
        else:
            ch = cells[cb:cb + nch]
            assert np.all(ch[:, 6] == c) and np.all(ch[:, 0] == lev + 1)
            assert ch[0, 4] == b and np.sum(ch[:, 5]) == cnt
            assert np.all(ch[1:, 4] == ch[:-1, 4] + ch[:-1, 5])
    assert np.all(covered == 1)


@pytest.mark.parametrize("images", [0, 1, 2])
@pytest.mark.parametrize("traversal", [0, 1])
@pytest.mark.parametrize("theta", [(3, 10), (1, 2), (4, 5)])
def test_traversal_coverage_exact(oracle_mod, images, traversal, theta):
    x, a, s = synth.random_cloud(1500, seed=1106)
    f = _fmm(oracle_mod, x, a, s, images=images, traversal=traversal, theta=theta, ncrit=16)
    cov = f.coverage()
    assert np.all(cov == len(x) * 27 ** images)


def test_m2l_pairs_satisfy_mac_and_p2p_pairs_are_leaves(oracle_mod):
    x, a, s = synth.taylor_green(16)
    f = _fmm(oracle_mod, x, a, s, images=3, theta=(1, 2), ncrit=64)
    cells = f.cells()
    lo, L = f.box()
    m2l = f.m2l_list()
    p2p = f.p2p_list()
    lev = cells[:, 0]
    ctr = lo + (cells[:, 1:4] + 0.5) * (L / 2.0 ** lev)[:, None]
    rad = np.sqrt(3) / 2 * L / 2.0 ** lev
    img = np.stack([m2l[:, 2] % 3 - 1, (m2l[:, 2] // 3) % 3 - 1, m2l[:, 2] // 9 - 1], -1)
    R = np.linalg.norm(ctr[m2l[:, 0]] - ctr[m2l[:, 1]] - img * L, axis=1)
    assert np.all(rad[m2l[:, 0]] + rad[m2l[:, 1]] < 0.5 * R * (1 + 1e-12))
    # reading Z5: accepted pairs are >= 5.7 sigma apart for sigma = h (closest particles)
    h = 2 * np.pi / 16
    assert np.all(R - rad[m2l[:, 0]] - rad[m2l[:, 1]] > 5.7 * h)
    assert np.all(cells[p2p[:, 0], 9] == 1) and np.all(cells[p2p[:, 1], 9] == 1)
    # lists are sets: canonical order and no duplicates
    for lst in (m2l, p2p):
        key = (lst[:, 0] * 2 ** 22 + lst[:, 1]) * 32 + lst[:, 2]
        assert np.all(np.diff(key) > 0)


def test_theta_to_zero_is_all_p2p_and_equals_direct(oracle_mod):
    x, a, s = synth.random_cloud(400, seed=5273)
    f = _fmm(oracle_mod, x, a, s, images=1, theta=(1, 64), ncrit=16)
    assert len(f.m2l_list()) == 0
    r = f.evaluate()
    u, st = oracle_mod.direct(x, a, x, a, s, images=1)
    assert oracle_mod.rel_l2(r["u"], u) < 1e-13 and oracle_mod.rel_l2(r["s"], st) < 1e-13
    assert np.all(r["u_far"] == 0)
