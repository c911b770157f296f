"""Pins of the oracle's normalised coefficient dumps (reading Z18) and of
its target-subset near field.

Z18: the oracle stores physical M, L and dumps M~_n = M_n / s^n and
L~_n = L_n s^(n+1) (s = cell side) -- the scaling the GPU's coefficients are
compared in.  The pins undo the scaling for every degree n and check the
result against something other than the dump itself:

* M~ -> M evaluated at far points with or_m2p equals the direct Laplace sum
  sum_j alpha_j,c / |y - x_j| of the cell's particles (the expansion of
  1/|x - y|), so a wrong power of s at any n >= 1 shows.
* L~ -> L shifted to the leaf's particles with or_l2p_derivs gives
  grad phi and the Hessian; u_far = (1/4 pi) eps grad phi and
  s_far = (1/4 pi) alpha_d eps H_db (8c-2 item 16) reproduce the oracle's own
  far field (itself pinned against direct sums in test_oracle_fmm.py).

near_subset (used by the C3-scale GPU parity test) is pinned against the
full evaluation: bit-identical near field for the selected leaves, and the
same number of P2P entries as the full list restricted to them.
"""
import numpy as np
import pytest

import synth

K4 = 1.0 / (4.0 * np.pi)


def _geometry(f):
    lo, L = f.box()
    cells = f.cells()
    side = L / (2.0 ** cells[:, 0])
    ctr = lo[None, :] + (cells[:, 1:4] + 0.5) * side[:, None]
    return cells, side, ctr


def _nm(P):
    return [(n, m) for n in range(P) for m in range(n + 1)]


@pytest.mark.parametrize("case", ["tg12_k2", "rand_free"])
def test_multipole_normalisation_all_degrees(oracle_mod, case):
    P = 10
    if case == "tg12_k2":
        x, a, s = synth.taylor_green(12)
        f = oracle_mod.OracleFMM(x, a, s, order=P, ncrit=16, images=2)
    else:
        x, a, s = synth.random_cloud(1500, seed=11, sigma=0.05)
        f = oracle_mod.OracleFMM(x, a, s, order=P, ncrit=24, images=0)
    Mt = f.multipoles()
    cells, side, ctr = _geometry(f)
    xw = f.positions()
    _, perm = f.keys()
    deg = np.array([n for n, _ in _nm(P)])
    rng = np.random.default_rng(5)
    checked = 0
    for c in rng.choice(len(cells), size=min(25, len(cells)), replace=False):
        b, cnt = cells[c, 4], cells[c, 5]
        if cnt == 0:
            continue
        src = xw[perm[b:b + cnt]]
        q = a.astype(np.float64)[perm[b:b + cnt]]
        for _ in range(3):
            dirv = rng.normal(size=3)
            y = ctr[c] + 3.0 * side[c] * dirv / np.linalg.norm(dirv)      # |y - c| = 3 s: n >= 1 terms matter
            for comp in range(3):
                M = Mt[c, comp] * side[c] ** deg                            # undo Z18
                phi = oracle_mod.m2p(P, M, y - ctr[c])
                ref = np.sum(q[:, comp] / np.linalg.norm(y[None, :] - src, axis=1))
                scale = np.sum(np.abs(q[:, comp]) / np.linalg.norm(y[None, :] - src, axis=1))
                assert abs(phi - ref) <= 1e-6 * scale, (c, comp, phi, ref)
                # and the wrong scaling (no Z18 undo) would not pass
                if comp == 0 and np.abs(Mt[c, comp][deg >= 1]).max() > 1e-3 * np.abs(Mt[c, comp]).max():
                    phi_bad = oracle_mod.m2p(P, Mt[c, comp], y - ctr[c])
                    assert abs(phi_bad - ref) > 100 * abs(phi - ref) + 1e-9 * scale
        checked += 1
    assert checked >= 10


def test_local_normalisation_reproduces_far_field(oracle_mod):
    P = 10
    x, a, s = synth.taylor_green(12)
    f = oracle_mod.OracleFMM(x, a, s, order=P, ncrit=16, images=2)
    r = f.evaluate()
    Lt = f.locals()
    cells, side, ctr = _geometry(f)
    xw = f.positions()
    _, perm = f.keys()
    a64 = a.astype(np.float64)
    deg = np.array([n for n, _ in _nm(P)])
    leaves = np.nonzero(cells[:, 9])[0]
    rng = np.random.default_rng(3)
    for c in rng.choice(leaves, size=12, replace=False):
        b, cnt = cells[c, 4], cells[c, 5]
        for i in perm[b:b + cnt]:
            g = np.zeros((3, 3))
            H = np.zeros((3, 3, 3))
            for comp in range(3):
                L = Lt[c, comp] / side[c] ** (deg + 1)                      # undo Z18
                _, gr, h = oracle_mod.l2p_derivs(P, L, xw[i] - ctr[c])
                g[comp] = gr
                hx = np.array([[h[0], h[3], h[4]], [h[3], h[1], h[5]], [h[4], h[5], h[2]]])
                H[comp] = hx
            u = K4 * np.array([g[2, 1] - g[1, 2], g[0, 2] - g[2, 0], g[1, 0] - g[0, 1]])
            sv = K4 * np.array([a64[i] @ (H[2][:, 1] - H[1][:, 2]), a64[i] @ (H[0][:, 2] - H[2][:, 0]),
                                a64[i] @ (H[1][:, 0] - H[0][:, 1])])
            nu = np.linalg.norm(r["u_far"][i]) + 1e-30
            ns = np.linalg.norm(r["s_far"][i]) + 1e-30
            assert np.linalg.norm(u - r["u_far"][i]) <= 1e-10 * nu + 1e-16
            assert np.linalg.norm(sv - r["s_far"][i]) <= 1e-10 * ns + 1e-16


@pytest.mark.parametrize("case", ["c1_tg16_k3", "rand_k1_leaf_first", "rand_free"])
def test_near_subset_equals_full_evaluation(oracle_mod, case):
    if case == "c1_tg16_k3":
        x, a, s = synth.taylor_green(16)
        kw = dict(images=3, ncrit=64)
    elif case == "rand_k1_leaf_first":
        x, a, s = synth.random_cloud(2500, seed=5273, sigma=0.05)
        kw = dict(images=1, ncrit=32, traversal=1)
    else:
        x, a, s = synth.random_cloud(3000, seed=1106, sigma=0.05)
        kw = dict(images=0, ncrit=24)
    f = oracle_mod.OracleFMM(x, a, s, order=10, **kw)
    r = f.evaluate()
    cells = f.cells()
    p2p = f.p2p_list()
    leaves = np.nonzero(cells[:, 9])[0]
    sel = np.random.default_rng(9).choice(leaves, size=min(12, len(leaves)), replace=False)
    g = oracle_mod.OracleFMM(x, a, s, order=10, **kw)      # fresh object: nothing traversed before
    pidx, un, sn, ne = g.near_subset(sel)
    assert len(pidx) == int(cells[sel, 5].sum())
    assert np.array_equal(np.sort(pidx), np.sort(np.concatenate(
        [g.keys()[1][cells[c, 4]:cells[c, 4] + cells[c, 5]] for c in sel])))
    assert np.array_equal(un, r["u_near"][pidx]) and np.array_equal(sn, r["s_near"][pidx])
    assert ne == int(np.isin(p2p[:, 0], sel).sum())
