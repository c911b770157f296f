"""NEXT-2: velocity at strength-free target points through
fmm_evaluate_targets, against the oracle FMM on the same union (identical tree
and lists) and against the oracle's direct sum."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _targets(nt, seed):
    rng = np.random.default_rng(seed)
    return (-np.pi + 2 * np.pi * rng.random((nt, 3))).astype(np.float32)


@pytest.mark.parametrize("side,nt,images", [(16, 500, 3), (12, 2000, 1)])
def test_targets_match_oracle(oracle_mod, side, nt, images):
    import torch
    import paper_1106_5273_b200 as P
    x, a, s = synth.taylor_green(side)
    y = _targets(nt, 1106 + nt)
    f = P.FMM(images=images)
    u = torch.empty((nt, 3), dtype=torch.float32, device="cuda")
    f.evaluate_targets(*(torch.from_numpy(v).cuda() for v in (x, a, s, y)), u)
    ug = u.cpu().numpy().astype(np.float64)
    # the oracle FMM on the union: targets as zero-strength particles with sigma = 1
    xu = np.concatenate([x, y])
    au = np.concatenate([a, np.zeros_like(y)])
    su = np.concatenate([s, np.ones(nt, np.float32)])
    o = oracle_mod.OracleFMM(xu, au, su, order=10, theta=(1, 2), ncrit=64, images=images)
    r = o.evaluate()
    assert oracle_mod.rel_l2(ug, r["u"][len(x):]) <= 2e-5
    # and the plain direct sum at the targets (FMM truncation bar; the image
    # lattice sum is only affordable for k <= 1)
    if images <= 1:
        ud, sd = oracle_mod.direct(y, np.zeros_like(y), x, a, s, images=images)
        assert oracle_mod.rel_l2(ug, ud) <= 1e-3
        assert np.abs(sd).max() == 0.0               # no stretching without strength
    f.close()


def test_targets_host_pointers_and_empty(oracle_mod):
    import paper_1106_5273_b200 as P
    x, a, s = synth.taylor_green(8)
    y = _targets(64, 7)
    f = P.FMM(images=1)
    u = np.zeros((64, 3), np.float32)
    f.evaluate_targets(x, a, s, y, u)                # host buffers are staged by the library
    ud, _ = oracle_mod.direct(y, np.zeros_like(y), x, a, s, images=1)
    assert oracle_mod.rel_l2(u.astype(np.float64), ud) <= 1e-3
    u0 = np.zeros((0, 3), np.float32)
    f.evaluate_targets(x, a, s, np.zeros((0, 3), np.float32), u0)
    f.close()
