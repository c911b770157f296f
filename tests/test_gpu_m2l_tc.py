"""Tensor-core M2L (csrc/m2l_tc.cu, 3xTF32 on tcgen05) vs the register M2L
(csrc/m2l.cu, FP32 CUDA cores) and vs the CPU oracle.

The tensor path takes the levels whose cells share one offset set (uniform
periodic lattices); everything else stays on the register kernel.  Both
compute the same M2L of P:228 with the same lists, so the local expansions
agree to FP32 rounding, and the full field keeps the oracle bars.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _run(x, a, s, path, **cfg):
    from gpu_util import GpuRun
    g = GpuRun(x, a, s, m2l_path=path, **cfg)
    u, st = g.evaluate()
    M, L = g.expansions()
    stats = g.stats()
    lists = g.lists()
    g.close()
    return u, st, L, stats, lists


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("side,cfg", [(32, dict(images=3, ncrit=8)), (64, dict(images=3)),
                                      (32, dict(images=1, ncrit=32)), (48, dict(images=2, ncrit=32))])
def test_tc_matches_register_kernel(oracle_mod, side, cfg):
    x, a, s = synth.taylor_green(side)
    u0, s0, L0, st0, l0 = _run(x, a, s, 1, **cfg)
    u1, s1, L1, st1, l1 = _run(x, a, s, 0, **cfg)
    assert st0["m2l_tc_list"] == 0
    assert st1["m2l_tc_list"] > 0, "uniform lattice should take the tensor path"
    assert np.array_equal(l0[1], l1[1])
    # local expansions of every cell: FP32-level agreement (which of the two is
    # closer to the double-precision oracle: test_tc_full_field_vs_oracle)
    assert _rel(L1, L0) <= 1e-5
    assert _rel(u1, u0) <= 1e-5 and _rel(s1, s0) <= 1e-5


@pytest.mark.parametrize("side,cfg", [(32, dict(images=3, ncrit=8)), (32, dict(images=1, ncrit=32))])
def test_tc_full_field_vs_oracle(oracle_mod, side, cfg):
    x, a, s = synth.taylor_green(side)
    u, st, L, stats, _ = _run(x, a, s, 0, **cfg)
    u0, s0, L0, _, _ = _run(x, a, s, 1, **cfg)
    assert stats["m2l_tc_list"] >= 0.6 * stats["m2l_list"]
    o = oracle_mod.OracleFMM(x, a, s, order=10, theta=(1, 2), ncrit=cfg.get("ncrit", 64), images=cfg["images"])
    r = o.evaluate()
    Lo = o.locals()
    print("L err tensor %.2e register %.2e; u err %.2e / %.2e" % (_rel(L, Lo), _rel(L0, Lo),
                                                               oracle_mod.rel_l2(u, r["u"]),
                                                               oracle_mod.rel_l2(u0, r["u"])))
    # the tensor path is at least as accurate as the FP32 register kernel
    assert _rel(L, Lo) <= 1e-5 and _rel(L, Lo) <= 1.5 * _rel(L0, Lo)
    assert oracle_mod.rel_l2(u, r["u"]) <= 2e-5 and oracle_mod.rel_l2(st, r["s"]) <= 2e-5
    print("L err tensor %.2e register %.2e; u err %.2e / %.2e" % (_rel(L, Lo), _rel(L0, Lo),
                                                               oracle_mod.rel_l2(u, r["u"]),
                                                               oracle_mod.rel_l2(u0, r["u"])))


def test_tc_declines_adaptive_tree(oracle_mod):
    x, a, s = synth.random_cloud(4000, seed=11, sigma=0.05)
    u0, s0, L0, st0, _ = _run(x, a, s, 1, images=1, ncrit=16)
    u1, s1, L1, st1, _ = _run(x, a, s, 0, images=1, ncrit=16)
    assert st1["m2l_tc_list"] < st1["m2l_list"]
    assert _rel(u1, u0) <= 1e-5 and _rel(s1, s0) <= 1e-5
