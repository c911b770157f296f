"""Worker of tests/test_gpu_poison.py (run as a subprocess, so FMM_POISON is
read at library load): evaluates a set of small cases through the C ABI that
together take every kernel of the path -- full periodic path (C1-sized),
tensor-core M2L on four levels, an adaptive free-space cloud (register M2L,
small-leaf P2P variants), a jittered lattice (tensor M2L subset cells), host
buffers, one RK2 step (NEXT-1), strength-free targets (NEXT-2) and an RBF
reinitialisation (NEXT-4) -- and writes every output to an .npz file.

usage: python tests/poison_worker.py OUT.npz
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1106_5273_b200 as P  # noqa: E402
import synth  # noqa: E402


def dev(*arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


def evaluate(x, a, s, host=False, **cfg):
    f = P.FMM(**cfg)
    n = len(x)
    if host:
        f.set_particles(np.ascontiguousarray(x), np.ascontiguousarray(a), np.ascontiguousarray(s))
        u = np.empty((n, 3), np.float32)
        d = np.empty((n, 3), np.float32)
        f.evaluate(u, d)
    else:
        xd, ad, sd = dev(x, a, s)
        f.set_particles(xd, ad, sd)
        u = torch.empty((n, 3), device="cuda")
        d = torch.empty((n, 3), device="cuda")
        f.evaluate(u, d)
        u, d = u.cpu().numpy(), d.cpu().numpy()
    st = f.stats()
    f.close()
    return u, d, st


def main():
    want = 1 if os.environ.get("FMM_POISON", "0") not in ("", "0") else 0
    assert P.fmm_debug_mode() & 1 == want, "FMM_POISON not in effect"
    out = {}
    cases = {
        "c1_tg16_k3": (synth.taylor_green(16), dict(images=3)),
        "tg32_ncrit8_k2": (synth.taylor_green(32), dict(images=2, ncrit=8)),
        "cloud_free": (synth.random_cloud(6000, seed=11, sigma=0.05), dict(images=0, ncrit=24)),
        "clustered_k1": (synth.clustered_cloud(5000, sigma=0.02), dict(images=1, ncrit=32)),
        "jitter20_k1": (synth.jittered_lattice(20), dict(images=1)),
        "leaf_first": (synth.random_cloud(3000, seed=5, sigma=0.05), dict(images=1, ncrit=16, traversal=1)),
    }
    for name, ((x, a, s), cfg) in cases.items():
        u, d, st = evaluate(x, a, s, **cfg)
        out[name + "_u"], out[name + "_s"] = u, d
        out[name + "_lists"] = np.array([st["p2p_list"], st["m2l_list"], st["m2l_tc_list"]], dtype=np.int64)
    x, a, s = synth.taylor_green(12)
    u, d, _ = evaluate(x, a, s, host=True, images=3)
    out["host_u"], out["host_s"] = u, d
    # NEXT-1: one midpoint-RK2 step
    x, a, s = synth.taylor_green(12)
    xd, ad, sd = dev(x, a, s)
    f = P.FMM(images=1)
    f.step(xd, ad, sd, 0.5 * float(s[0]), 0.01)
    out["step_x"], out["step_a"], out["step_s"] = xd.cpu().numpy(), ad.cpu().numpy(), sd.cpu().numpy()
    f.close()
    # NEXT-2: strength-free targets
    x, a, s = synth.taylor_green(12)
    y = synth.random_cloud(500, seed=3)[0]
    xd, ad, sd, yd = dev(x, a, s, y)
    u = torch.empty((len(y), 3), device="cuda")
    f = P.FMM(images=1)
    f.evaluate_targets(xd, ad, sd, yd, u)
    out["targets_u"] = u.cpu().numpy()
    f.close()
    # NEXT-4: RBF reinitialisation of a jittered field onto the lattice
    xj, aj, sj = synth.jittered_lattice(10, amp=0.2)
    yl = synth.taylor_green(10)[0]
    xd, ad, sd, yd = dev(xj, aj, sj, yl)
    beta = torch.empty((len(yl), 3), device="cuda")
    f = P.FMM(images=1)
    it, res = f.rbf_reinit(xd, ad, sd, yd, float(sj[0]), beta, tol=1e-4, maxit=400)
    out["rbf_beta"] = beta.cpu().numpy()
    out["rbf_it"] = np.array([it], dtype=np.int64)
    f.close()
    np.savez(sys.argv[1], **out)
    print("ok", len(out))


if __name__ == "__main__":
    main()
