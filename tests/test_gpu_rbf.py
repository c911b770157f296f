"""NEXT-4 on the GPU (fmm_rbf_reinit): the Gaussian sums (1)/(2)
of rbf.cu over the P2P lists and the CG solve, against the oracle's dense
solve (tests/test_oracle_rbf.py pins it) and the Taylor-Green closed form."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def _gpu(x, a, s, y, s0, tol=1e-7, maxit=500, **kw):
    import torch
    import paper_1106_5273_b200 as P
    f = P.FMM(images=3, order=10, device=0, **kw)
    dev = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).cuda()
    beta = torch.empty((len(y), 3), device="cuda")
    it, res = f.rbf_reinit(dev(x), dev(a), dev(s), dev(y), s0, beta, tol=tol, maxit=maxit)
    return f, beta.cpu().numpy().astype(np.float64), it, res


def test_rbf_taylor_green_closed_form_and_oracle():
    n = 12
    x, a, s = synth.taylor_green(n)
    h = 2 * np.pi / n
    f, beta, it, res = _gpu(x, a, s, x, 1.1 * h, tol=1e-6)
    f.close()
    want = np.exp(1.5 * ((1.1 * h) ** 2 - h ** 2)) * a.astype(np.float64)
    print("TG: iters %d resid %.2e closed %.2e" % (it, res, oracle.rel_l2(beta, want)))
    assert res <= 1e-6 and it <= 5, (it, res)         # one Fourier mode: CG converges at once
    assert oracle.rel_l2(beta, want) <= 1e-5
    ref = oracle.rbf_reinit(x, a, s, x, 1.1 * h, images=1)
    assert oracle.rel_l2(beta, ref) <= 1e-5


def test_rbf_jittered_field_vs_oracle():
    """A smooth field carried by jittered particles onto the lattice (sigma0 = h).
    The collocation matrix is ill-conditioned (kappa ~ e^{3 pi^2 / 2}), so the
    strengths themselves are defined only loosely (3.6% from the oracle's exact
    solve at residual 1e-5); what is well-posed is checked: the interpolation
    condition (the new field at the sites, evaluated in double by the oracle)
    and the total strength."""
    n = 12
    x, a, s = synth.jittered_lattice(n)
    y, _ya, _ys = synth.taylor_green(n)
    h = 2 * np.pi / n
    f, beta, it, res = _gpu(x, a, s, y, h, tol=1e-5, maxit=400)
    f.close()
    b_ref = oracle.gauss_field(y, x, a, s, images=1)
    b_gpu = oracle.gauss_field(y, y, beta, np.full(len(y), h), images=1)
    print("jittered: iters %d resid %.2e field %.2e" % (it, res, oracle.rel_l2(b_gpu, b_ref)))
    assert res <= 1e-5
    assert oracle.rel_l2(b_gpu, b_ref) <= 3e-5
    assert np.abs(beta.sum(0) - a.astype(np.float64).sum(0)).max() <= 1e-4 * np.abs(a).sum()


def test_rbf_context_holds_the_sites():
    """After the reinitialisation the context evaluates the new field: equal to a
    fresh set_particles(y, beta, sigma0) + evaluate (same tree, same strengths)."""
    import torch
    import paper_1106_5273_b200 as P
    n = 12
    x, a, s = synth.jittered_lattice(n)
    y, _ya, _ys = synth.taylor_green(n)
    h = 2 * np.pi / n
    f, beta, _it, _res = _gpu(x, a, s, y, h, tol=1e-4, maxit=300)
    u1 = torch.empty((len(y), 3), device="cuda")
    d1 = torch.empty((len(y), 3), device="cuda")
    f.evaluate(u1, d1)
    f.close()
    g = P.FMM(images=3, order=10, device=0)
    g.set_particles(torch.from_numpy(y).cuda(), torch.from_numpy(beta.astype(np.float32)).cuda(),
                    torch.full((len(y),), h, dtype=torch.float32, device="cuda"))
    u2 = torch.empty_like(u1)
    d2 = torch.empty_like(d1)
    g.evaluate(u2, d2)
    g.close()
    assert torch.equal(u1, u2) and torch.equal(d1, d2)


def test_rbf_no_convergence_and_errors():
    import paper_1106_5273_b200 as P
    x, a, s = synth.jittered_lattice(8)
    with pytest.raises(P.FMMError) as e:
        _gpu(x, a, s, x, 0.9 * float(s[0]), tol=1e-14, maxit=1)
    assert e.value.status == P.fmm.FMM_E_NOCONV
    with pytest.raises(P.FMMError):
        _gpu(x, a, s, x, -1.0)
