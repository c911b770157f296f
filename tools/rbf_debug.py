import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1106_5273_b200 as P, synth, oracle
n = 12; h = 2*np.pi/n
for name, (x, a, s), y, s0 in [("tg", synth.taylor_green(n), synth.taylor_green(n)[0], 1.1*h),
                               ("jit", synth.jittered_lattice(n), synth.taylor_green(n)[0], h)]:
    f = P.FMM(images=3, order=10, device=0)
    dev = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).cuda()
    beta = torch.empty((len(y), 3), device="cuda")
    try:
        it, res = f.rbf_reinit(dev(x), dev(a), dev(s), dev(y), s0, beta, tol=1e-7, maxit=60)
    except P.FMMError as e:
        print(name, e)
    bg = beta.cpu().numpy().astype(np.float64)
    ref = oracle.rbf_reinit(x, a, s, y, s0, images=1)
    print(name, "beta vs oracle", oracle.rel_l2(bg, ref), "field", oracle.rel_l2(oracle.gauss_field(y, y, bg, np.full(len(y), s0)), oracle.gauss_field(y, x, a, s)))
    f.close()
