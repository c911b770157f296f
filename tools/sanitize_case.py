"""Small cases for compute-sanitizer (one tool per gpurun call): C1 (Taylor-Green
16^3, k = 3, p = 10: every 8a row incl. the periodic far field) and TG 32^3 with
8 particles per leaf on the tensor-core M2L path (tcgen05/TMEM/mbarrier/
cp.async.bulk code of m2l_tc.cu), plus the NEXT rows (step, targets, RBF) on
tiny inputs.  Exits non-zero on any library error."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1106_5273_b200 as P  # noqa: E402
import synth  # noqa: E402


def run(x, a, s, **cfg):
    f = P.FMM(**cfg)
    xd, ad, sd = (torch.from_numpy(v).cuda() for v in (x, a, s))
    f.set_particles(xd, ad, sd)
    u = torch.empty((len(x), 3), device="cuda")
    d = torch.empty((len(x), 3), device="cuda")
    f.evaluate(u, d)
    st = f.stats()
    f.close()
    torch.cuda.synchronize()
    return st


st = run(*synth.taylor_green(16), images=3)
print("C1 ok", st["p2p_list"], st["m2l_list"])
st = run(*synth.taylor_green(32), images=3, ncrit=8)
print("TG32 tensor-core M2L ok", st["m2l_tc_list"], st["m2l_list"])
assert st["m2l_tc_list"] > 0
x, a, s = synth.jittered_lattice(8)
f = P.FMM(images=1, ncrit=16)
xd, ad, sd = (torch.from_numpy(v).cuda() for v in (x, a, s))
f.step(xd, ad, sd, 0.01, 0.001)
y = torch.from_numpy(synth.lattice(4)[0].astype(np.float32)).cuda()
uy = torch.empty((len(y), 3), device="cuda")
f.evaluate_targets(xd, ad, sd, y, uy)
beta = torch.empty((len(y), 3), device="cuda")
try:
    f.rbf_reinit(xd, ad, sd, y, float(s[0]) * 2, beta, tol=1e-3, maxit=50)
except P.FMMError as e:
    if e.status != P.fmm.FMM_E_NOCONV:
        raise
f.close()
torch.cuda.synchronize()
print("NEXT rows ok")
