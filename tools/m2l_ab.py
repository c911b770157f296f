"""Development tool: time the tensor-core M2L (ms_m2l_tc) at C3 for the library
in FMM_LIB (default build if unset) and save the far field for an A/B diff."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1106_5273_b200 as P, synth
x, a, s = synth.taylor_green(256)
f = P.FMM(images=3)
xd, ad, sd = (torch.from_numpy(v).cuda() for v in (x, a, s))
f.set_particles(xd, ad, sd)
u = torch.empty((len(x), 3), device="cuda"); d = torch.empty_like(u)
ms = []
for i in range(6):
    f.evaluate(u, d, 2)
    torch.cuda.synchronize()
    if i: ms.append(f.stats()["ms_m2l_tc"])
print("m2l_tc %.2f ms (min %.2f)" % (statistics.median(ms), min(ms)), "m2l", f.stats()["ms_m2l"])
np.save(sys.argv[1], torch.cat([u, d], 1).cpu().numpy())
