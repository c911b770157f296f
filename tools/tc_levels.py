"""Development tool: per-level M2L list composition of C3 (lattice) -- which levels the
tensor path takes and how many entries stay on the register kernel."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1106_5273_b200 as P, synth
side = int(sys.argv[1]) if len(sys.argv) > 1 else 64
x, a, s = synth.taylor_green(side)
f = P.FMM(images=3)
xd, ad, sd = (torch.from_numpy(v).cuda() for v in (x, a, s))
f.set_particles(xd, ad, sd)
u = torch.empty((len(x), 3), device="cuda"); d = torch.empty_like(u)
f.evaluate(u, d)
st = f.stats()
print({k: st[k] for k in ("m2l_list", "m2l_tc_list", "m2l_reg_list")})
cells = P.fmm_get_cells(f.ctx)
p2p, m2l = P.fmm_get_lists(f.ctx)
lv = cells[m2l[:, 0], 0]
for l in np.unique(lv):
    print("level", l, "cells", int((cells[:, 0] == l).sum()), "entries", int((lv == l).sum()))
