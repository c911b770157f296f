"""Development tool: near field (parts = 1) of TG n^3 saved as .npy, for
bit-identity checks between two library builds (FMM_LIB)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1106_5273_b200 as P  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
x, a, s = synth.taylor_green(n)
f = P.FMM(order=10, images=3, device=0)
xd, ad, sd = (torch.from_numpy(v).cuda() for v in (x, a, s))
f.set_particles(xd, ad, sd)
u = torch.empty((len(x), 3), device='cuda')
d = torch.empty_like(u)
f.evaluate(u, d, 1)
np.save(sys.argv[1], torch.cat([u, d], 1).cpu().numpy())
