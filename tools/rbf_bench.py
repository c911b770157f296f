"""Development tool: time the NEXT-4 RBF reinitialisation at C3 scale (one
B200): old particles = the Taylor-Green 256^3 lattice jittered by +-h/4 (the
field after some steps), sites = the lattice, sigma0 = h, tol 1e-4.  Prints
one JSON line (CUDA events around fmm_rbf_reinit, iterations, per-matvec
Gaussian pairs)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1106_5273_b200 as P
    import synth
    side = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    x, a, s = synth.jittered_lattice(side)
    y, _ya, _ys = synth.taylor_green(side)
    h = 2 * np.pi / side
    f = P.FMM(images=3, order=10, device=0)
    dev = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).cuda()
    xd, ad, sd, yd = dev(x), dev(a), dev(s), dev(y)
    beta = torch.empty((len(y), 3), device="cuda")
    f.rbf_reinit(xd, ad, sd, yd, h, beta, tol=1e-4, maxit=400)      # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    it, res = f.rbf_reinit(xd, ad, sd, yd, h, beta, tol=1e-4, maxit=400)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = f.stats()
    print(json.dumps({"tool": "rbf_bench", "sites": len(y), "particles": len(x), "iterations": it, "resid": res,
                      "ms_total": ms, "ms_per_iteration": ms / max(it, 1), "p2p_pairs_sites_tree": st["p2p_pairs"],
                      "note": "total = union tree + b + sites tree + CG (one Gaussian matvec per iteration)"}))
    f.close()


if __name__ == "__main__":
    main()
