"""Development tool: time the near-field kernel variants (FMM_P2P_VARIANT) and
the M2L/P2P phases on the C3 workload (or --side N); checks every variant
reproduces variant 0's near field.  Not part of the product path."""
import argparse
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--variants", default="0")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--full", action="store_true", help="also time full evaluate phases")
    ap.add_argument("--m2l-path", type=int, default=0)
    ap.add_argument("--save", default="", help="save variant 0's (u, d) here (.npy) for an A/B of two FMM_LIB builds")
    args = ap.parse_args()
    import torch
    import paper_1106_5273_b200 as P
    import synth
    x, a, s = synth.taylor_green(args.side)
    f = P.FMM(order=10, images=3, theta=(1, 2), ncrit=64, m2l_path=args.m2l_path)
    xt, at, st = (torch.from_numpy(v).cuda() for v in (x, a, s))
    f.set_particles(xt, at, st)
    n = len(x)
    u = torch.empty((n, 3), device="cuda")
    d = torch.empty((n, 3), device="cuda")
    ref = None
    for v in [int(t) for t in args.variants.split(",")]:
        os.environ["FMM_P2P_VARIANT"] = str(v)
        f.evaluate(u, d, 1)
        torch.cuda.synchronize()
        ms = []
        for _ in range(args.reps):
            f.evaluate(u, d, 1)
            torch.cuda.synchronize()
            ms.append(f.stats()["ms_p2p"])
        out = torch.cat([u, d], 1).cpu().numpy()
        if ref is None:
            ref = out
            if args.save:
                np.save(args.save, out)
        diff = float(np.abs(out - ref).max() / np.abs(ref).max())
        print("variant %d  p2p %.2f ms (min %.2f)  max rel diff vs v0 %.2e" % (v, statistics.median(ms), min(ms), diff),
              flush=True)
    os.environ["FMM_P2P_VARIANT"] = "0"
    if args.full:
        for _ in range(2):
            f.evaluate(u, d, 3)
        torch.cuda.synchronize()
        st = f.stats()
        print({k: round(v, 2) for k, v in st.items() if k.startswith("ms_")})
        print("m2l_list %d  m2l_tc_list %d" % (st["m2l_list"], st["m2l_tc_list"]))
    f.close()


if __name__ == "__main__":
    main()
