"""Multi-GPU parity check (a14), run under torchrun with one process per GPU:

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 \
        --master-port 29511 tests/mgpu_check.py --side 16

Every rank evaluates its octant block of the weak-scaling Taylor-Green lattice
(synth.taylor_green_rank) through the C ABI with nranks = P.  Rank 0 then runs
the single-GPU evaluation of the union of all blocks and checks:
* each rank's P2P and M2L lists == the single-GPU lists restricted to the
  targets that rank owns (bit-exact, global cell ids),
* the near field (P2P) is bit-identical and the full field agrees to 1e-6,
* both match the Taylor-Green closed form to 1e-3.
Prints one JSON line; exit code 1 on any failure.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1106_5273_b200 as P  # noqa: E402
import synth  # noqa: E402


def tg_closed(x, alpha, sigma):
    from test_oracle_kernel import _tg_closed_form
    return _tg_closed_form(x.astype(np.float64), alpha.astype(np.float64), float(sigma))


def run(fmm, x, a, s, parts=3):
    n = len(x)
    xd, ad, sd = (torch.from_numpy(v).cuda() for v in (x, a, s))
    fmm.set_particles(xd, ad, sd)
    u = torch.empty((n, 3), device="cuda")
    st = torch.empty((n, 3), device="cuda")
    fmm.evaluate(u, st, parts)
    return u.cpu().numpy().astype(np.float64), st.cpu().numpy().astype(np.float64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=16)
    ap.add_argument("--mode", choices=["tiled", "refined", "balanced", "balanced_cloud"], default="tiled")
    args = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [P.fmm_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    balanced = args.mode.startswith("balanced")
    if balanced:
        # NEXT-3: every rank passes an arbitrary (seeded random) subset; the
        # library cuts equal-count Morton ranges at leaf boundaries
        full = synth.taylor_green(args.side) if args.mode == "balanced" else synth.clustered_cloud(args.side ** 3)
        gen = lambda side, w, r: tuple(v[synth.scatter_to_ranks(len(full[0]), w, r)] for v in full)
    else:
        gen = synth.taylor_green_tile if args.mode == "tiled" else synth.taylor_green_rank
    tiles = synth.RANK_TILES[world] if args.mode == "tiled" else (1, 1, 1)
    x, a, s = gen(args.side, world, rank)
    fmm = P.FMM(images=3, nranks=world, rank=rank, device=local, nccl_id=obj[0], tiles=tiles,
                partition=1 if balanced else 0)
    un, sn = run(fmm, x, a, s, parts=1)
    u, st = run(fmm, x, a, s)
    p2p, m2l = P.fmm_get_lists(fmm.ctx)
    stats = fmm.stats()
    fmm.close()
    gathered = [None] * world
    dist.all_gather_object(gathered, dict(u=u, s=st, un=un, sn=sn, p2p=p2p, m2l=m2l, n=len(x), stats=stats))
    ok, msg = True, {}
    if rank == 0:
        blocks = [gen(args.side, world, r) for r in range(world)]
        X = np.concatenate([b[0] for b in blocks])
        A = np.concatenate([b[1] for b in blocks])
        S = np.concatenate([b[2] for b in blocks])
        single = P.FMM(images=3, device=local, tiles=tiles)
        Un, Sn = run(single, X, A, S, parts=1)
        U, SS = run(single, X, A, S)
        gp2p, gm2l = P.fmm_get_lists(single.ctx)
        cells = P.fmm_get_cells(single.ctx)
        single.close()
        off = np.cumsum([0] + [g["n"] for g in gathered])
        if balanced:
            # owned ranges partition [0, N), cut at leaf boundaries; a rank's
            # targets are the cells overlapping its range
            ob = [(g["stats"]["own_begin"], g["stats"]["own_count"]) for g in gathered]
            off = np.array([b for b, _ in ob] + [ob[-1][0] + ob[-1][1]])
            leaves = cells[cells[:, 9] == 1]
            ends = set(leaves[:, 4].tolist()) | set((leaves[:, 4] + leaves[:, 5]).tolist())
            msg["own_ranges"] = [int(v) for v in off]
            msg["ranges_ok"] = bool(off[0] == 0 and off[-1] == len(X) and np.all(np.diff(off) >= 0)
                                    and all(int(v) in ends for v in off))
            msg["imbalance"] = float(np.diff(off).max() / (len(X) / world))
            ok &= msg["ranges_ok"]
        for r in range(world):
            if balanced:
                owned = (cells[:, 4] < off[r + 1]) & (cells[:, 4] + cells[:, 5] > off[r])
            else:
                owned = (cells[:, 4] >= off[r]) & (cells[:, 4] + cells[:, 5] <= off[r + 1])
            for name, glst in (("p2p", gp2p), ("m2l", gm2l)):
                want = glst[owned[glst[:, 0]]]
                got = gathered[r][name]
                same = got.shape == want.shape and np.array_equal(got, want)
                ok &= bool(same)
                msg["%s_rank%d_bitexact" % (name, r)] = bool(same)
        du = np.concatenate([g["un"] for g in gathered])
        ds = np.concatenate([g["sn"] for g in gathered])
        msg["near_bitexact"] = bool(np.array_equal(du, Un) and np.array_equal(ds, Sn))
        ok &= msg["near_bitexact"]
        DU = np.concatenate([g["u"] for g in gathered])
        DS = np.concatenate([g["s"] for g in gathered])
        rel = lambda p, q: float(np.linalg.norm(p - q) / np.linalg.norm(q))
        msg["full_vs_single_u"] = rel(DU, U)
        msg["full_vs_single_s"] = rel(DS, SS)
        ok &= msg["full_vs_single_u"] <= 1e-6 and msg["full_vs_single_s"] <= 1e-6
        if args.mode != "balanced_cloud":
            uc, sc = tg_closed(X, A, S[0])
            msg["closed_form_u"] = rel(DU, uc)
            msg["closed_form_s"] = rel(DS, sc)
            ok &= msg["closed_form_u"] <= 1e-3 and msg["closed_form_s"] <= 1e-3
        msg["let"] = [{k: g["stats"][k] for k in ("let_bytes_sent", "let_bytes_recv", "let_cells", "let_leaves",
                                                   "ms_let", "redist_bytes")} for g in gathered]
        msg["ok"] = bool(ok)
        msg["world"] = world
        msg["mode"] = args.mode
        print(json.dumps(msg), flush=True)
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(okt, src=0)
    dist.destroy_process_group()
    sys.exit(0 if okt.item() == 1 else 1)


if __name__ == "__main__":
    main()
