"""Development tool (torchrun, P GPUs): LET size and load balance of the two
domain decompositions on the clustered cloud (fig:partitioning P:121):
equal-count Morton ranges (the ranks pass contiguous ranges of the Morton-sorted
particles, partition = 0) against ORB multisection (partition = 1).  Prints one
JSON line per partition from rank 0."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1106_5273_b200 as P  # noqa: E402
import synth  # noqa: E402


def morton_keys(x, lo=-np.pi, L=2 * np.pi):
    q = np.clip(np.floor((x.astype(np.float64) - lo) * (2 ** 21 / L)), 0, 2 ** 21 - 1).astype(np.uint64)
    key = np.zeros(len(x), dtype=np.uint64)
    for b in range(21):
        for d in range(3):
            key |= ((q[:, d] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + d)
    return key


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"]); rank = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    x, a, s = synth.clustered_cloud(args.n, sigma=0.002)
    order = np.argsort(morton_keys(x), kind="stable")
    for part in (0, 1):
        if part == 0:
            idx = np.array_split(order, world)[rank]
        else:
            idx = synth.scatter_to_ranks(len(x), world, rank)
        obj = [P.fmm_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        f = P.FMM(images=1, nranks=world, rank=rank, device=local, nccl_id=obj[0], partition=part)
        xd, ad, sd = (torch.from_numpy(np.ascontiguousarray(v[idx])).cuda() for v in (x, a, s))
        u = torch.empty((len(idx), 3), device="cuda"); d = torch.empty_like(u)
        ms = []
        for _ in range(args.steps + 1):
            torch.cuda.synchronize(); dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); f.set_particles(xd, ad, sd); f.evaluate(u, d); e1.record(); torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        st = f.stats()
        f.close()
        row = dict(rank=rank, part=part, n_own=st["n"], let_mb=st["let_bytes_recv"] / 1e6, let_cells=st["let_cells"],
                   let_bodies=st["let_leaves"], fallback=st["let_fallback"], ms=float(np.median(ms[1:])),
                   ms_p2p=st["ms_p2p"], ms_m2l=st["ms_m2l"], p2p_pairs=st["p2p_pairs"])
        g = [None] * world
        dist.all_gather_object(g, row)
        if rank == 0:
            N = len(x)
            print(json.dumps({"partition": ["morton_ranges", "orb"][part], "world": world, "N": N,
                              "imbalance_particles": max(r["n_own"] for r in g) / (N / world),
                              "imbalance_pairs": max(r["p2p_pairs"] for r in g) / np.mean([r["p2p_pairs"] for r in g]),
                              "let_mb_per_rank": [round(r["let_mb"], 1) for r in g],
                              "let_mb_total": round(sum(r["let_mb"] for r in g), 1),
                              "fallback": [r["fallback"] for r in g],
                              "ms_step_max": max(r["ms"] for r in g), "ranks": g}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
