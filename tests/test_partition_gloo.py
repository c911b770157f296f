"""CPU (gloo, world_size 2) model of the multi-GPU host logic of a14, checked
against the CPU oracle: Morton-octant ownership, target-side pruning of the
dual traversal, and the exact LET request sets.

Each rank builds the oracle tree of the global particle set, keeps the list
entries whose target it owns, derives the remote sources it must receive
(multipoles for M2L sources, bodies for P2P source leaves) grouped by owner,
and exchanges the request counts with gloo all-to-all.  Checked:
* the ranks' lists partition the global lists (each entry exactly once);
* every request goes to the rank that owns the requested cell, and the counts
  each rank sends equal the counts its peer receives;
* with its own and the requested sources, every owned target particle is
  covered exactly N * 27^k times (the counting kernel of S:313).
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        blocks = [synth.taylor_green_rank(6, world, r) for r in range(world)]
        x = np.concatenate([b[0] for b in blocks])
        a = np.concatenate([b[1] for b in blocks])
        s = np.concatenate([b[2] for b in blocks])
        f = oracle.OracleFMM(x, a, s, images=1, ncrit=8)
        cells = f.cells()
        p2p, m2l = f.p2p_list(), f.m2l_list()
        n = np.array([len(b[0]) for b in blocks])
        off = np.concatenate([[0], np.cumsum(n)])
        b0, cnt = cells[:, 4], cells[:, 5]
        owned = (b0 >= off[rank]) & (b0 + cnt <= off[rank + 1])
        mine_p2p = p2p[owned[p2p[:, 0]]]
        mine_m2l = m2l[owned[m2l[:, 0]]]
        owner = np.searchsorted(off, b0, side="right") - 1
        need_m = np.unique(mine_m2l[:, 1][~owned[mine_m2l[:, 1]]])
        need_p = np.unique(mine_p2p[:, 1][~owned[mine_p2p[:, 1]]])
        ok = True
        # requests go to the owner of the whole requested cell
        for cid in np.concatenate([need_m, need_p]):
            q_ = owner[cid]
            ok &= bool(q_ != rank and b0[cid] >= off[q_] and b0[cid] + cnt[cid] <= off[q_ + 1])
        send = torch.zeros(world, dtype=torch.int64)
        for cid in np.concatenate([need_m, need_p]):
            send[owner[cid]] += 1
        recv = torch.zeros(world, dtype=torch.int64)
        dist.all_to_all_single(recv, send)
        allsend = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allsend, send)
        for p_ in range(world):
            ok &= int(recv[p_]) == int(allsend[p_][rank])
        # coverage of owned targets with local + received sources
        cover = np.zeros(len(x), dtype=np.int64)
        for (t, src, _img) in mine_p2p:
            cover[b0[t]:b0[t] + cnt[t]] += cnt[src]
        for (t, src, _img) in mine_m2l:
            cover[b0[t]:b0[t] + cnt[t]] += cnt[src]
        mine = np.arange(off[rank], off[rank + 1])
        ok &= bool(np.all(cover[mine] == len(x) * 27))
        # the ranks' lists partition the global lists
        sizes = torch.tensor([len(mine_p2p), len(mine_m2l)], dtype=torch.int64)
        dist.all_reduce(sizes)
        ok &= int(sizes[0]) == len(p2p) and int(sizes[1]) == len(m2l)
        q.put((rank, bool(ok), int(len(need_m)), int(len(need_p))))
    finally:
        dist.destroy_process_group()


def test_two_rank_let_requests_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = 29650
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    assert all(r[2] + r[3] > 0 for r in res), res      # a real exchange happens
