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


def _balanced_worker(rank, world, port, q):
    """Model of the balanced partition (cfg.partition = 1, NEXT-3):
    every rank holds a random subset of a clustered cloud; the Morton curve of
    the global tree is cut into equal-count ranges moved to the nearest leaf
    boundary (the library's k_splits rule), particles are sent to their owners
    (counts exchanged with gloo) and straddling cells are the only partial
    multipoles."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        x, a, s = synth.clustered_cloud(3000)
        mine = synth.scatter_to_ranks(len(x), world, rank)
        f = oracle.OracleFMM(x, a, s, images=1, ncrit=16)
        cells = f.cells()
        _keys, perm = f.keys()                  # perm[g] = input index at global position g
        N = len(x)
        b0, cnt, leaf = cells[:, 4], cells[:, 5], cells[:, 9]
        cb, nch = cells[:, 7], cells[:, 8]

        def split(k):                           # the leaf holding k N / P, nearer boundary
            xk = k * N // world
            c = 0
            while not leaf[c]:
                kids = range(cb[c], cb[c] + nch[c])
                c = next((ch for ch in kids if xk < b0[ch] + cnt[ch]), cb[c] + nch[c] - 1)
            return b0[c] if xk - b0[c] <= b0[c] + cnt[c] - xk else b0[c] + cnt[c]

        off = np.array([0] + [split(k) for k in range(1, world)] + [N])
        ok = bool(np.all(np.diff(off) >= 0))
        # no leaf is cut
        lv = np.nonzero(leaf)[0]
        for k in range(1, world):
            ok &= not bool(np.any((b0[lv] < off[k]) & (off[k] < b0[lv] + cnt[lv])))
        # balance: every range within one leaf of N / P
        ok &= bool(np.all(np.abs(np.diff(off) - N / world) <= 2 * 16 + 1))
        # redistribution counts: my particles' global positions -> owners
        gpos = np.empty(N, dtype=np.int64)
        gpos[perm] = np.arange(N)
        owner = np.searchsorted(off, gpos[mine], side="right") - 1
        send = torch.tensor(np.bincount(owner, minlength=world), dtype=torch.int64)
        recv = torch.zeros(world, dtype=torch.int64)
        dist.all_to_all_single(recv, send)
        ok &= int(recv.sum()) == int(off[rank + 1] - off[rank])
        # straddling cells: non-leaves only, nested (at most one per level per split)
        st = np.zeros(len(cells), dtype=bool)
        for k in range(1, world):
            st |= (b0 < off[k]) & (off[k] < b0 + cnt)
        ok &= not bool(np.any(st & (leaf == 1)))
        lev = cells[:, 0]
        for k in range(1, world):
            sk = (b0 < off[k]) & (off[k] < b0 + cnt)
            ok &= bool(np.all(np.bincount(lev[sk]) <= 1))
        # M is linear: the per-rank partial multipoles of a straddling cell
        # (its particles split by owner) sum to the full one -- modelled on the
        # monopole (sum of alpha) of every straddling cell
        for c in np.nonzero(st)[0]:
            idx = perm[b0[c]:b0[c] + cnt[c]]
            gp = np.arange(b0[c], b0[c] + cnt[c])
            mono = torch.tensor(a[idx[(gp >= off[rank]) & (gp < off[rank + 1])]].astype(np.float64).sum(0))
            dist.all_reduce(mono)
            ok &= bool(np.allclose(mono.numpy(), a[idx].astype(np.float64).sum(0), rtol=1e-12, atol=1e-18))
        q.put((rank, bool(ok), int(st.sum()), [int(v) for v in off]))
    finally:
        dist.destroy_process_group()


def test_three_rank_balanced_partition_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 3
    port = 29660
    procs = [ctx.Process(target=_balanced_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    assert all(r[2] > 0 for r in res), res              # the splits cut through some cells
    assert len({tuple(r[3]) for r in res}) == 1, res    # all ranks agree on the ranges
