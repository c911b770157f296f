"""CPU (gloo) models of the multi-GPU host logic of a14 and NEXT-3, checked
against the CPU oracle and numpy:

* ORB multisection (partition.cu): every rank holds a random
  subset of a clustered cloud; the distributed nth-element is the same radix
  select the library runs (8-bit digits of (order-preserving coordinate bits,
  rank << 28 | index), one all-reduce of per-group histograms per digit), the
  groups split at floor(N m1 / m) along x, y, z, ...  Checked: every selected
  key is the exact k-th smallest of the group (numpy partition on the
  gathered keys), final counts are the floor splits for a cloud; on a
  lattice (planes of ties) a sparse sliver of the cut plane moves to the
  plane's edge (reading Z28) and the counts stay within 5% of a share.
* LET completeness (let.cu): with Morton-octant ownership, every
  rank builds the oracle tree of ITS OWN particles, walks it against the other
  rank's bounding box with the library's LET-MAC ((1 + theta) max(2 r_B,
  rleaf) + r_B < theta d_B over the first-layer images, rleaf = the other
  rank's largest leaf near this domain) and sends the cell tuples; the
  receiver checks, on the global tree's lists restricted to its own targets,
  that every remote M2L source is in the received LET and every remote P2P
  source leaf came with its bodies (so the remote branch of Alg. 2 is never
  taken), and that received + local sources cover each owned target exactly
  N 27^k times (the counting kernel of S:313).
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _fbits(v):
    u = np.asarray(v, dtype=np.float32).view(np.uint32).astype(np.uint64)
    neg = (u & 0x80000000) != 0
    return np.where(neg, (~u) & 0xffffffff, u | 0x80000000)


def _orb_worker(rank, world, port, q, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, a, s = synth.clustered_cloud(4000) if case == "cloud" else synth.taylor_green(40)
        mine = synth.scatter_to_ranks(len(x), world, rank)
        xm = x[mine]
        ids = (np.uint64(rank) << np.uint64(28)) | np.arange(len(xm), dtype=np.uint64)
        grp = np.zeros(len(xm), dtype=np.int64)
        groups = [(0, world, len(x))]
        ok = True
        sel_log = []
        moved = []
        for depth in range(8):
            if not any(hi - lo > 1 for lo, hi, _ in groups):
                break
            axis = depth % 3
            keys = (_fbits(xm[:, axis]) << np.uint64(32)) | ids
            act = [hi - lo > 1 for lo, hi, _ in groups]
            kth = [cnt * ((hi - lo) // 2) // (hi - lo) if hi - lo > 1 else 0 for lo, hi, cnt in groups]
            prefix = [np.uint64(0)] * len(groups)
            for ps in range(8):
                shift = np.uint64(56 - 8 * ps)
                hist = np.zeros((len(groups), 256), dtype=np.int64)
                for g in range(len(groups)):
                    if not act[g]:
                        continue
                    sel = grp == g
                    k = keys[sel]
                    if ps > 0:
                        up = np.uint64(64 - 8 * ps)
                        k = k[(k >> up) == (prefix[g] >> up)]
                    np.add.at(hist[g], ((k >> shift) & np.uint64(255)).astype(np.int64), 1)
                th = torch.from_numpy(hist)
                dist.all_reduce(th)
                hist = th.numpy()
                for g in range(len(groups)):
                    if not act[g] or groups[g][2] == 0:
                        continue
                    c = np.cumsum(hist[g])
                    d = int(np.searchsorted(c, kth[g], side="right"))
                    kth[g] -= int(c[d - 1]) if d > 0 else 0
                    prefix[g] = prefix[g] | (np.uint64(d) << shift)
            # check: the selected key is the exact k-th smallest of the gathered group keys
            allk = [None] * world
            dist.all_gather_object(allk, (keys, grp))
            nxt = []
            newgrp = grp.copy()
            for g, (lo, hi, cnt) in enumerate(groups):
                if not act[g]:
                    newgrp[grp == g] = len(nxt)
                    nxt.append((lo, hi, cnt))
                    continue
                gk = np.concatenate([k[gg == g] for k, gg in allk])
                m1 = (hi - lo) // 2
                nlow = cnt * m1 // (hi - lo)
                ok &= bool(len(gk) == cnt)
                if cnt:
                    ok &= bool(np.sort(gk)[nlow] == prefix[g])
                    sel_log.append(int(prefix[g] >> np.uint64(32)))
                    # reading Z28: a sparse sliver of a plane of ties moves to the plane's edge
                    cs = prefix[g] >> np.uint64(32)
                    gc = gk >> np.uint64(32)
                    below, plane = int((gc < cs).sum()), int((gc == cs).sum())
                    dlo, dhi = nlow - below, below + plane - nlow
                    sh = min(dlo, dhi)
                    if plane > 1 and 4 * sh < plane and 20 * sh <= cnt // (hi - lo):
                        moved.append(sh)
                        prefix[g] = cs << np.uint64(32) if dlo <= dhi else (cs + np.uint64(1)) << np.uint64(32)
                        nlow = below if dlo <= dhi else below + plane
                    ok &= int((gk < prefix[g]).sum()) == nlow
                low = (grp == g) & (keys < prefix[g])
                newgrp[low] = len(nxt)
                nxt.append((lo, lo + m1, nlow))
                newgrp[(grp == g) & ~(keys < prefix[g])] = len(nxt)
                nxt.append((lo + m1, hi, cnt - nlow))
            grp = newgrp
            groups = nxt
        own = np.array([groups[g][0] for g in range(len(groups))])[grp]
        cnt = torch.tensor(np.bincount(own, minlength=world), dtype=torch.int64)
        dist.all_reduce(cnt)
        N = len(x)
        ok &= int(cnt.sum()) == N
        # exact floor splits without ties; a moved cut costs <= 5% of a share per level
        tol = 1.0 if not moved else 0.05 * 2 * N / world + 1
        ok &= bool(np.all(np.abs(cnt.numpy() - N / world) <= tol))
        q.put((rank, bool(ok), [int(v) for v in cnt], sel_log, moved))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("cloud", 3), ("lattice", 3), ("lattice", 6)])
def test_orb_radix_select_gloo(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29670 + world + (0 if case == "cloud" else 10)
    procs = [ctx.Process(target=_orb_worker, args=(r, world, port, q, case)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    assert len({tuple(r[2]) for r in res}) == 1
    if case == "cloud":
        assert not any(r[4] for r in res)           # continuous coordinates: no ties, exact splits
    print(case, world, res[0][2], res[0][4])


def _cell_geom(cells, lo, L):
    s = L / (2.0 ** cells[:, 0])
    c = lo + (cells[:, 1:4] + 0.5) * s[:, None]
    return c, s


def _dmin(c, box, shifts):
    cc = c[None, :] + shifts
    d = np.maximum(0, np.maximum(box[0] - cc, cc - box[1]))
    return np.sqrt((d * d).sum(1)).min()


def _leaf_reach(cells, lo, L, box, theta, per):
    """k_leaf_reach: the largest leaf radius that can meet a smaller cell of `box`."""
    ctr, side = _cell_geom(cells, lo, L)
    shifts = np.array([[(i % 3 - 1) * per, ((i // 3) % 3 - 1) * per, (i // 9 - 1) * per] for i in range(27)])
    r = 0.8660254037844386 * side
    best = 0.0
    for c in np.nonzero(cells[:, 9])[0]:
        if _dmin(ctr[c], box, shifts) < (1.5 / theta + 0.5) * r[c]:
            best = max(best, r[c])
    return best


def _let_walk(cells, lo, L, box, theta, per, rleaf):
    """The LET-MAC walk of let.cu on an oracle tree: {(level, q): bodies?}."""
    ctr, side = _cell_geom(cells, lo, L)
    shifts = np.array([[(i % 3 - 1) * per, ((i // 3) % 3 - 1) * per, (i // 9 - 1) * per] for i in range(27)])
    out = {}
    stack = [0]
    while stack:
        c = stack.pop()
        dmin = _dmin(ctr[c], box, shifts)
        r = 0.8660254037844386 * side[c]
        acc = ((1 + theta) * max(2 * r, rleaf) + r) / theta * (1 + 1e-9) < dmin
        key = tuple(int(v) for v in cells[c, :4])
        if cells[c, 9]:
            out[key] = not acc
        elif acc:
            out[key] = False
        else:
            out[key] = False
            stack.extend(range(cells[c, 7], cells[c, 7] + cells[c, 8]))
    return out


def _let_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        side, theta, L = 8, 0.5, 2 * np.pi
        lo = np.full(3, -np.pi)
        blocks = [synth.taylor_green_octants(side, world, r) for r in range(world)]
        x, a, s = blocks[rank]
        mine = oracle.OracleFMM(x, a, s, images=1, ncrit=8)
        cells_m = mine.cells()
        box = np.array([x.min(0), x.max(0)], dtype=np.float64)
        boxes = [None] * world
        dist.all_gather_object(boxes, box)
        reach = {r: _leaf_reach(cells_m, lo, L, boxes[r], theta, L) for r in range(world) if r != rank}
        reaches = [None] * world
        dist.all_gather_object(reaches, reach)
        lets = {r: _let_walk(cells_m, lo, L, boxes[r], theta, L, reaches[r][rank]) for r in range(world) if r != rank}
        got = [None] * world
        dist.all_gather_object(got, lets)
        recv = {}
        for r in range(world):
            if r != rank:
                recv.update(got[r][rank])
        # the global tree's lists restricted to my targets
        X = np.concatenate([b[0] for b in blocks])
        A = np.concatenate([b[1] for b in blocks])
        S = np.concatenate([b[2] for b in blocks])
        g = oracle.OracleFMM(X, A, S, images=1, ncrit=8)
        gc = g.cells()
        p2p, m2l = g.p2p_list(), g.m2l_list()
        key = [tuple(int(v) for v in r[:4]) for r in gc]
        mykeys = {tuple(int(v) for v in r[:4]) for r in cells_m if r[0] >= 1}
        owned = np.array([k in mykeys for k in key])
        ok = True
        nremote = 0
        for t, src, _img in m2l[owned[m2l[:, 0]]]:
            if key[src] in mykeys:
                continue
            nremote += 1
            ok &= key[src] in recv
        for t, src, _img in p2p[owned[p2p[:, 0]]]:
            if key[src] in mykeys:
                continue
            nremote += 1
            ok &= bool(recv.get(key[src], False))
        # coverage of my targets with local + received sources
        b0, cnt = gc[:, 4], gc[:, 5]
        cover = np.zeros(len(X), dtype=np.int64)
        for lst in (p2p, m2l):
            for t, src, _img in lst[owned[lst[:, 0]]]:
                cover[b0[t]:b0[t] + cnt[t]] += cnt[src]
        _, perm = g.keys()
        off = np.cumsum([0] + [len(b[0]) for b in blocks])
        gpos = np.empty(len(X), dtype=np.int64)
        gpos[perm] = np.arange(len(X))
        me = gpos[off[rank]:off[rank + 1]]
        ok &= bool(np.all(cover[me] == len(X) * 27))
        q.put((rank, bool(ok), nremote, len(recv)))
    finally:
        dist.destroy_process_group()


def test_two_rank_let_mac_complete_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = 29650
    procs = [ctx.Process(target=_let_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    assert all(r[2] > 0 and r[3] > 0 for r in res), res      # a real exchange happens
