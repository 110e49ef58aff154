"""CPU (gloo, world_size 2 and 3) test of the multi-GPU row-cluster algorithm
(SURVEY 8(e)): each process takes its ownership masks from the product's host
partition (igb_plan_owned), computes its share of the H² matvec from the
oracle's assembled operator (near blocks, couplings, moments, transfers) --
leaf moments + upward pass of its own clusters, all-gather of the level>=1 up
moments, far field of its own targets, downward pass and near rows of its own
block rows, partial DOF gather -- and all-reduces y.  The result must equal
the oracle's single-process matvec.  This pins the partition and exchange
pattern the device path (DistH2Matrix) implements with NCCL."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _node_decode(node, L, npp, offs):
    p, r = divmod(node, npp)
    l = max(i for i in range(L + 1) if offs[i] <= r)
    s = r - offs[l]
    return p, l, s % (1 << l), s >> l


def _worker(rank, world, port, case, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_1906_00785_b200 as igb
    from oracle import pyoracle as po

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kind, P, L, m = case
    kap = 3.0 if kind != "laplace" else 0.0
    od = po.Discretization(kind, P, 1, L, kappa=kap)
    oh = po.H2Matrix(od, m=m)
    pde = igb.Pde.laplace() if kind == "laplace" else igb.Pde.helmholtz(kap)
    plan = igb.H2Plan(igb.Discretization(igb.make_sphere(), pde, P, 1, L), igb.H2Options(m=m))
    masks = [plan.owned(world, r, od.element_count) for r in range(world)]
    eown, nown = masks[rank]

    dt = np.complex128 if od.is_complex else np.float64
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, od.dof_count).astype(dt)
    if od.is_complex:
        x = x + 1j * rng.uniform(-1, 1, od.dof_count)
    y_ref = oh.apply(x)

    ne, nl, mm = od.element_count, od.local_count, m * m
    npp = sum(4 ** l for l in range(L + 1))
    offs = [sum(4 ** j for j in range(l)) for l in range(L + 1)]
    nn = 6 * npp
    g, sg = od.l2g()
    coef = sg * x[g]
    mom = oh.moments()              # [e][row][l]
    tl, tr = oh.transfer()          # [i][j]
    near = oh.nearfield_pairs()
    blocks = oh.near_blocks()       # [q][la][lb]
    far = oh.farfield_pairs()
    K = oh.couplings()              # [q][nu][mu]
    dec = [_node_decode(t, L, npp, offs) for t in range(nn)]

    def node_id(p, l, sx, sy):
        return p * npp + offs[l] + sx + (1 << l) * sy

    def leaf(e):
        return (e // 4 ** L) * npp + offs[L] + e % 4 ** L

    up = np.zeros((nn, mm), dtype=dt)
    for e in np.nonzero(eown)[0]:
        up[leaf(e)] = mom[e] @ coef[e]

    def upward(t):
        p, l, sx, sy = dec[t]
        Y = np.zeros((m, m), dtype=dt)
        for k in range(4):
            c = node_id(p, l + 1, 2 * sx + (k & 1), 2 * sy + (k >> 1))
            tu, tv = (tr if k & 1 else tl), (tr if k >> 1 else tl)
            Y += tu @ up[c].reshape(m, m, order="F") @ tv.T
        up[t] = Y.reshape(-1, order="F")

    for l in range(L - 1, 0, -1):
        for t in range(nn):
            if dec[t][1] == l and nown[t]:
                upward(t)
    # all-gather of the owned level>=1 up moments (padded, rank-major)
    packs = [[t for t in range(nn) if masks[r][1][t] and dec[t][1] >= 1] for r in range(world)]
    pmax = max(len(p) for p in packs)
    send = np.zeros((pmax, mm), dtype=dt)
    send[:len(packs[rank])] = up[packs[rank]]
    gathered = [torch.zeros(send.shape, dtype=torch.float64 if dt == np.float64 else torch.complex128)
                for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(send))
    for r in range(world):
        up[packs[r]] = gathered[r].numpy()[:len(packs[r])]
    for t in range(nn):
        if dec[t][1] == 0:
            upward(t)
    down = np.zeros((nn, mm), dtype=dt)
    for q, (t, s) in enumerate(far):
        if nown[t]:
            down[t] += K[q] @ up[s]
    for l in range(L):
        for c in range(nn):
            p, lc, sx, sy = dec[c]
            if lc == l + 1 and nown[c]:
                par = node_id(p, l, sx // 2, sy // 2)
                tu, tv = (tr if sx & 1 else tl), (tr if sy & 1 else tl)
                down[c] += (tu.T @ down[par].reshape(m, m, order="F") @ tv).reshape(-1, order="F")
    y = np.zeros(od.dof_count, dtype=dt)
    nrow = np.zeros((ne, nl), dtype=dt)
    for q, (ea, eb) in enumerate(near):
        if eown[ea]:
            nrow[ea] += blocks[q] @ coef[eb]
    for e in np.nonzero(eown)[0]:
        loc = nrow[e] + mom[e].T @ down[leaf(e)]
        np.add.at(y, g[e], sg[e] * loc)
    yt = torch.from_numpy(y)
    dist.all_reduce(yt)
    rel = float(np.linalg.norm(yt.numpy() - y_ref) / np.linalg.norm(y_ref))
    out[rank] = (rel, int(eown.sum()), int(nown.sum()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [("laplace", 1, 2, 4), ("helmholtz", 1, 2, 4)], ids=["laplace", "helmholtz"])
def test_row_partition_gloo(world, case):
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    rels = [out[r][0] for r in range(world)]
    assert max(rels) < 1e-13, rels
    assert sum(out[r][1] for r in range(world)) == 6 * 16  # every block row owned once
