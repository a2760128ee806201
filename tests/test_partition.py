"""Host logic of the subtree partition (include/dh2.h dh2_dist) without a GPU:
structure-only contexts (device = DH2_DEVICE_NONE) expose each shard's ownership and exchange
lists.  Checked against an independent recomputation from the exported blocks and the cluster
tree, and across processes (torch.distributed gloo, world size 2): what one rank sends is
exactly what its peer expects to receive."""
import os

import numpy as np
import pytest

from synth import get_config, mesh_for

CONFIGS = ["P1", "P2", "P3", "P4", "C1"]


def _ctx(name, world, rank=0, uid=None):
    from paper_1809_04384_b200.dh2 import DH2
    cfg = get_config(name)
    xyz, tri = mesh_for(cfg)
    return DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], device=-1,
               world=world, rank=rank, nccl_uid=uid)


def _expected(h, world):
    """Recompute owners, own blocks and exchange items from exported structure arrays."""
    lev = h.export("c_level", np.int64)
    beg, end = h.export("c_begin", np.int64), h.export("c_end", np.int64)
    cut = world.bit_length() - 1
    tops = [t for t in range(len(lev)) if lev[t] == cut]
    assert len(tops) == world
    # owner by position range containment (clusters are contiguous ranges of the permutation)
    owner = np.full(len(lev), -1)
    for r, t0 in enumerate(tops):
        inside = (lev >= cut) & (beg >= beg[t0]) & (end <= end[t0])
        owner[inside] = r
    blocks = h.export("blocks", np.int64).reshape(-1, 3)
    basis = h.export("basis_pairs", np.int64).reshape(-1, 3)
    bp_id = {(int(t), int(c)): i for i, (l, t, c) in enumerate(basis)}
    col = h.export("col_pairs", np.int64).reshape(-1, 3)
    col_id = {(int(t), int(c)): i for i, (l, t, c) in enumerate(col)}
    k = h.k
    return owner, blocks, bp_id, col_id, beg, end, k, tops


@pytest.mark.parametrize("name", CONFIGS)
@pytest.mark.parametrize("world", [2, 4])
def test_virtual_partition(name, world):
    h = _ctx(name, world)
    owner, blocks, bp_id, col_id, beg, end, k, tops = _expected(h, world)
    ex_owner = h.export("owner", np.int32, shard=0)
    assert np.array_equal(ex_owner, owner)
    lev = h.export("c_level", np.int64)
    nb = len(blocks)
    covered = np.zeros(nb, dtype=int)
    send = {}
    recv = {}
    for r in range(world):
        b_lo, b_hi, p_lo, p_hi = h.export("own_range", np.int32, shard=r)
        assert (p_lo, p_hi) == (beg[tops[r]], end[tops[r]])
        covered[b_lo:b_hi] += 1
        assert np.all(owner[blocks[b_lo:b_hi, 0]] == r)
        lists = h.exchange_lists(shard=r)
        for kind in ("xR", "xC"):
            for peer in range(world):
                send[(kind, r, peer)] = lists[kind + "_send"][peer]
                recv[(kind, r, peer)] = lists[kind + "_recv"][peer]
    assert np.all(covered == 1)  # the shards partition the admissible blocks
    # consistency: a's send list to b is b's receive list from a
    for kind in ("xR", "xC"):
        for a in range(world):
            assert send[(kind, a, a)] == [] and recv[(kind, a, a)] == []
            for b in range(world):
                assert send[(kind, a, b)] == recv[(kind, b, a)]
    # independent recomputation of the items: blocks (t,s,c) with owner(t) != owner(s)
    bp_neg = h.export("bp_neg", np.int32)
    basis = h.export("basis_pairs", np.int64).reshape(-1, 3)
    dirs, dir_off = h.export("dirs", np.float64).reshape(-1, 3), h.export("dir_off", np.int64)
    for i in range(0, len(basis), 7):  # (t,-c) really is the antipodal direction
        l, t, c = (int(v) for v in basis[i])
        l2, t2, c2 = (int(v) for v in basis[bp_neg[i]])
        assert (l2, t2) == (l, t) and np.array_equal(dirs[dir_off[l] + c2], -dirs[dir_off[l] + c])
    is_leaf = lambda t: not np.any((lev == lev[t] + 1) & (beg >= beg[t]) & (end <= end[t]))  # noqa: E731
    for a in range(world):
        for b in range(world):
            if a == b:
                continue
            sel = blocks[(owner[blocks[:, 1]] == a) & (owner[blocks[:, 0]] == b)]
            xc = sorted({col_id[(int(s), int(c))] for t, s, c in sel})
            # R of the row basis pair (s,-c): the column side is its conjugate (adjoint symmetry)
            xr = sorted({int(bp_neg[bp_id[(int(s), int(c))]]) for t, s, c in sel if not is_leaf(s) or end[s] - beg[s] > k})
            assert send[("xC", a, b)] == xc
            assert send[("xR", a, b)] == xr


def test_partition_requires_cut_above_active_levels():
    from paper_1809_04384_b200.dh2 import DH2Error, DH2_ENOTIMPL, DH2_EINVAL
    with pytest.raises(DH2Error) as e:
        _ctx("C1", 64)  # cut level 6 lies below the only active level (5)
    assert e.value.code == DH2_ENOTIMPL
    with pytest.raises(DH2Error) as e:
        _ctx("C1", 3)
    assert e.value.code == DH2_EINVAL


def _gloo_worker(rank, world, port, name, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = _ctx(name, world, rank=rank, uid=b"\0" * 128)  # one shard per process (NCCL layout)
        mine = h.exchange_lists()
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        ok = all(allv[a]["xR_send"][b] == allv[b]["xR_recv"][a] and allv[a]["xC_send"][b] == allv[b]["xC_recv"][a]
                 for a in range(world) for b in range(world))
        rng = h.export("own_range", np.int32)
        ranges = [None] * world
        dist.all_gather_object(ranges, rng.tolist())
        q.put((rank, ok, ranges))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["P2", "C1"])
def test_gloo_two_ranks(name):
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, ranges in res:
        assert ok
        b = sorted((r[0], r[1]) for r in ranges)
        assert b[0][0] == 0 and b[0][1] == b[1][0]  # the two ranks' blocks tile [0, nblocks)
