"""Host logic of the memory-lean chunked plan, on structure-only contexts (no GPU):
chunks are whole subtrees below the top active level, every row pair and block belongs to exactly
one chunk, the persistent basis weights are exactly those of the direct pairs, and no two slabs
that can be live at the same time overlap."""
import numpy as np
import pytest

from synth import get_config, mesh_for


def _ctx(name):
    from paper_1809_04384_b200 import DH2
    cfg = get_config(name)
    xyz, tri = mesh_for(cfg)
    return DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], device=-1), cfg


def _no_overlap(segs):
    segs = sorted((a, b) for a, b in segs if b > a)
    for (a0, b0), (a1, b1) in zip(segs, segs[1:]):
        assert a1 >= b0, ((a0, b0), (a1, b1))


@pytest.mark.parametrize("name,G", [("P2", 1), ("P2", 3), ("P4", 2), ("C1", 5), ("C2", 7), ("C2", 64)])
def test_lean_plan_invariants(name, G):
    h, cfg = _ctx(name)
    k = cfg["m"] ** 3
    h.set_option("lean_chunks", G)
    s = h.stats()["lean"]
    G = s["chunks"]
    l0 = s["l0"]
    c_begin, c_end = h.export("c_begin", np.int64), h.export("c_end", np.int64)
    lev_ptr = h.export("lev_ptr_row", np.int32)
    L = len(lev_ptr) - 2
    pairs = h.export("row_pairs", np.int64).reshape(-1, 3)
    p_lo = h.export("lean_p_lo", np.int32).reshape(G, L + 1)
    p_hi = h.export("lean_p_hi", np.int32).reshape(G, L + 1)
    blocks = h.export("blocks", np.int64).reshape(-1, 3)
    # chunk extents in triangle positions: the top clusters of chunk g cover [lo_g, hi_g)
    ext = []
    for g in range(G):
        lo = hi = None
        for l in range(L + 1):
            for p in range(p_lo[g, l], p_hi[g, l]):
                t = int(pairs[p, 1])
                lo = c_begin[t] if lo is None else min(lo, c_begin[t])
                hi = c_end[t] if hi is None else max(hi, c_end[t])
        ext.append((lo, hi))
    for g in range(G - 1):
        if ext[g][0] is not None and ext[g + 1][0] is not None:
            assert ext[g][1] <= ext[g + 1][0]

    def chunk_of_cluster(t):
        for g, (lo, hi) in enumerate(ext):
            if lo is not None and lo <= c_begin[t] and c_end[t] <= hi:
                return g
        return -1

    # pairs: per level a partition in chunk order, each pair's cluster inside its chunk
    for l in range(L + 1):
        a, b = lev_ptr[l], lev_ptr[l + 1]
        if b <= a:
            continue
        assert l >= l0
        assert p_lo[0, l] == a and p_hi[G - 1, l] == b
        for g in range(G):
            assert p_lo[g, l] <= p_hi[g, l]
            if g + 1 < G:
                assert p_hi[g, l] == p_lo[g + 1, l]
            for p in range(p_lo[g, l], p_hi[g, l]):
                assert chunk_of_cluster(int(pairs[p, 1])) == g
    # blocks: each exactly once, in the chunk of its row cluster; slot = position in the chunk
    bptr, blk = h.export("lean_blk_ptr", np.int32), h.export("lean_blk", np.int32)
    slot = h.export("lean_slot", np.int32)
    assert sorted(blk.tolist()) == list(range(len(blocks)))
    for g in range(G):
        for i, b in enumerate(blk[bptr[g]:bptr[g + 1]]):
            assert chunk_of_cluster(int(blocks[b, 0])) == g
            assert slot[b] == i
    mirror, lmir = h.export("blk_mirror", np.int32), h.export("lean_mirror", np.int32)
    for b in range(len(blocks)):
        same = mirror[b] >= 0 and chunk_of_cluster(int(blocks[mirror[b], 0])) == chunk_of_cluster(int(blocks[b, 0]))
        assert lmir[b] == (mirror[b] if same else -1)
    # persistent weights: exactly the direct row basis pairs (t,c) and (s,-c) of the blocks
    bpcs = h.export("blk_bpcs", np.int32)
    bp = h.export("basis_pairs", np.int64).reshape(-1, 3)
    bp_id = {(int(t), int(c)): i for i, (_, t, c) in enumerate(bp)}
    keep = h.export("lean_keep", np.int8)
    direct = np.zeros(len(bp), bool)
    for b, (t, _, c) in enumerate(blocks):
        direct[bp_id[(int(t), int(c))]] = True
        direct[bpcs[b]] = True
    assert np.array_equal(keep.astype(bool), direct)
    keepC = h.export("lean_keepC", np.int8)
    assert np.array_equal(keepC.astype(bool), np.array([direct[bp_id[(int(t), int(c))]] for _, t, c in pairs]))
    # layout: persistent slabs disjoint; a chunk's scratch slabs disjoint and beyond the persistent region
    V_off, R_off = h.export("bp_V_off", np.int64), h.export("bp_R_off", np.int64)
    R_rows = h.export("bp_R_rows", np.int32)
    size = lambda i: int(c_end[bp[i, 1]] - c_begin[bp[i, 1]])
    persist = s["VR_persist_bytes"] / 16
    segs_p = []
    for i in np.nonzero(direct)[0]:
        if V_off[i] >= 0 and V_off[i] == R_off[i]:
            segs_p.append((V_off[i], V_off[i] + size(i) * k))
        else:
            segs_p.append((R_off[i], R_off[i] + int(R_rows[i]) * k))
    _no_overlap(segs_p)
    assert max(b for _, b in segs_p) <= persist
    for g in range(G):
        segs = []
        for l in range(l0, L + 1):
            for p in range(p_lo[g, l], p_hi[g, l]):
                i = bp_id[(int(pairs[p, 1]), int(pairs[p, 2]))]
                if direct[i]:
                    continue
                assert R_off[i] >= persist
                if V_off[i] >= 0:
                    assert V_off[i] >= persist
                    segs.append((V_off[i], V_off[i] + size(i) * k))
                if V_off[i] != R_off[i]:
                    segs.append((R_off[i], R_off[i] + int(R_rows[i]) * k))
        _no_overlap(segs)
    # every row pair of the chunks has its Zhat slab, disjoint within the chunk
    Z_off, Z_rows = h.export("Z_off_row", np.int64), h.export("Z_rows_row", np.int32)
    for g in range(G):
        _no_overlap([(Z_off[p], Z_off[p] + int(Z_rows[p]) * k) for l in range(L + 1) for p in range(p_lo[g, l], p_hi[g, l])])
    assert h.stats()["device_bytes"] > 0


def test_lean_plan_memory_estimates():
    """C4 and C5 (BASELINE configs[3..4]) cannot be materialised on one 180 GB B200 (full plan
    1.5 / 1.9 TB) but fit the lean plan with enough chunks (estimate < 180 GB)."""
    for name in ("C4", "C5"):
        h, _ = _ctx(name)
        full = h.stats()["device_bytes"]
        assert full > 1e12
        h.set_option("lean_chunks", 32)
        est = h.stats()["device_bytes"]
        assert est < 160e9, (name, est)


def test_lean_plan_partitioned_c4_fits_110gb_per_gpu():
    """C4 on 8 GPUs: the full plan exceeds a B200 per shard, the lean plan of every
    shard stays below 110 GB with 4 chunks (planner estimates; virtual structure-only context)."""
    from paper_1809_04384_b200 import DH2
    cfg = get_config("C4")
    xyz, tri = mesh_for(cfg)
    h = DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], device=-1, world=8)
    assert min(h.stats()["shard_device_bytes"]) > 183e9
    h.set_option("lean_chunks", 4)
    per = h.stats()["shard_device_bytes"]
    assert len(per) == 8 and max(per) < 110e9, per
