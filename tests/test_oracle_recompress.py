"""Pins of the oracle recompression (§3): the paper's identities, the dense §3.1
algorithm as brute force, closed forms of the rank rule and the error identities."""
import numpy as np
import pytest

from oracle import ops
from oracle.dense import DenseCompression
from oracle.recompress import select_rank, tail_sums

from conftest import oracle_run

CFGS = ["P0", "P1", "P3", "P8", "P9"]


def test_rank_rule_examples():
    # SPEC kernels examples (cluster-relative Frobenius / spectral) and eps = 0
    s = np.array([1.0, 1e-3, 1e-9])
    assert select_rank(s, 1e-2, "FROB_CLUSTERREL") == 1
    assert select_rank(np.array([1.0, 1.0, 1.0]), 0.5, "SPEC_BLOCKREL") == 3
    assert select_rank(np.array([3.0, 1.0, 0.0]), 0.0, "FROB_BLOCKREL") == 2
    # block-relative Frobenius: smallest k with tail <= eps^2
    s = np.array([1.0, 0.1, 0.01, 0.001])
    assert select_rank(s, 0.0101, "FROB_BLOCKREL") == 2
    assert select_rank(s, 0.00999, "FROB_BLOCKREL") == 3
    assert np.allclose(tail_sums(s)[:4], [1.010101, 0.010101, 0.000101, 0.000001])
    assert select_rank(np.zeros(0), 1e-4, "FROB_BLOCKREL") == 0


@pytest.mark.parametrize("name", CFGS)
def test_basis_weights_gram(name):
    """R_tc^* R_tc = V_tc^* V_tc with V_tc expanded by Eq. 11 (Eq. 18: V = P R, P isometric)."""
    rc = oracle_run(name)
    st = rc.st
    cache = {}
    for l in st.active_levels:
        for (t, c) in st.basis_pairs[l][:: max(1, len(st.basis_pairs[l]) // 40)]:
            V = ops.expand_V(rc, t, c, cache)
            R = rc.R[(t, c)]
            G = V.conj().T @ V
            assert np.abs(R.conj().T @ R - G).max() <= 1e-12 * np.abs(G).max()


@pytest.mark.parametrize("name", CFGS)
@pytest.mark.parametrize("side", ["row", "col"])
def test_fast_equals_dense_section31(name, side):
    """§3.2 reproduces §3.1 "without changing the result": for every pair,
    sigma(V Zhat^*) = sigma(Ghat_tc) of the dense algorithm, identical ranks and projectors."""
    rc = oracle_run(name)
    res = rc.row if side == "row" else rc.col
    dc = DenseCompression(rc, side).run()
    qcache = {}
    for key, s_fast in res.sigma.items():
        s_dense = dc.sigma[key]
        n = min(len(s_fast), len(s_dense))
        smax = max(s_fast.max() if len(s_fast) else 0.0, s_dense.max() if len(s_dense) else 0.0)
        assert np.all(s_fast[n:] <= 1e-12 * max(smax, 1e-300)) and np.all(s_dense[n:] <= 1e-12 * max(smax, 1e-300))
        assert np.abs(s_fast[:n] - s_dense[:n]).max(initial=0.0) <= 1e-11 * max(smax, 1e-300)
        assert res.rank[key] == dc.rank[key]
        Q = ops.expand_Q(rc, res, key[0], key[1], qcache)
        Qd = dc.Q[key]
        assert np.abs(Q @ Q.conj().T - Qd @ Qd.conj().T).max(initial=0.0) <= 1e-10


@pytest.mark.parametrize("name", CFGS)
def test_total_weights_singular_values(name):
    """sigma(V_tc Zhat_tc^*) = sigma(G_tc) with G_tc assembled densely over row+(t,c) (Eq. 17)."""
    rc = oracle_run(name)
    st = rc.st
    dc = DenseCompression(rc, "row")
    pmap = st.parent_map(st.row_pairs)
    vcache = {}
    for l in st.active_levels:
        for (t, c) in st.row_pairs[l][:: max(1, len(st.row_pairs[l]) // 25)]:
            G = dc.G_tc(t, c, pmap)
            V = ops.expand_V(rc, t, c, vcache)
            M = V @ rc.row.Zhat[(t, c)].conj().T
            sG = np.linalg.svd(G, compute_uv=False)
            sM = np.linalg.svd(M, compute_uv=False)
            n = min(len(sG), len(sM))
            assert np.abs(sG[:n] - sM[:n]).max() <= 1e-10 * sG[0]
            assert np.all(sG[n:] <= 1e-10 * sG[0]) and np.all(sM[n:] <= 1e-10 * sG[0])
            ZZ = rc.row.Zhat[(t, c)].conj().T @ rc.row.Zhat[(t, c)]
            assert ZZ.shape == (st.k, st.k)


@pytest.mark.parametrize("name", CFGS)
def test_new_basis_orthogonal_and_nested(name):
    rc = oracle_run(name)
    st, ct = rc.st, rc.st.ct
    for res in (rc.row, rc.col):
        cache = {}
        for (t, c), kk in res.rank.items():
            Q = ops.expand_Q(rc, res, t, c, cache)
            assert Q.shape[1] == kk
            assert np.abs(Q.conj().T @ Q - np.eye(kk)).max(initial=0.0) <= 1e-12
            if not ct.is_leaf(t):
                l = int(ct.level[t])
                c2 = st.sd(l, c)
                # Q_tc|_{t'} = Q_{t'c'} F_{t'c} (exact by construction)
                for i, ch in enumerate(ct.children[t]):
                    ch = int(ch)
                    off = ct.begin[ch] - ct.begin[t]
                    sub = Q[off:off + ct.size(ch)]
                    assert np.abs(sub - cache[(ch, c2)] @ res.F[(t, c)][i]).max(initial=0.0) <= 1e-14
            # C_tc = Q_tc^* V_tc (Eq. 19) with expanded matrices
            V = ops.expand_V(rc, t, c)
            assert np.abs(res.C[(t, c)] - Q.conj().T @ V).max(initial=0.0) <= 1e-12 * max(1.0, np.abs(V).max())


@pytest.mark.parametrize("name", CFGS)
def test_error_identities(name):
    """(i) sum_b w_b^2 ||G_b - Q Q^* G_b||^2 = E_row (Pythagoras, Eq. 14);
    (ii) sum_b w_b^2 ||G_b - G~_b||^2 <= E_row + E_col;
    (iii) ||G_b - G~_b||^2 = ||G_b||^2 - ||S~_b||^2 (orthogonal projection)."""
    rc = oracle_run(name)
    st = rc.st
    vc, qr_, qc = {}, {}, {}
    e_i, e_ii = 0.0, 0.0
    for b in range(len(st.blocks)):
        t, s, c = (int(v) for v in st.blocks[b])
        G = ops.dense_block_orig(rc, b, vc)
        Q = ops.expand_Q(rc, rc.row, t, c, qr_)
        Gt = ops.dense_block_recomp(rc, b, qr_, qc)
        w2 = rc.omega[b] ** 2
        e_i += w2 * np.linalg.norm(G - Q @ (Q.conj().T @ G)) ** 2
        d2 = np.linalg.norm(G - Gt) ** 2
        e_ii += w2 * d2
        g2 = np.linalg.norm(G) ** 2
        assert abs(d2 - (g2 - np.linalg.norm(rc.St[b]) ** 2)) <= 1e-12 * g2
        assert abs(np.sqrt(g2) - rc.normG[b]) <= 1e-12 * np.sqrt(g2)
    E_row, E_col = rc.discarded(rc.row), rc.discarded(rc.col)
    assert abs(e_i - E_row) <= 1e-9 * E_row + 1e-15 * len(st.blocks)
    assert e_ii <= (E_row + E_col) * (1 + 1e-9)


def test_eps_to_zero_reproduces_far_field():
    rc = oracle_run("P1", eps=1e-14)
    st = rc.st
    vc, qr_, qc = {}, {}, {}
    num = den = 0.0
    for b in range(len(st.blocks)):
        G = ops.dense_block_orig(rc, b, vc)
        num += np.linalg.norm(G - ops.dense_block_recomp(rc, b, qr_, qc)) ** 2
        den += np.linalg.norm(G) ** 2
    assert np.sqrt(num / den) <= 1e-12


def test_monotone_in_eps():
    """Decreasing eps never decreases any rank (SPEC recompression invariant)."""
    r3 = oracle_run("P1", eps=1e-3)
    r4 = oracle_run("P1", eps=1e-4)
    r5 = oracle_run("P1", eps=1e-5)
    for key in r4.row.rank:
        assert r3.row.rank[key] <= r4.row.rank[key] <= r5.row.rank[key]


def test_kappa0_real_h2():
    """kappa = 0: all plane waves are 1, V and S real -> real recompressed factors (H^2 case)."""
    rc = oracle_run("P0")
    for key, Q in rc.row.Q.items():
        V = rc.V(*key)
        assert np.all(V.imag == 0)
    for b in range(0, len(rc.st.blocks), 17):
        assert np.all(rc.S(b).imag == 0)


@pytest.mark.parametrize("mode", ["FROB_CLUSTERREL", "SPEC_BLOCKREL"])
def test_other_modes_match_dense(mode):
    rc = oracle_run("P1", mode=mode)
    dc = DenseCompression(rc, "row").run()
    for key in rc.row.rank:
        assert rc.row.rank[key] == dc.rank[key]


@pytest.mark.parametrize("name", ["P1", "P3"])
def test_matvec_against_dense_blocks(name):
    from synth import seeded_vector
    rc = oracle_run(name)
    x = seeded_vector(rc.st.n, 1)
    for which in ("orig", "recomp"):
        y = ops.matvec(rc, x, which)
        yd = ops.matvec_dense_blocks(rc, x, which)
        assert np.linalg.norm(y - yd) <= 1e-12 * np.linalg.norm(yd)
    assert np.all(ops.matvec(rc, np.zeros(rc.st.n)) == 0)
    x2 = seeded_vector(rc.st.n, 2)
    a = 0.3 - 1.2j
    lhs = ops.matvec(rc, a * x + x2)
    rhs = a * ops.matvec(rc, x) + ops.matvec(rc, x2)
    assert np.linalg.norm(lhs - rhs) <= 1e-13 * np.linalg.norm(rhs)


def test_storage_hand_count():
    rc = oracle_run("C1")
    st, ct, k = rc.st, rc.st.ct, rc.k
    rep = ops.storage(rc, "orig")
    # C1: every active pair is on the leaf level (16 triangles): V is 16 x 27 per basis pair
    nrow = sum(len(p) for p in st.row_pairs)
    ncol = sum(len(p) for p in st.col_pairs)
    assert rep["row_basis_bytes"] == nrow * 16 * k * 16
    assert rep["col_basis_bytes"] == ncol * 16 * k * 16
    assert rep["coupling_bytes"] == len(st.blocks) * k * k * 16
    assert rep["kb_per_dof_matrix"] == (rep["row_basis_bytes"] + rep["col_basis_bytes"] + rep["coupling_bytes"]
                                        + rep["nearfield_bytes"]) / st.n / 1024.0
    rr = ops.storage(rc, "recomp")
    assert rr["kb_per_dof_matrix"] < rep["kb_per_dof_matrix"]


@pytest.mark.parametrize("name", ["C1", "P1", "P2"])
def test_storage_recomp_counts_stored_coefficients(name):
    """storage('recomp') (16 B per complex coefficient, 1 KB = 1024 B) equals
    the number of coefficients the recompressed matrix actually holds: the leaf matrices Q_tc, the
    transfer blocks F_{t'c} and the couplings S~_b, counted from the arrays themselves (their
    shapes), not from the rank formula.  Ranks: the column counts of those arrays."""
    rc = oracle_run(name)
    st, ct = rc.st, rc.st.ct
    rep = ops.storage(rc, "recomp")
    side_bytes, cols = [], []
    for res, pairs in ((rc.row, st.row_pairs), (rc.col, st.col_pairs)):
        tot = 0
        for l in range(ct.depth + 1):
            for (t, c) in pairs[l]:
                if ct.is_leaf(t):
                    Q = res.Q[(t, c)]
                    assert Q.shape[0] == ct.size(t)
                    tot += Q.size
                    cols.append(Q.shape[1])
                else:
                    F = res.F[(t, c)]
                    assert len(F) == 2 and F[0].shape[1] == F[1].shape[1]
                    tot += F[0].size + F[1].size
                    cols.append(F[0].shape[1])
        side_bytes.append(16.0 * tot)
    coup = 16.0 * sum(rc.St[b].size for b in range(len(st.blocks)))
    near = 16.0 * sum(ct.size(int(t)) * ct.size(int(s)) for t, s in st.near)
    assert rep["row_basis_bytes"] == side_bytes[0]
    assert rep["col_basis_bytes"] == side_bytes[1]
    assert rep["coupling_bytes"] == coup
    assert rep["nearfield_bytes"] == near
    assert rep["kb_per_dof_matrix"] == pytest.approx((sum(side_bytes) + coup + near) / st.n / 1024.0, rel=1e-15)
    assert rep["max_rank"] == max(cols)
    assert rep["mean_rank"] == pytest.approx(np.mean(cols), rel=1e-14)
    assert 0 < rep["kb_per_dof_matrix"] < ops.storage(rc, "orig")["kb_per_dof_matrix"]
