"""Oracle operations on DH^2 matrices (TEST INFRASTRUCTURE ONLY).

* dense expansion of nested bases (Eq. 11): V_tc|_{t'} = V_{t'c'} E_{t'c};
  recompressed Q_tc|_{t'} = Q_{t'c'} F_{t'c}
* dense far-field blocks G_b = V_tc S_b V_sc^* (Eq. vsw) and their
  recompressed versions Q_tc S~_b Q'_sc^*
* far-field matvec y = sum_b G_b x|_s (forward / coupling / backward transformations)
* storage accounting in KB per DoF, 1 KB = 1024 B, 16 B per complex entry
"""
import numpy as np


# ---------------------------------------------------------------- expansion
def expand_V(rc, t, c, cache=None):
    """Dense V_tc (#t x k) of the interpolation basis via Eq. 11."""
    st, ct = rc.st, rc.st.ct
    if cache is not None and (t, c) in cache:
        return cache[(t, c)]
    if ct.is_leaf(t):
        out = rc.V(t, c)
    else:
        l = int(ct.level[t])
        c2 = st.sd(l, c)
        out = np.vstack([expand_V(rc, int(ch), c2, cache) @ rc.E(int(ch), c) for ch in ct.children[t]])
    if cache is not None:
        cache[(t, c)] = out
    return out


def expand_Q(rc, res, t, c, cache=None):
    """Dense new basis Q_tc (#t x k_tc) via Q_tc|_{t'} = Q_{t'c'} F_{t'c}."""
    st, ct = rc.st, rc.st.ct
    if cache is not None and (t, c) in cache:
        return cache[(t, c)]
    if ct.is_leaf(t):
        out = res.Q[(t, c)]
    else:
        l = int(ct.level[t])
        c2 = st.sd(l, c)
        F = res.F[(t, c)]
        out = np.vstack([expand_Q(rc, res, int(ch), c2, cache) @ F[i] for i, ch in enumerate(ct.children[t])])
    if cache is not None:
        cache[(t, c)] = out
    return out


def dense_block_orig(rc, b, cache=None):
    t, s, c = (int(v) for v in rc.st.blocks[b])
    return expand_V(rc, t, c, cache) @ rc.S(b) @ expand_V(rc, s, c, cache).conj().T


def dense_block_recomp(rc, b, qcache_row=None, qcache_col=None):
    t, s, c = (int(v) for v in rc.st.blocks[b])
    return expand_Q(rc, rc.row, t, c, qcache_row) @ rc.St[b] @ expand_Q(rc, rc.col, s, c, qcache_col).conj().T


# ---------------------------------------------------------------- matvec
def _forward(rc, basis_leaf, transfer, pairs, xp):
    """xhat_sc = B_sc^* x|_s, computed leaf-up through the transfers."""
    st, ct = rc.st, rc.st.ct
    xh = {}
    for l in range(ct.depth, -1, -1):
        for (s, c) in pairs[l]:
            if ct.is_leaf(s):
                B = basis_leaf(s, c)
                xh[(s, c)] = B.conj().T @ xp[ct.begin[s]:ct.end[s]]
            else:
                c2 = st.sd(l, c)
                acc = None
                for i, ch in enumerate(ct.children[s]):
                    v = transfer(s, int(ch), i, c).conj().T @ xh[(int(ch), c2)]
                    acc = v if acc is None else acc + v
                xh[(s, c)] = acc
    return xh


def _backward(rc, basis_leaf, transfer, pairs, yh, n):
    st, ct = rc.st, rc.st.ct
    yp = np.zeros(n, dtype=np.complex128)
    yh = dict(yh)
    for l in range(ct.depth + 1):
        for (t, c) in pairs[l]:
            v = yh.get((t, c))
            if v is None:
                continue
            if ct.is_leaf(t):
                yp[ct.begin[t]:ct.end[t]] += basis_leaf(t, c) @ v
            else:
                c2 = st.sd(l, c)
                for i, ch in enumerate(ct.children[t]):
                    key = (int(ch), c2)
                    w = transfer(t, int(ch), i, c) @ v
                    yh[key] = w if key not in yh else yh[key] + w
    return yp


def matvec(rc, x, which="recomp"):
    """Far-field product y = G_far x (original triangle order in and out)."""
    st, ct = rc.st, rc.st.ct
    x = np.asarray(x, dtype=np.complex128)
    xp = x[ct.perm]
    if which == "orig":
        leaf = lambda t, c: rc.V(t, c)
        tr = lambda tp, ch, i, c: rc.E(ch, c)
        xh = _forward(rc, leaf, tr, st.col_pairs, xp)
        yh = {}
        for b in range(len(st.blocks)):
            t, s, c = (int(v) for v in st.blocks[b])
            v = rc.S(b) @ xh[(s, c)]
            yh[(t, c)] = v if (t, c) not in yh else yh[(t, c)] + v
        yp = _backward(rc, leaf, tr, st.row_pairs, yh, st.n)
    else:
        xh = _forward(rc, lambda s, c: rc.col.Q[(s, c)], lambda sp, ch, i, c: rc.col.F[(sp, c)][i], st.col_pairs, xp)
        yh = {}
        for b in range(len(st.blocks)):
            t, s, c = (int(v) for v in st.blocks[b])
            v = rc.St[b] @ xh[(s, c)]
            yh[(t, c)] = v if (t, c) not in yh else yh[(t, c)] + v
        yp = _backward(rc, lambda t, c: rc.row.Q[(t, c)], lambda tp, ch, i, c: rc.row.F[(tp, c)][i],
                       st.row_pairs, yh, st.n)
    y = np.empty_like(yp)
    y[ct.perm] = yp
    return y


def matvec_dense_blocks(rc, x, which="recomp"):
    """Brute force: y = sum_b dense(G_b) x|_s."""
    st, ct = rc.st, rc.st.ct
    xp = np.asarray(x, dtype=np.complex128)[ct.perm]
    yp = np.zeros(st.n, dtype=np.complex128)
    vc, qr_, qc = {}, {}, {}
    for b in range(len(st.blocks)):
        t, s, c = (int(v) for v in st.blocks[b])
        G = dense_block_orig(rc, b, vc) if which == "orig" else dense_block_recomp(rc, b, qr_, qc)
        yp[ct.begin[t]:ct.end[t]] += G @ xp[ct.begin[s]:ct.end[s]]
    y = np.empty_like(yp)
    y[ct.perm] = yp
    return y


# ---------------------------------------------------------------- storage
def storage(rc, which="recomp"):
    """Coefficient counts x 16 B.  ORIG counts V leaves and the E of
    every non-leaf basis pair (k x k per child) for the row and the column basis and k x k
    per coupling; RECOMP counts Q leaves, F and S~ with the adaptive ranks.  The
    nearfield is counted from the block sizes (it is not assembled)."""
    st, ct, k = rc.st, rc.st.ct, rc.k
    near = sum(ct.size(int(t)) * ct.size(int(s)) for t, s in st.near) * 16.0

    def basis_bytes(pairs, res):
        tot = 0
        for l in range(ct.depth + 1):
            for (t, c) in pairs[l]:
                if ct.is_leaf(t):
                    tot += ct.size(t) * (k if res is None else res.rank[(t, c)])
                else:
                    c2 = st.sd(l, c)
                    for ch in ct.children[t]:
                        if res is None:
                            tot += k * k
                        else:
                            tot += res.rank[(int(ch), c2)] * res.rank[(t, c)]
        return tot * 16.0

    if which == "orig":
        rb = basis_bytes(st.row_pairs, None)
        cb = basis_bytes(st.col_pairs, None)
        coup = len(st.blocks) * k * k * 16.0
        ranks = [k]
    else:
        rb = basis_bytes(st.row_pairs, rc.row)
        cb = basis_bytes(st.col_pairs, rc.col)
        coup = 0.0
        for b in range(len(st.blocks)):
            t, s, c = (int(v) for v in st.blocks[b])
            coup += rc.row.rank[(t, c)] * rc.col.rank[(s, c)] * 16.0
        ranks = list(rc.row.rank.values()) + list(rc.col.rank.values())
    n = st.n
    return dict(n=n, row_basis_bytes=rb, col_basis_bytes=cb, coupling_bytes=coup, nearfield_bytes=near,
                kb_per_dof_basis=(rb + cb) / n / 1024.0,
                kb_per_dof_matrix=(rb + cb + coup + near) / n / 1024.0,
                max_rank=int(max(ranks)) if ranks else 0,
                mean_rank=float(np.mean(ranks)) if ranks else 0.0)
