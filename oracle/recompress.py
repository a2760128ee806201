"""Oracle "O-fast": the DH^2 recompression of PAPER.md §3.2 (TEST INFRASTRUCTURE ONLY).

Step by step, in the paper's order and notation (W = V for the single layer
potential):

  basis weights  R_tc      bottom-up  (Eq. 18; [BO10, Alg. 16]):
      leaf:      V_tc = P R_tc  (R = V, P = I, when #t <= k; else R of QR(V_tc))
      non-leaf:  R_tc = R of QR([R_{t1c1} E_{t1c}; R_{t2c2} E_{t2c}])
  block weights  w_b = 1/||R_tc S_b R_sc^*||_F = 1/||G_b||_F   (reading Q12, FROB_BLOCKREL)
  total weights  Zhat_tc   top-down:
      Z_tc = [w_b S_b R_sc^* (s in row(t,c)) | E_{tc+} Zhat_{t+c+}^* (c+ in sd^{-1}(c))],
      Zhat_tc = R of the skinny QR  Phat Zhat = Z_tc^*; gamma = 0 at the root
  truncation     Q_tc, F, C bottom-up:
      leaf:      SVD of V_tc Zhat_tc^*, Q = first k_tc left singular vectors, C = Q^* V
      non-leaf:  Vhat = [C_{t1c1} E_{t1c}; C_{t2c2} E_{t2c}], SVD of Vhat Zhat^*,
                 Qhat = [F_{t1c}; F_{t2c}], C = Qhat^* Vhat            (Eq. 19)
  column basis   the same on the adjoint G^*
  projection     S~_b = C_tc S_b C'_sc^*  (Lemma Projections)

Rank rule (reading Q12):
  FROB_BLOCKREL   k = min{k : sum_{i>k} sigma_i^2 <= eps^2}, blocks weighted by w_b
  FROB_CLUSTERREL k = min{k : sum_{i>k} sigma_i^2 <= eps^2 sum_i sigma_i^2}, w_b = 1
  SPEC_BLOCKREL   k = min{k : sigma_{k+1} <= eps}, blocks weighted by w_b
Isometric factors P are never formed.
"""
import numpy as np
import scipy.linalg as sla

from .interp import Interpolation

MODES = ("FROB_BLOCKREL", "FROB_CLUSTERREL", "SPEC_BLOCKREL")


def qr_r(A, k):
    """R factor of a Householder QR of A (rows x k): shape (min(rows,k), k)."""
    if A.shape[0] == 0:
        return np.zeros((0, k), dtype=np.complex128)
    return np.linalg.qr(A, mode="r")


def svd_left(M):
    """Left singular vectors and ordered singular values (LAPACK zgesvd)."""
    if M.shape[0] == 0 or M.shape[1] == 0:
        return np.zeros((M.shape[0], 0), dtype=np.complex128), np.zeros(0)
    U, s, _ = sla.svd(M, full_matrices=False, lapack_driver="gesvd")
    return U, s


def tail_sums(sigma):
    """tail[k] = sum_{i>=k} sigma_i^2 (0-based), accumulated from the smallest value."""
    sq = sigma * sigma
    tail = np.zeros(len(sigma) + 1)
    acc = 0.0
    for i in range(len(sigma) - 1, -1, -1):
        acc += sq[i]
        tail[i] = acc
    return tail


def select_rank(sigma, eps, mode):
    """Smallest k satisfying the rule of `mode` (see module docstring)."""
    n = len(sigma)
    if mode == "SPEC_BLOCKREL":
        for k in range(n + 1):
            nxt = sigma[k] if k < n else 0.0
            if nxt <= eps:
                return k
        return n
    tail = tail_sums(sigma)
    thr = eps * eps if mode == "FROB_BLOCKREL" else eps * eps * tail[0]
    for k in range(n + 1):
        if tail[k] <= thr:
            return k
    return n


class PassResult:
    def __init__(self, name):
        self.name = name
        self.Zhat, self.Q, self.F, self.C, self.rank, self.sigma = {}, {}, {}, {}, {}, {}


class Recompression:
    def __init__(self, st, eps, mode="FROB_BLOCKREL", interp=None, forced_ranks=None):
        if mode not in MODES:
            raise ValueError("unknown mode %r" % (mode,))
        self.st = st
        self.eps = float(eps)
        self.mode = mode
        self.ip = interp if interp is not None else Interpolation(st)
        self.forced = forced_ranks or {}
        self.k = st.k
        self._V, self._E, self._S = {}, {}, {}

    # ---- cached interpolation quantities ----
    def V(self, t, c):
        key = (t, c)
        if key not in self._V:
            self._V[key] = self.ip.leaf_V(t, c)
        return self._V[key]

    def E(self, tchild, c):
        key = (tchild, c)
        if key not in self._E:
            self._E[key] = self.ip.E(tchild, c)
        return self._E[key]

    def S(self, b):
        if b not in self._S:
            t, s, c = (int(v) for v in self.st.blocks[b])
            self._S[b] = self.ip.S(t, s, c)
        return self._S[b]

    # ---- basis weights (Eq. 18) ----
    def basis_weights(self):
        st, ct, k = self.st, self.st.ct, self.k
        self.R = {}
        for l in range(ct.depth, -1, -1):
            for (t, c) in st.basis_pairs[l]:
                if ct.is_leaf(t):
                    V = self.V(t, c)
                    self.R[(t, c)] = V if V.shape[0] <= k else qr_r(V, k)
                else:
                    c2 = st.sd(l, c)
                    X = np.vstack([self.R[(int(ch), c2)] @ self.E(int(ch), c) for ch in ct.children[t]])
                    self.R[(t, c)] = qr_r(X, k)

    # ---- block weights (reading Q12) ----
    def block_weights(self):
        st = self.st
        nb = len(st.blocks)
        self.normG = np.zeros(nb)
        for b in range(nb):
            t, s, c = (int(v) for v in st.blocks[b])
            self.normG[b] = np.linalg.norm(self.R[(t, c)] @ self.S(b) @ self.R[(s, c)].conj().T)
        if self.mode == "FROB_CLUSTERREL":
            self.omega = np.ones(nb)
        else:
            self.omega = 1.0 / self.normG

    # ---- total weights + truncation for one side ----
    def run_pass(self, side):
        st, ct, k = self.st, self.st.ct, self.k
        res = PassResult(side)
        pairs = st.row_pairs if side == "row" else st.col_pairs
        blocks_of = st.row_blocks if side == "row" else st.col_blocks
        pmap = st.parent_map(pairs)
        # total weights, top-down
        for l in range(ct.depth + 1):
            for (t, c) in pairs[l]:
                rows = []
                for b in blocks_of.get((t, c), []):
                    bt, bs, _ = (int(v) for v in st.blocks[b])
                    if side == "row":
                        # (w_b S_b R_sc^*)^* = w_b R_sc S_b^*
                        rows.append(self.omega[b] * (self.R[(bs, c)] @ self.S(b).conj().T))
                    else:
                        # adjoint: block contributes w_b S_b^* R_tc^*, i.e. rows w_b R_tc S_b
                        rows.append(self.omega[b] * (self.R[(bt, c)] @ self.S(b)))
                tp = int(ct.parent[t])
                for cp in pmap.get((t, c), []):
                    # (E_{tc+} Zhat_{t+c+}^*)^* = Zhat_{t+c+} E_{tc+}^*
                    rows.append(res.Zhat[(tp, cp)] @ self.E(t, cp).conj().T)
                Zs = np.vstack(rows) if rows else np.zeros((0, k), dtype=np.complex128)
                res.Zhat[(t, c)] = qr_r(Zs, k)
        # truncation, bottom-up
        for l in range(ct.depth, -1, -1):
            for (t, c) in pairs[l]:
                Zh = res.Zhat[(t, c)]
                if ct.is_leaf(t):
                    Vt = self.V(t, c)
                else:
                    c2 = st.sd(l, c)
                    Vt = np.vstack([res.C[(int(ch), c2)] @ self.E(int(ch), c) for ch in ct.children[t]])
                M = Vt @ Zh.conj().T
                U, s = svd_left(M)
                kk = self.forced.get((side, t, c))
                if kk is None:
                    kk = select_rank(s, self.eps, self.mode)
                Q = U[:, :kk]
                res.rank[(t, c)] = kk
                res.sigma[(t, c)] = s
                res.C[(t, c)] = Q.conj().T @ Vt
                if ct.is_leaf(t):
                    res.Q[(t, c)] = Q
                else:
                    k1 = res.rank[(int(ct.children[t, 0]), st.sd(l, c))]
                    res.F[(t, c)] = (Q[:k1], Q[k1:])
        return res

    # ---- projection (Lemma Projections) ----
    def project(self):
        st = self.st
        self.St = {}
        for b in range(len(st.blocks)):
            t, s, c = (int(v) for v in st.blocks[b])
            self.St[b] = self.row.C[(t, c)] @ self.S(b) @ self.col.C[(s, c)].conj().T

    def run(self):
        self.basis_weights()
        self.block_weights()
        self.row = self.run_pass("row")
        self.col = self.run_pass("col")
        self.project()
        return self

    # ---- certified quantities ----
    def discarded(self, res):
        tot = 0.0
        for key, s in res.sigma.items():
            kk = res.rank[key]
            tot += float(np.sum(s[kk:] * s[kk:]))
        return tot

    def far_norm2(self):
        return float(np.sum(self.normG * self.normG))
