"""Read the CUDA path's results back through dh2_export and arrange them like the oracle's
result objects (same (t,c) keys), so tests can compare invariants pair by pair and reuse the
oracle's dense-expansion helpers.  Test infrastructure only."""
import numpy as np

from oracle.recompress import PassResult


def _cm(a, off, rows, cols, ld=None):
    """Column-major slab -> (rows, cols) array."""
    ld = rows if ld is None else ld
    if rows == 0 or cols == 0:
        return np.zeros((rows, cols), dtype=np.complex128)
    return a[off:off + ld * cols].reshape(cols, ld).T[:rows, :].copy()


class GpuView:
    def __init__(self, h, st, recompressed=True):
        self.h = h
        self.st = st
        self.k = st.k
        k = self.k
        bp = h.export("basis_pairs", np.int64).reshape(-1, 3)
        self.bp_key = [(int(t), int(c)) for _, t, c in bp]
        self.bp_id = {key: i for i, key in enumerate(self.bp_key)}
        self.VR = h.export("VR", np.complex128)
        self.V_off = h.export("bp_V_off", np.int64)
        self.R_off = h.export("bp_R_off", np.int64)
        self.R_rows = h.export("bp_R_rows", np.int32)
        self.E_off = h.export("bp_E_off", np.int64)
        # adjoint symmetry: only ROW basis pairs are set up / weighted; a column-only pair (t,c) is
        # the conjugate of the row pair (t,-c)
        self.bp_neg = h.export("bp_neg", np.int32)
        rp = h.export("row_pairs", np.int64).reshape(-1, 3)
        self.is_row = np.zeros(len(bp), bool)
        for _, t, c in rp:
            self.is_row[self.bp_id[(int(t), int(c))]] = True
        sym = h.stats()["adjoint_symmetry"]
        self.sym_ve = bool(sym.get("row_only_setup", False))
        self.sym_r = bool(sym["used"])
        self.Eall = h.export("E", np.complex128)
        self.S_all = h.export("S", np.complex128)
        if recompressed:
            self.omega = h.export("omega", np.float64)
            self.normG2 = h.export("normG2", np.float64)
            self.row = self._pass("row")
            self.col = self._pass("col")
            St = h.export("St", np.complex128)
            St_off = h.export("blk_St_off", np.int64)
            prow, pcol = h.export("blk_prow", np.int32), h.export("blk_pcol", np.int32)
            self.St = {}
            for b in range(len(st.blocks)):
                kt = self.row.rank_arr[prow[b]]
                ks = self.col.rank_arr[pcol[b]]
                self.St[b] = _cm(St, St_off[b], kt, ks, self.row.kb[prow[b]])
        del k

    def _mirror(self, t, c, flag):
        """(basis pair id holding the data, conjugate?) for (t,c)."""
        i = self.bp_id[(t, c)]
        if flag and not self.is_row[i]:
            return int(self.bp_neg[i]), True
        return i, False

    def V(self, t, c):
        i, cj = self._mirror(t, c, self.sym_ve)
        rows = self.st.ct.size(t)
        v = _cm(self.VR, self.V_off[i], rows, self.k)
        return v.conj() if cj else v

    def R(self, t, c):
        i, cj = self._mirror(t, c, self.sym_r)
        r = _cm(self.VR, self.R_off[i], int(self.R_rows[i]), self.k)
        return r.conj() if cj else r

    def E_factors(self, t, c, child):
        i, cj = self._mirror(t, c, self.sym_ve)
        m = self.st.m
        off = self.E_off[i] + child * 3 * m * m
        f = [self.Eall[off + a * m * m: off + (a + 1) * m * m].reshape(m, m) for a in range(3)]
        return [x.conj() for x in f] if cj else f

    def E_dense(self, t, c, child):
        ex, ey, ez = self.E_factors(t, c, child)
        return np.kron(ez, np.kron(ey, ex))

    def S(self, b):
        k = self.k
        return self.S_all[b * k * k:(b + 1) * k * k].reshape(k, k).T.copy()

    def _pass(self, side):
        h, st, k = self.h, self.st, self.k
        res = PassResult(side)
        pairs = h.export(side + "_pairs", np.int64).reshape(-1, 3)
        keys = [(int(t), int(c)) for _, t, c in pairs]
        Z = h.export("Z_" + side, np.complex128)
        Z_off = h.export("Z_off_" + side, np.int64)
        Z_rows = h.export("Z_rows_" + side, np.int32)
        rank = h.export("rank_" + side, np.int32)
        sig = h.export("sigma_" + side, np.float64)
        sig_off = h.export("sig_off_" + side, np.int64)
        nsig = h.export("nsig_" + side, np.int32)
        Q = h.export("Q_" + side, np.complex128)
        Q_off = h.export("Q_off_" + side, np.int64)
        C = h.export("C_" + side, np.complex128)
        C_off = h.export("C_off_" + side, np.int64)
        kb = h.export("kb_" + side, np.int32)
        rowsb = h.export("rowsb_" + side, np.int32)
        child0 = h.export("child0_" + side, np.int32)
        child1 = h.export("child1_" + side, np.int32)
        disc = h.export("disc_" + side, np.float64)
        res.rank_arr = rank
        res.kb = kb
        res.disc = {}
        for p, key in enumerate(keys):
            t, c = key
            res.Zhat[key] = _cm(Z, Z_off[p], int(Z_rows[p]), k)
            kk = int(rank[p])
            res.rank[key] = kk
            res.sigma[key] = sig[sig_off[p]:sig_off[p] + nsig[p]].copy()
            res.C[key] = _cm(C, C_off[p], kk, k, int(kb[p]))
            res.disc[key] = float(disc[p])
            if child0[p] < 0:
                res.Q[key] = _cm(Q, Q_off[p], st.ct.size(t), kk)
            else:
                k1 = int(rank[child0[p]])
                k2 = int(rank[child1[p]])
                Qh = _cm(Q, Q_off[p], k1 + k2, kk, int(rowsb[p]))
                res.F[key] = (Qh[:k1], Qh[k1:])
        return res
