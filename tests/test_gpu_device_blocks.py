"""Unit tests of the device building blocks (QR, pivoted QR, one-sided Jacobi) against numpy,
through a test-only CUDA harness (tests/cuda/devtest.cu) built with the same flags."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cuda", "devtest.cu")
LIB = os.path.join(HERE, "cuda", "libdevtest.so")


@pytest.fixture(scope="module")
def dev():
    hdr = os.path.join(HERE, "..", "paper_1809_04384_b200", "csrc", "dh2_device.cuh")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(hdr)):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                        "-Xcompiler", "-fPIC", "-o", LIB, SRC], check=True)
    lib = ctypes.CDLL(LIB)
    lib.devtest_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    return lib


def run(lib, op, A, threads=128):
    batch, M, N = A.shape
    a = np.ascontiguousarray(A.transpose(0, 2, 1)).astype(np.complex128)  # column-major per matrix
    out = np.empty_like(a)
    iout = np.empty(batch * (N + 1), dtype=np.int32)
    dout = np.empty(batch * M, dtype=np.float64)
    rc = lib.devtest_run(op, a.ctypes.data, out.ctypes.data, iout.ctypes.data, dout.ctypes.data, batch, M, N, threads)
    assert rc == 0
    return out.transpose(0, 2, 1), iout.reshape(batch, N + 1), dout.reshape(batch, M)


def graded(rng, batch, M, N, decay):
    U = np.linalg.qr(rng.normal(size=(batch, M, M)) + 1j * rng.normal(size=(batch, M, M)))[0]
    V = np.linalg.qr(rng.normal(size=(batch, N, N)) + 1j * rng.normal(size=(batch, N, N)))[0]
    k = min(M, N)
    s = decay ** np.arange(k)
    S = np.zeros((batch, M, N))
    S[:, np.arange(k), np.arange(k)] = s
    return U @ S @ V.conj().transpose(0, 2, 1), s


def r_factor(out, iout, op, K, N):
    """R in pivoted (logical) column order: ops 7/8 leave the columns in place and report the
    pivot order piv[0:steps]; the columns never pivoted follow in increasing order."""
    if op in (7, 8):
        steps = iout[0]
        piv = list(iout[1:1 + steps])
        piv += [c for c in range(N) if c not in piv]
        piv = np.array(piv)
        return np.triu(out[:K][:, piv]), piv
    piv = iout[1:] if op else np.arange(N)
    return np.triu(out[:K]), piv


@pytest.mark.parametrize("M,N", [(5, 3), (27, 5), (52, 32), (64, 64), (100, 64), (128, 64)])
@pytest.mark.parametrize("op", [0, 1, 2, 7])
def test_qr_variants(dev, op, M, N):
    rng = np.random.default_rng(M * 100 + N)
    A = rng.normal(size=(6, M, N)) + 1j * rng.normal(size=(6, M, N))
    out, iout, _ = run(dev, op, A)
    K = min(M, N)
    for b in range(6):
        R, piv = r_factor(out[b], iout[b], op, K, N)
        Ap = A[b][:, piv]
        assert sorted(piv.tolist()) == list(range(N))
        G = Ap.conj().T @ Ap
        assert np.abs(R.conj().T @ R - G).max() <= 1e-13 * np.abs(G).max()
        if op:  # pivoting makes |r_jj| non-increasing
            d = np.abs(np.diag(R))
            assert np.all(d[1:] <= d[:-1] * (1 + 1e-12))


@pytest.mark.parametrize("nv,L", [(2, 3), (5, 5), (5, 12), (14, 20), (32, 32), (20, 64), (32, 100)])
@pytest.mark.parametrize("op", [3, 4])
def test_jacobi_rows(dev, op, nv, L):
    rng = np.random.default_rng(nv * 1000 + L)
    X, s = graded(rng, 5, nv, L, 0.3)
    out, iout, dout = run(dev, op, X)
    for b in range(5):
        Y = out[b]
        # rows mutually orthogonal, row space preserved, norms = singular values
        G = Y @ Y.conj().T
        off = G - np.diag(np.diag(G))
        assert np.abs(off).max() <= 1e-14 * np.abs(G).max() * nv
        sv = np.sort(np.sqrt(np.real(np.diag(G))))[::-1]
        ref = np.linalg.svd(X[b], compute_uv=False)
        assert np.abs(sv - ref).max() <= 1e-13 * ref[0]
        assert np.allclose(np.sort(np.sqrt(dout[b][:nv]))[::-1], ref, rtol=0, atol=1e-13 * ref[0])


@pytest.mark.parametrize("M,N", [(27, 13), (16, 14), (52, 32), (64, 64)])
@pytest.mark.parametrize("op", [5, 6, 8])
def test_qrcp_rank_stop(dev, op, M, N):
    """With the numerical-rank stop (trailing ||R22||_F^2 <= 1e-26 max column norm^2, the
    truncation's threshold), a graded matrix is factorised at least while the singular-value tail
    exceeds 1e-13 sigma_1 (||R22||_F^2 >= sum_{j > i} sigma_j^2), and an exactly rank-r matrix
    stops at r or r + 1 with the leading rows exact."""
    rng = np.random.default_rng(7)
    A, s = graded(rng, 4, M, N, 0.6)
    out, iout, _ = run(dev, op, A)
    K = min(M, N)
    tail2 = np.cumsum((s * s)[::-1])[::-1]  # tail2[i] = sum_{j >= i} sigma_j^2
    need = int(np.sum(tail2 > 1e-26 * s[0] ** 2))
    assert np.all((iout[:, 0] >= need) & (iout[:, 0] <= K)), (iout[:, 0], need)
    r = 5
    B = A[:, :, :r] @ (rng.normal(size=(4, r, N)) + 1j * rng.normal(size=(4, r, N)))
    out, iout, _ = run(dev, op, B)
    assert np.all(iout[:, 0] <= r + 1), iout[:, 0]
    for b in range(4):
        k = iout[b, 0]
        R, piv = r_factor(out[b], iout[b], op, k, N)
        Bp = B[b][:, piv]
        G = Bp.conj().T @ Bp
        assert np.abs(R.conj().T @ R - G).max() <= 1e-12 * np.abs(G).max()


@pytest.mark.parametrize("op", [5, 6, 8])
def test_qrcp_on_oracle_truncation_matrices(dev, op):
    """M^* = Zhat Vhat^* of every non-leaf row pair of P1 (from the oracle): the rank-stopped
    pivoted QR keeps R^*R = (M^* Pi)^*(M^* Pi) up to the dropped trailing block."""
    from conftest import oracle_run
    rc = oracle_run("P1")
    st, ct = rc.st, rc.st.ct
    mats = []
    for l in st.active_levels:
        for (t, c) in st.row_pairs[l]:
            if ct.is_leaf(t):
                continue
            c2 = st.sd(l, c)
            Vh = np.vstack([rc.row.C[(int(ch), c2)] @ rc.E(int(ch), c) for ch in ct.children[t]])
            mats.append((Vh @ rc.row.Zhat[(t, c)].conj().T).conj().T)
    shapes = {}
    for A in mats:
        shapes.setdefault(A.shape, []).append(A)
    for (M, N), As in shapes.items():
        A = np.stack(As)
        out, iout, _ = run(dev, op, A)
        for b in range(len(As)):
            k = iout[b, 0]
            R, piv = r_factor(out[b], iout[b], op, k, N)
            sv = np.linalg.svd(A[b], compute_uv=False)
            svR = np.linalg.svd(R, compute_uv=False)
            n = min(len(sv), len(svR))
            assert np.abs(sv[:n] - svR[:n]).max() <= 2e-13 * sv[0], (M, N, k, sv, svR)  # Weyl: dropped block <= 1e-13 sigma_1
            assert np.all(sv[n:] <= 1e-13 * sv[0]), (M, N, k, sv)


@pytest.mark.parametrize("nb", [1, 8, 13, 32, 64])
@pytest.mark.parametrize("conj_s,strided", [(1, 0), (0, 0), (0, 1)])
def test_dmma_gemm(dev, nb, conj_s, strided):
    """FP64 tensor-core (DMMA) complex GEMM: out = 0.5 X op(S) to 1e-14 relative."""
    rng = np.random.default_rng(nb * 10 + conj_s + 2 * strided)
    k = 64
    X = rng.normal(size=(nb, k)) + 1j * rng.normal(size=(nb, k))
    S = rng.normal(size=(k, k)) + 1j * rng.normal(size=(k, k))
    Xc = np.ascontiguousarray(X.T).astype(np.complex128)   # column-major
    Sc = np.ascontiguousarray(S.T).astype(np.complex128)   # column-major: Sg[i + j k] = S[i, j]
    out = np.empty(nb * k, dtype=np.complex128)
    dev.devtest_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4
    assert dev.devtest_gemm(Xc.ctypes.data, Sc.ctypes.data, out.ctypes.data, nb, k, conj_s, strided) == 0
    got = out.reshape(k, nb).T
    # op(S)[mu, nu] = Sg[nu + mu k] = S[nu, mu] (transposed), or Sg[mu + nu k] = S[mu, nu] if strided
    opS = S if strided else S.T
    if conj_s:
        opS = opS.conj()
    ref = 0.5 * X @ opS
    assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max() * 4


@pytest.mark.parametrize("M,N", [(250, 125), (96, 64), (40, 27), (300, 125), (33, 125)])
@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4, 5])
def test_qr_append_chunks(dev, M, N, mode):
    """R of a tall A by 32-row chunks appended into a triangle (structured Householder; modes 1/3 the
    blocked compact-WY form with DMMA trailing updates, 4/5 flag-synchronised without block barriers,
    2/3/5 on the packed triangle): R^*R = A^*A."""
    if mode in (0, 1, 4) and N > 100:
        pytest.skip("the dense k x k triangle does not fit shared memory for k > 100 (the library packs it)")
    dev.devtest_append.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int]
    rng = np.random.default_rng(M * 7 + N + mode)
    A = rng.normal(size=(M, N)) + 1j * rng.normal(size=(M, N))
    A[:, 3] = 0.0  # a numerically zero column (HH_TINY path)
    A[:, 5] = A[:, 4]  # exactly dependent columns
    a = np.ascontiguousarray(A.T)  # column-major
    R = np.empty((N, N), dtype=np.complex128)
    assert dev.devtest_append(mode, a.ctypes.data, R.ctypes.data, M, N, 512) == 0
    R = R.T.copy()  # column-major -> (N, N)
    assert np.allclose(np.tril(R, -1), 0)
    G0 = A.conj().T @ A
    assert np.abs(R.conj().T @ R - G0).max() <= 1e-12 * np.abs(G0).max()
    # (with a zero and two equal columns R is not unique: only its Gram matrix is compared)
