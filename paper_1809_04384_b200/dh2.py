"""Thin ctypes binding of libdh2.so (include/dh2.h): argument marshalling only.

Every step of the DH^2 path runs in the library's sm_100a kernels; there is no
Python or CPU fallback.  If libdh2.so is missing the import fails loudly.
"""
import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdh2.so")

DH2_OK, DH2_EINVAL, DH2_ENOMEM, DH2_ECUDA, DH2_ENCCL, DH2_ESTATE, DH2_EMISMATCH, DH2_ENOTIMPL, DH2_ENUMERIC = (
    0, -1, -2, -3, -4, -5, -6, -7, -8)
ERROR_NAMES = {-1: "DH2_EINVAL", -2: "DH2_ENOMEM", -3: "DH2_ECUDA", -4: "DH2_ENCCL", -5: "DH2_ESTATE",
               -6: "DH2_EMISMATCH", -7: "DH2_ENOTIMPL", -8: "DH2_ENUMERIC"}
MODES = {"FROB_BLOCKREL": 0, "FROB_CLUSTERREL": 1, "SPEC_BLOCKREL": 2}
DH2_ORIG, DH2_RECOMP = 0, 1
DH2_HOST_PTRS, DH2_DEVICE_PTRS, DH2_ADD_NEAR = 0, 1, 2

# every symbol include/dh2.h declares
EXPORTED = ["dh2_build_interp", "dh2_setup_device", "dh2_recompress", "dh2_matvec", "dh2_nearfield_assemble", "dh2_storage",
            "dh2_set_stream", "dh2_set_option", "dh2_set_profiling", "dh2_get_stats", "dh2_export", "dh2_export_shard",
            "dh2_nccl_unique_id", "dh2_destroy", "dh2_last_error"]


class dh2_mesh(ctypes.Structure):
    _fields_ = [("nv", ctypes.c_int64), ("nt", ctypes.c_int64),
                ("xyz", ctypes.POINTER(ctypes.c_double)), ("tri", ctypes.POINTER(ctypes.c_int64))]


class dh2_params(ctypes.Structure):
    _fields_ = [("kappa", ctypes.c_double), ("m", ctypes.c_int32), ("leaf_size", ctypes.c_int32),
                ("eta1", ctypes.c_double), ("eta2", ctypes.c_double), ("quad", ctypes.c_int32)]


class dh2_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_uid", ctypes.c_void_p),
                ("device", ctypes.c_int32)]


class dh2_storage_report(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("row_basis_bytes", ctypes.c_double), ("col_basis_bytes", ctypes.c_double),
                ("coupling_bytes", ctypes.c_double), ("nearfield_bytes", ctypes.c_double),
                ("kb_per_dof_basis", ctypes.c_double), ("kb_per_dof_matrix", ctypes.c_double),
                ("max_rank", ctypes.c_int32), ("mean_rank", ctypes.c_double)]


class DH2Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s (%d): %s" % (ERROR_NAMES.get(code, "?"), code, msg))
        self.code = code


_lib = None


def load_library(path=LIB_PATH):
    """Load libdh2.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError("libdh2.so not built at %s (run paper_1809_04384_b200/build.py)" % path)
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    lib.dh2_build_interp.argtypes = [P(dh2_mesh), P(dh2_params), P(dh2_dist), P(vp)]
    lib.dh2_setup_device.argtypes = [vp]
    lib.dh2_recompress.argtypes = [vp, ctypes.c_double, ctypes.c_int32]
    lib.dh2_matvec.argtypes = [vp, ctypes.c_int32, vp, vp, ctypes.c_int32]
    lib.dh2_nearfield_assemble.argtypes = [vp, ctypes.c_int32, ctypes.c_int32]
    lib.dh2_storage.argtypes = [vp, ctypes.c_int32, P(dh2_storage_report)]
    lib.dh2_set_stream.argtypes = [vp, vp]
    lib.dh2_set_profiling.argtypes = [vp, ctypes.c_int32]
    lib.dh2_set_option.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
    lib.dh2_get_stats.argtypes = [vp, ctypes.c_char_p, P(ctypes.c_int64)]
    lib.dh2_export.argtypes = [vp, ctypes.c_char_p, vp, P(ctypes.c_int64)]
    lib.dh2_export_shard.argtypes = [vp, ctypes.c_int32, ctypes.c_char_p, vp, P(ctypes.c_int64)]
    lib.dh2_nccl_unique_id.argtypes = [vp]
    lib.dh2_destroy.argtypes = [vp]
    lib.dh2_last_error.argtypes = [vp]
    lib.dh2_last_error.restype = ctypes.c_char_p
    for name in EXPORTED:
        if name != "dh2_last_error":
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def nccl_unique_id():
    """128-byte ncclUniqueId (bytes) for dh2_build_interp with world > 1 (rank 0 creates it)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    rc = lib.dh2_nccl_unique_id(buf)
    if rc != DH2_OK:
        raise DH2Error(rc, lib.dh2_last_error(None).decode())
    return buf.raw


class DH2:
    """One DH^2 matrix: dh2_build_interp -> dh2_recompress -> dh2_matvec / dh2_storage.

    world > 1 partitions the matrix into `world` subtree shards (include/dh2.h, dh2_dist):
    with nccl_uid (bytes from nccl_unique_id() on rank 0) this process is shard `rank` of an
    NCCL job; without it, all shards run in this process on `device` (virtual mode)."""

    def __init__(self, xyz, tri, kappa, m, leaf, eta1=1.0, eta2=10.0, device=0, world=1, rank=0, nccl_uid=None):
        self.lib = load_library()
        self._xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        self._tri = np.ascontiguousarray(tri, dtype=np.int64)
        mesh = dh2_mesh(self._xyz.shape[0], self._tri.shape[0],
                        self._xyz.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                        self._tri.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
        prm = dh2_params(float(kappa), int(m), int(leaf), float(eta1), float(eta2), 7)
        self._uid = ctypes.create_string_buffer(bytes(nccl_uid), 128) if nccl_uid is not None else None
        dist = dh2_dist(int(rank), int(world), ctypes.cast(self._uid, ctypes.c_void_p) if self._uid is not None else None,
                        int(device))
        h = ctypes.c_void_p()
        rc = self.lib.dh2_build_interp(ctypes.byref(mesh), ctypes.byref(prm), ctypes.byref(dist), ctypes.byref(h))
        if rc != DH2_OK:
            raise DH2Error(rc, self.lib.dh2_last_error(None).decode())
        self.h = h
        self.n = int(self._tri.shape[0])
        self.k = int(m) ** 3

    def _check(self, rc):
        if rc != DH2_OK:
            raise DH2Error(rc, self.lib.dh2_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.dh2_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def setup_device(self):
        self._check(self.lib.dh2_setup_device(self.h))

    def recompress(self, eps, mode="FROB_BLOCKREL"):
        self._check(self.lib.dh2_recompress(self.h, float(eps), MODES[mode] if isinstance(mode, str) else int(mode)))

    def matvec(self, x, which=DH2_RECOMP, add_near=False):
        """y = G_far x (admissible blocks); with add_near, y = G x = G_far x + N x (the nearfield
        of nearfield_assemble)."""
        x = np.ascontiguousarray(x, dtype=np.complex128)
        if x.shape != (self.n,):
            raise ValueError("x must have shape (n,)")
        y = np.empty_like(x)
        self._check(self.lib.dh2_matvec(self.h, which, x.ctypes.data, y.ctypes.data,
                                        DH2_HOST_PTRS | (DH2_ADD_NEAR if add_near else 0)))
        return y

    def matvec_device(self, x_ptr, y_ptr, which=DH2_RECOMP, add_near=False):
        """x_ptr, y_ptr: device pointers to n complex128 values (e.g. torch tensor data_ptr())."""
        self._check(self.lib.dh2_matvec(self.h, which, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                        DH2_DEVICE_PTRS | (DH2_ADD_NEAR if add_near else 0)))

    def nearfield_assemble(self, nq_singular=5, nq_regular=3):
        """Assemble the nearfield blocks on the device (NEXT-4; the paper's orders by default)."""
        self._check(self.lib.dh2_nearfield_assemble(self.h, int(nq_singular), int(nq_regular)))

    def storage(self, which=DH2_RECOMP):
        rep = dh2_storage_report()
        self._check(self.lib.dh2_storage(self.h, which, ctypes.byref(rep)))
        return {f: getattr(rep, f) for f, _ in dh2_storage_report._fields_}

    def set_stream(self, stream_ptr):
        self._check(self.lib.dh2_set_stream(self.h, ctypes.c_void_p(stream_ptr)))

    def set_option(self, name, value):
        self._check(self.lib.dh2_set_option(self.h, name.encode(), int(value)))

    def set_profiling(self, on=True):
        self._check(self.lib.dh2_set_profiling(self.h, 1 if on else 0))

    def stats(self):
        ln = ctypes.c_int64(0)
        self._check(self.lib.dh2_get_stats(self.h, None, ctypes.byref(ln)))
        buf = ctypes.create_string_buffer(ln.value)
        self._check(self.lib.dh2_get_stats(self.h, buf, ctypes.byref(ln)))
        return json.loads(buf.value.decode())

    def export(self, name, dtype, shard=None):
        nb = ctypes.c_int64(0)
        if shard is None:
            call = lambda buf: self.lib.dh2_export(self.h, name.encode(), buf, ctypes.byref(nb))  # noqa: E731
        else:
            call = lambda buf: self.lib.dh2_export_shard(self.h, int(shard), name.encode(), buf, ctypes.byref(nb))  # noqa: E731
        self._check(call(None))
        out = np.empty(nb.value // np.dtype(dtype).itemsize, dtype=dtype)
        if nb.value:
            self._check(call(out.ctypes.data))
        return out

    def exchange_lists(self, shard=None):
        """Partition exchange items: {kind: [ids per peer]} for kind in xR_send, xR_recv,
        xC_send, xC_recv (see include/dh2.h, dh2_export_shard)."""
        out = {}
        for kind in ("xR_send", "xR_recv", "xC_send", "xC_recv"):
            a = self.export(kind, np.int32, shard=0 if shard is None else shard)
            lists, i = [], 0
            while i < len(a):
                c = int(a[i])
                lists.append(a[i + 1:i + 1 + c].tolist())
                i += 1 + c
            out[kind] = lists
        return out
