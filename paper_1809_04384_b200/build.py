"""In-tree build of libdh2.so for sm_100a (nvcc; no JIT cache, so the .so travels with the repo)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libdh2.so")
SOURCES = ["csrc/dh2_kernels.cu", "csrc/dh2_api.cu", "csrc/dh2_lean.cu", "csrc/dh2_cq.cu", "csrc/dh2_near.cu", "csrc/dh2_host.cpp"]
HEADERS = ["csrc/dh2_device.cuh", "csrc/dh2_kernels.cuh", "csrc/dh2_host.h", "csrc/dh2_shard.h", "../include/dh2.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fopenmp",
    "-diag-suppress", "550,177",
    "-shared",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(HERE, f)) > t for f in SOURCES + HEADERS)


def build(force=False, verbose=False):
    """Compile every source to an object in parallel (one nvcc per file), then link libdh2.so."""
    if not force and not needs_build():
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    with tempfile.TemporaryDirectory() as tmp:
        objs, cmds = [], []
        for src in SOURCES:
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            objs.append(obj)
            cmds.append([_nvcc()] + flags + ["-c", "-o", obj, os.path.join(HERE, src)])
        with ThreadPoolExecutor(len(cmds)) as ex:
            for cmd in cmds:
                if verbose:
                    print(" ".join(cmd), file=sys.stderr)
            list(ex.map(lambda c: subprocess.run(c, check=True, cwd=HERE), cmds))
        link = [_nvcc()] + NVCC_FLAGS + ["-o", LIB] + objs + ["-lgomp"]
        if verbose:
            print(" ".join(link), file=sys.stderr)
        subprocess.run(link, check=True, cwd=HERE)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
