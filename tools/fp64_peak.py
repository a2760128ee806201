"""Measure the B200's FP64 peaks on the box ("must be measured"):
scalar DFMA, the FP64 tensor core (mma.sync m8n8k4 -> DMMA.8x8x4), and cuBLAS DGEMM / ZGEMM
through torch.matmul, each as a burst (best of 10 launches) and sustained (back to back for
~4 s), with nvidia-smi clocks sampled during the sustained loops.  Writes one JSON document
(stdout and --out)."""
import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "fp64_peak.so")


def build():
    src = os.path.join(HERE, "fp64_peak.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                        "-o", SO, src], check=True)
    lib = ctypes.CDLL(SO)
    lib.fp64_run.restype = ctypes.c_double
    lib.fp64_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    lib.fp64_flops.restype = ctypes.c_double
    lib.fp64_flops.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    return lib


class Clocks:
    def __init__(self):
        self.samples, self.stop = [], False

    def run(self):
        q = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"
        while not self.stop:
            try:
                o = subprocess.run(["nvidia-smi", "--query-gpu=" + q, "--format=csv,noheader,nounits", "-i", "0"],
                                   capture_output=True, text=True, timeout=5).stdout.strip().split(",")
                self.samples.append([float(o[0]), float(o[1]), float(o[2]), o[3].strip()])
            except Exception:
                pass
            time.sleep(0.2)

    def __enter__(self):
        self.th = threading.Thread(target=self.run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop = True
        self.th.join()

    def summary(self):
        if not self.samples:
            return None
        sm = sorted(s[0] for s in self.samples)
        return {"sm_mhz_median": sm[len(sm) // 2], "sm_max_mhz": self.samples[0][1],
                "power_w_max": max(s[2] for s in self.samples), "reasons": sorted({s[3] for s in self.samples})}


def kernel_peak(lib, kind, nsm):
    blocks, iters = nsm * 8, 2000
    lib.fp64_run(kind, blocks, 100)  # warm-up
    fl = lib.fp64_flops(kind, blocks, iters)
    best = min(lib.fp64_run(kind, blocks, iters) for _ in range(10))
    t0, n, tot = time.time(), 0, 0.0
    with Clocks() as ck:
        while time.time() - t0 < 4.0:
            tot += lib.fp64_run(kind, blocks, iters)
            n += 1
    return {"burst_tflops": fl / best / 1e9, "sustained_tflops": fl * n / tot / 1e9, "launch_ms": best,
            "blocks": blocks, "clocks": ck.summary()}


def gemm_peak(dtype, N):
    import torch
    a = torch.randn(N, N, dtype=dtype, device="cuda")
    b = torch.randn(N, N, dtype=dtype, device="cuda")
    fl = (8.0 if dtype.is_complex else 2.0) * N ** 3
    torch.matmul(a, b)
    torch.cuda.synchronize()
    times = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    t0, n = time.time(), 0
    with Clocks() as ck:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        while time.time() - t0 < 4.0:
            torch.matmul(a, b)
            n += 1
            if n % 4 == 0:
                torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        tot = e0.elapsed_time(e1)
    return {"burst_tflops": fl / min(times) / 1e9, "sustained_tflops": fl * n / tot / 1e9, "N": N,
            "clocks": ck.summary()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    lib = build()
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    res = {"gpu": torch.cuda.get_device_name(0), "sms": nsm,
           "dfma": kernel_peak(lib, 0, nsm), "dmma_m8n8k4": kernel_peak(lib, 1, nsm),
           "cublas_dgemm": gemm_peak(torch.float64, 8192), "cublas_zgemm": gemm_peak(torch.complex128, 4096),
           "how": "DFMA: 148x8 CTAs x 256 threads, 8 independent FMA chains per thread; DMMA: same grid, "
                  "4 independent mma.sync.m8n8k4.f64 accumulators per warp (512 flop each); cuBLAS via torch.matmul "
                  "(DGEMM 8192^3 = 2N^3, ZGEMM 4096^3 = 8N^3 flops); burst = best of 10 (5 for GEMM) CUDA-event "
                  "timed launches, sustained = back to back for 4 s"}
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    sys.exit(main())
