#!/usr/bin/env python
"""Benchmark of the B200 DH^2 hot path (BASELINE.json metric, workload configs[1] = C2).

A step = one pass of the whole hot path of SURVEY §8(a) over the resident input:
device set-up (quadrature, grids, leaf V, transfer factors E, couplings S), the hybrid
recompression (basis weights, block weights, total weights and truncation for rows and
columns, projection) and one far-field matvec of the recompressed matrix.
value = n / device time per step (Mdof/s); e2e = the same through the C ABI from HOST
buffers (mesh in, x in, y out), host structure build and all copies included.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

Under torchrun (N > 1) the matrix is partitioned into N subtree shards, one per GPU, with
NCCL exchanges of the cross-shard factors (include/dh2.h dh2_dist):
the total work is fixed ("strong" scaling) and value = n / (max over ranks of the device
time per step).  The timed region is bracketed by barriers + synchronisation.
--shards P (single process) runs the same partition in the virtual mode on one GPU.
"""
import argparse
import threading
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import get_config, mesh_for, seeded_vector  # noqa: E402

METRIC = "DH2 recompression Mdof/s"
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 148 SMs x 64 DFMA/clk x 2 flop x max SM clock


def workload_desc(cfg):
    shape = "sphere (octahedron refined, q=%d)" % cfg["q"] if cfg["mesh"] == "sphere" else "cube [0,1]^3 (q=%d)" % cfg["q"]
    return "%s: %s, kappa=%g, m=%d (k=%d), leaf %d, eta1=%g, eta2=%g, eps=%g, FROB_BLOCKREL, complex fp64" % (
        cfg["name"], shape, cfg["kappa"], cfg["m"], cfg["m"] ** 3, cfg["leaf"], cfg["eta1"], cfg["eta2"], cfg["eps"])


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi in loop mode (every 50 ms) on a reader thread; start() returns once the first
    sample arrived, begin()/end() bracket the timed region and only samples inside it count."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line))

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        deadline = time.monotonic() + 10.0
        while not self.lines and time.monotonic() < deadline and self.proc.poll() is None:
            time.sleep(0.01)

    def begin(self):
        self.t0 = time.monotonic()

    def end(self):
        self.t1 = time.monotonic()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=10)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=5)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for t, line in self.lines:
            if self.t0 is None or self.t1 is None or not (self.t0 <= t <= self.t1):
                continue
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------- oracle legs
def oracle_sample(cfg, frac=0.125, seed=0):
    """Time the oracle (as it stands) on a bounded sample of the workload: the full §3.2
    pipeline on the sub-matrix made of a seeded random `frac` of the admissible blocks
    (pairs re-closed over them).  Returns (seconds, work units sample, work units full)."""
    from oracle.structure import DH2Structure
    from oracle.recompress import Recompression

    xyz, tri = mesh_for(cfg)
    st = DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])

    def units(s):
        return (sum(len(p) for p in s.basis_pairs) + sum(len(p) for p in s.row_pairs)
                + sum(len(p) for p in s.col_pairs) + len(s.blocks))

    full = units(st)
    rng = np.random.default_rng(seed)
    keep = np.sort(rng.choice(len(st.blocks), size=max(1, int(frac * len(st.blocks))), replace=False))
    st.blocks = st.blocks[keep]
    st._build_pairs()
    samp = units(st)
    t0 = time.perf_counter()
    Recompression(st, cfg["eps"]).run()
    return time.perf_counter() - t0, samp, full


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    times = []
    for i in range(args.warmup + args.steps):
        sec, samp, full = oracle_sample(cfg, args.sample_frac, seed=i)
        if i >= args.warmup:
            times.append(sec * full / samp)
    t = float(np.mean(times))
    n = cfg["n"]
    val = n / t / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "Mdof/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "n": n},
            "cpu_baseline": {"value": val, "unit": "Mdof/s", "cores": 1, "kind": "oracle",
                             "sample": "full §3.2 oracle pipeline on a seeded %.3g fraction of the admissible blocks of "
                                       "the same matrix, extrapolated by work units (pairs+blocks)" % args.sample_frac},
            "e2e": {"value": val, "unit": "Mdof/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--sample-frac", type=float, default=0.125)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shards", type=int, default=1, help="virtual shards on one GPU (single process)")
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="dh2_set_option before recompress (A/B of kernel variants)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = get_config(args.config)
    xyz, tri = mesh_for(cfg)
    cfg["n"] = int(tri.shape[0])

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1809_04384_b200 import DH2, nccl_unique_id

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def make():
        h = make_ctx()
        for o in args.option:
            k, v = o.split("=")
            h.set_option(k, int(v))
        return h

    def make_ctx():
        """collective: one shard per rank (NCCL), or args.shards virtual shards on this GPU"""
        if world > 1:
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            return DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], device=local,
                       world=world, rank=rank, nccl_uid=obj[0])
        return DH2(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"], device=local,
                   world=args.shards)

    n = cfg["n"]
    try:
        h = make()
    except Exception as e:  # e.g. DH2_ENOMEM: the full-materialisation plan exceeds the GPU (C4/C5)
        if rank == 0:
            print(json.dumps({"metric": METRIC, "config": {"workload": workload_desc(cfg), "n": n},
                              "unavailable": str(e).splitlines()[0]}), flush=True)
        return
    stream = torch.cuda.current_stream()
    h.set_stream(stream.cuda_stream)
    x = torch.from_numpy(seeded_vector(n, 1)).to("cuda")
    y = torch.empty_like(x)

    def step():
        h.setup_device()
        h.recompress(cfg["eps"])
        h.matvec_device(x.data_ptr(), y.data_ptr(), 1)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    h.set_profiling(True)
    s0 = h.stats()
    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    torch.cuda.synchronize()
    sampler.begin()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    sampler.end()
    barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    s1 = h.stats()
    h.set_profiling(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n / (ms * 1e-3) / 1e6  # the whole matrix, partitioned over the ranks

    # per kernel class over the timed region (classes "name@level" are grouped by name;
    # "truncate_row@8" -> class "truncate", detail kept per level)
    kern, detail = {}, {}
    for cls, v1 in s1["kernels"].items():
        v0 = s0["kernels"].get(cls, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
        d = {key: v1[key] - v0[key] for key in ("launches", "ms", "flops", "bytes")}
        detail[cls] = d
        base = cls.split("@")[0].replace("_row", "").replace("_col", "")
        agg = kern.setdefault(base, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
        for key in agg:
            agg[key] += d[key]
    launches = s1["launches_total"] - s0["launches_total"]
    dom = max(kern.items(), key=lambda kv: kv[1]["ms"])
    dname, d = dom
    achieved = d["flops"] / (d["ms"] * 1e-3) / 1e12 if d["ms"] > 0 else 0.0
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(dname)
        traffic = tr["bytes_per_launch"] if tr else None
    except Exception:
        traffic = None
    roof = {"kernel": dname, "bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
            "traffic_note": "DRAM bytes of one full-capture launch (largest level) from profiles/ncu_traffic.json",
            "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (no FP64 entry in MEASURED_PEAKS.json)",
            "share_of_step": d["ms"] / (ms * args.steps) if ms > 0 else None,
            "avg_launch_ms": d["ms"] / max(d["launches"], 1)}
    phases = {cls: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                    "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] > 0 else 0.0}
              for cls, v in sorted(kern.items())}

    # end-to-end through the C ABI with host buffers
    e2e = None
    if args.e2e_steps > 0:
        xh = seeded_vector(n, 2)
        bi = xyz.nbytes + tri.nbytes + xh.nbytes
        bo = xh.nbytes
        h.close()
        torch.cuda.synchronize()
        tt, parts = [], []
        for i in range(args.e2e_steps + 1):
            barrier()
            t0 = time.perf_counter()
            g = make()
            ta = time.perf_counter()
            g.recompress(cfg["eps"])
            tb = time.perf_counter()
            yh = g.matvec(xh, 1)
            t1 = time.perf_counter()
            hb = g.stats()["host_build_ms"]
            g.close()
            print("e2e iter %d: build %.1f ms (host %.1f) recompress %.1f ms matvec %.1f ms" %
                  (i, 1e3 * (ta - t0), hb, 1e3 * (tb - ta), 1e3 * (t1 - tb)), file=sys.stderr)
            if i > 0:
                tt.append(t1 - t0)
                parts.append((ta - t0, hb * 1e-3, tb - ta, t1 - tb))
        te = float(np.mean(tt))
        pm = np.mean(np.array(parts), axis=0)
        if world > 1:
            t = torch.tensor([te], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": n / te / 1e6, "unit": "Mdof/s", "h2d_bytes_per_step": int(bi),
               "d2h_bytes_per_step": int(bo), "seconds_per_step": te,
               "breakdown_s": {"build_interp": pm[0], "of_which_host_structure": pm[1], "recompress": pm[2],
                               "matvec": pm[3]}}
        del yh

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
            sec, samp, full = oracle_sample(cfg, args.sample_frac)
            tfull = sec * full / samp
            cpu = {"value": n / tfull / 1e6, "unit": "Mdof/s", "cores": 1, "kind": "oracle",
                   "sample": "full §3.2 oracle pipeline on a seeded %.3g fraction of the admissible blocks "
                             "(%d of %d work units, %.1f s), extrapolated by work units" % (
                                 args.sample_frac, samp, full, sec),
                   "host_cores_available": cpu_cores()}
        line = {"metric": METRIC, "value": value, "unit": "Mdof/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_desc(cfg), "n": n, "kappa": cfg["kappa"], "m": cfg["m"],
                           "leaf": cfg["leaf"], "eps": cfg["eps"], "mode": "FROB_BLOCKREL",
                           "parallelism": ("subtree-shards%d (NCCL)" % world if world > 1 else
                                           "virtual-shards%d (1 GPU)" % args.shards if args.shards > 1 else "single"),
                           "l2": "inputs larger than L2 (%.1f GB resident device data)" % (s1["device_bytes"] / 1e9),
                           "blocks": s1["blocks"], "row_pairs": s1["row_pairs"], "basis_pairs": s1["basis_pairs"]},
                "seconds_per_step": ms * 1e-3,
                "roofline": roof, "cpu_baseline": cpu, "clocks": clocks, "e2e": e2e, "gpu_launches": launches,
                "exchange_bytes_per_step": s1.get("exchange_bytes"),
                "phases": phases,
                "launch_detail_ms_per_step": {c: round(v["ms"] / args.steps, 4) for c, v in sorted(detail.items())}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
