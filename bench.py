#!/usr/bin/env python
"""Benchmark of the B200 DH^2 hot path (BASELINE.json metric) on the largest BASELINE workload that
runs on one GPU: configs[3] = C4 (sphere, n = 131072, kappa = 64, m = 5, k = 125, eps = 1e-6; the
paper's own 131,072-triangle timing case), on the memory-lean chunked plan.

A step = one pass of the whole hot path of SURVEY §8(a) over the resident input:
device set-up (quadrature, grids, transfer factors E; leaf V and S_b are generated inside the
recompression on the lean plan), the hybrid recompression (basis weights, block weights, total
weights and truncation, the column pass by adjoint symmetry, projection) and one far-field matvec
of the recompressed matrix.  value = n / device time per step (Mdof/s); e2e = the same through the
C ABI from HOST buffers (mesh in, x in, y out), host structure build and all copies included.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

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


def fp64_peak():
    """Measured FP64 tensor-core (DMMA m8n8k4) throughput on this pool's B200, sustained for 4 s
    (tools/fp64_peak.py -> profiles/r02_fp64_peak.json; MEASURED_PEAKS.json has no FP64 entry)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")))
        return d["dmma_m8n8k4"]["sustained_tflops"], ("measured: DMMA m8n8k4 sustained %.2f TF/s (DFMA %.2f, cuBLAS ZGEMM "
                                                      "%.2f), profiles/r02_fp64_peak.json" % (
                                                          d["dmma_m8n8k4"]["sustained_tflops"], d["dfma"]["sustained_tflops"],
                                                          d["cublas_zgemm"]["sustained_tflops"]))
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (no measurement found)"


def hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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
# The oracle (oracle/, as it stands) on the host cores: one process per core, each with one BLAS
# thread, forked after the oracle's host structure is built once (copy-on-write); process i runs
# the full §3.2 pipeline on its own seeded sample of the workload -- the sub-matrix made of a
# random fraction of the admissible blocks, pairs re-closed over them.  A "step" is one such batch
# over all cores; its wall time is measured, nothing is extrapolated: value = the work the batch
# did, expressed in DoF of the full matrix (n x sample work units / full work units; units = basis
# + row + column pairs + blocks), per second of wall time.
_ORC = {}


def _units(s):
    return (sum(len(p) for p in s.basis_pairs) + sum(len(p) for p in s.row_pairs)
            + sum(len(p) for p in s.col_pairs) + len(s.blocks))


def _oracle_worker(args):
    import copy
    from oracle.recompress import Recompression
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)  # one BLAS thread per process
    seed, frac = args
    st0, eps = _ORC["st"], _ORC["eps"]
    st = copy.copy(st0)
    rng = np.random.default_rng(seed)
    keep = np.sort(rng.choice(len(st0.blocks), size=max(1, int(frac * len(st0.blocks))), replace=False))
    st.blocks = st0.blocks[keep]
    st._build_pairs()
    t0 = time.perf_counter()
    Recompression(st, eps).run()
    return _units(st), time.perf_counter() - t0


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class OracleBench:
    """Builds the oracle structure once, then times batches of parallel samples."""

    def __init__(self, cfg, frac):
        for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[v] = "1"
        from oracle.structure import DH2Structure
        xyz, tri = mesh_for(cfg)
        t0 = time.perf_counter()
        st = DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
        self.structure_s = time.perf_counter() - t0
        _ORC["st"], _ORC["eps"] = st, cfg["eps"]
        self.full = _units(st)
        self.n = int(tri.shape[0])
        self.frac = frac
        self.cores = cpu_cores()
        import multiprocessing as mp
        self.pool = mp.get_context("fork").Pool(self.cores)

    def batch(self, step):
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_worker, [(1000 * step + i, self.frac) for i in range(self.cores)])
        wall = time.perf_counter() - t0
        work = sum(u for u, _ in res)
        return wall, work, [t for _, t in res]

    def close(self):
        self.pool.terminate()

    def describe(self, work, wall):
        return ("oracle/ (numpy/scipy, as it stands) on %d host processes x 1 BLAS thread (%s): each runs the full "
                "§3.2 pipeline on its own seeded sample of %.2g of the admissible blocks (pairs re-closed); the batch "
                "did %d of the %d work units of the full matrix in %.1f s wall; value = n x done/full units / wall"
                % (self.cores, cpu_model(), self.frac, work, self.full, wall))


def default_frac(cfg):
    # ~5-15 s of CPU work per process for every configuration
    return {"C1": 0.5, "C2": 0.02, "C3": 0.003}.get(cfg["name"], 0.0005)


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    ob = OracleBench(cfg, args.sample_frac or default_frac(cfg))
    walls, works = [], []
    for i in range(args.warmup + args.steps):
        wall, work, _ = ob.batch(i)
        if i >= args.warmup:
            walls.append(wall)
            works.append(work)
    ob.close()
    wall = float(np.mean(walls))
    val = ob.n * float(np.mean(works)) / ob.full / wall / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "Mdof/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "n": ob.n},
            "cpu_baseline": {"value": val, "unit": "Mdof/s", "cores": ob.cores, "kind": "oracle",
                             "sample": ob.describe(int(np.mean(works)), wall),
                             "oracle_structure_s": ob.structure_s},
            "e2e": {"value": val, "unit": "Mdof/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-nearfield", dest="nearfield", action="store_false",
                    help="skip the (untimed-in-value) nearfield assembly + matvec measurement")
    ap.add_argument("--sample-frac", type=float, default=None)
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
    peak, peak_src = fp64_peak()
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        tr = tr.get(cfg["name"], {}).get(dname) if cfg["name"] in tr else None
        traffic = tr["bytes_per_launch"] if tr else None
    except Exception:
        traffic = None
    roof = {"kernel": dname, "bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic,
            "traffic_note": "DRAM bytes per launch of this class from an ncu --set full capture (profiles/ncu_traffic.json)",
            "peak_source": peak_src,
            "flops_model": "algorithmic flops of the executed work per DESIGN §8 (Kronecker E, k_new-dependent SVD model "
                           "C_svd = 10), summed over the class's launches in the timed steps",
            "share_of_step": d["ms"] / (ms * args.steps) if ms > 0 else None,
            "avg_launch_ms": d["ms"] / max(d["launches"], 1)}
    # the HBM-bound passes: leaf V / S_b writes and the compressed matvec's reads
    hbm, hbm_src = hbm_peak()
    st1 = h.storage(1)
    mv_bytes = 2.0 * st1["row_basis_bytes"] + st1["coupling_bytes"] + 16.0 * 4 * n  # Q/F read twice (fwd + bwd), S~, x/y
    hb = {}
    for cls in ("setup_leafV", "setup_S", "matvec"):
        v = kern.get(cls)
        if not v or v["ms"] <= 0:
            continue
        by = v["bytes"] if cls != "matvec" else mv_bytes * args.steps
        hb[cls] = {"GBps": by / (v["ms"] * 1e-3) / 1e9, "frac_of_hbm": by / (v["ms"] * 1e-3) / 1e9 / hbm,
                   "bytes_per_step": by / args.steps}
    roof["hbm_passes"] = {"peak_GBps": hbm, "peak_source": hbm_src, "passes": hb}
    phases = {cls: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                    "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] > 0 else 0.0}
              for cls, v in sorted(kern.items())}

    # NEXT-4 (not part of `value`): nearfield assembly (Sauter-Schwab / Duffy-Gauss, FP64 ALU bound)
    # and the nearfield matvec (every stored coefficient read once, HBM bound), timed by the library's
    # CUDA events on the bench stream
    near = None
    if args.nearfield:
        try:
            h.set_profiling(True)
            k0 = h.stats()["kernels"]
            h.nearfield_assemble()
            for _ in range(3):
                h.matvec_device(x.data_ptr(), y.data_ptr(), 1, add_near=True)
            torch.cuda.synchronize()
            s2 = h.stats()
            h.set_profiling(False)
            kd = lambda c, f: s2["kernels"].get(c, {}).get(f, 0.0) - k0.get(c, {}).get(f, 0.0)  # noqa: E731
            nf = s2["nearfield"]
            a_ms, m_ms = kd("nearfield", "ms"), kd("matvec_near", "ms") / 3
            gbps = 16.0 * nf["values"] / (m_ms * 1e-3) / 1e9 if m_ms > 0 else 0.0
            near = {"assemble_ms": a_ms, "blocks": nf["blocks"], "values": nf["values"],
                    "touching_entries": nf["touching_entries"], "kernel_evals": nf["kernel_evals"],
                    "gevals_per_s": nf["kernel_evals"] / (a_ms * 1e-3) / 1e9 if a_ms > 0 else 0.0,
                    "matvec_near_ms": m_ms, "matvec_near_GBps": gbps, "matvec_near_frac_of_hbm": gbps / hbm,
                    "note": "NEXT-4, outside the timed step; nq_singular 5, nq_regular 3 (P:1486-1492)"}
        except Exception as e:  # (e.g. device memory on the largest configs)
            near = {"unavailable": str(e).splitlines()[0]}

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
            ob = OracleBench(cfg, args.sample_frac or default_frac(cfg))
            wall, work, per = ob.batch(0)
            ob.close()
            cpu = {"value": n * work / ob.full / wall / 1e6, "unit": "Mdof/s", "cores": ob.cores, "kind": "oracle",
                   "sample": ob.describe(work, wall), "oracle_structure_s": ob.structure_s}
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
                "phases": phases, "nearfield": near,
                "launch_detail_ms_per_step": {c: round(v["ms"] / args.steps, 4) for c, v in sorted(detail.items())}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
