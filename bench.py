"""Benchmark of the B200 spaQR hot path (BASELINE.json metric, config C3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step = one full spaQR factorization (levels L..1: interior elimination,
interface scaling, threshold-CPQR sparsification, merges) of BASELINE config
3: 2D variable-coefficient upwind convection-diffusion on 256^2 (N=65,536),
L=10, eps=1e-3 (synthetic, seeded: kappa log-uniform [0.1,10], beta U(-50,50)^2).

* value: factorizations/s over the timed steps, device-timed with CUDA events
  on the library's own stream from the end of the (tiny) CSC upload to the
  end of the factorization (inputs resident in HBM), max over ranks.
* e2e: the same metric through the public API `factorize(A_host, tree)` —
  host CSC in, H2D upload and D2H of the result bookkeeping inside the region.
* Multi-GPU: the factorization does not shard under the reference's exact
  processing order, so N GPUs run N independent replicas
  ("scaling": "weak"); no data-path collective.
* roofline: the dominant device kernel family (by device time) against the
  measured fp64 DGEMM peak (cuBLAS via torch, this box) or the measured HBM
  copy bandwidth (MEASURED_PEAKS.json).
* cpu_baseline / --impl reference: the CPU oracle (numpy restatement of the
  reference, oracle/spaqr_oracle.py) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "spaQR factor time + batched-QR fp64 GFLOP/s (% roofline), 2D N=256^2, 1 B200"
UNIT = "factorizations/s"
WORKLOADS = {
    "C1": "C1: 2D upwind conv-diff 64^2 (N=4096), beta=(20,20), L=6, eps=1e-2",
    "C3": "C3: 2D var-coef upwind conv-diff 256^2 (N=65536), L=10, eps=1e-3, scaled sparsification",
    "C4": "C4: 3D upwind conv-diff 32^3 (N=32768), beta=(10,10,10), L=9, eps=1e-2",
    "C5": "C5: 3D var-coef upwind conv-diff 64^3 (N=262144), L=11, eps=1e-2",
    "C2": "C2: batched QR+Q^T apply of 4096 blocks (m~U{32..256}, k~U{16..128}, k<=m) and "
          "batched threshold RRQR of 4096 64x192 blocks at eps 1e-2 and 1e-4",
}
WORKLOAD = WORKLOADS["C3"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def spawn_ranks(args):
    """`--gpus N` without a launcher: re-run this script under torchrun with N
    ranks (one process per GPU, rendezvous on 127.0.0.1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_setup(n):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if os.environ.get("SPQ_BENCH_BACKEND") != "gloo" else "gloo")
        pg = dist
    return rank, world, local, pg


def config_dict(cfg, A, tree, eps, world):
    """The workload description, identical in both arms."""
    d = {"workload": WORKLOADS[cfg], "config": cfg, "N": int(A.ncols), "levels": int(tree.L),
         "eps": eps, "parallelism": f"replicas x{world}" if world > 1 else "single device",
         "l2": "256 MB buffer written between timed steps (L2 flush)"}
    return d


def problem(cfg):
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    A, dims, L, eps, b, tol = make_config(cfg)
    tree = partition_geometric(dims, L)
    return A, tree, eps, b, tol


def csc_bytes(A, tree):
    n = 8 * (A.indptr.size + A.indices.size + A.data.size)
    for c in tree.leaf_clusters():
        n += 8 * (len(c.cols) + len(c.rows if c.rows is not None else c.cols))
    return int(n)


class Clocks:
    """SM clock / throttle-reason sampler over the timed region (rank 0).

    In-process NVML (pynvml) on a sampling thread: `nvidia-smi -lms` -- the
    first implementation -- holds a driver lock for tens of ms per query,
    which showed up as +70..95 ms outlier steps in this host-bound benchmark
    (more samples, more outliers; profiles/r02g).  nvidia-smi remains the
    fallback when pynvml is missing.  Only samples taken inside `with
    clocks:` are summarised; the sampler itself is started before the
    warm-up so its start-up cost is not timed."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, period=0.1):
        self.index = index
        self.period = period
        self.p = None
        self.thread = None
        self.stop = False
        self.samples = []      # (time, sm_mhz, sm_max_mhz, reasons bitmask)
        self.t0 = self.t1 = None
        self.rows = []

    def _visible_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.index < len(ids) and ids[self.index].isdigit():
                return int(ids[self.index])
        return self.index

    def _loop(self, nv, h):
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h) \
                    if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((time.time(), float(sm), float(mx), int(rs)))
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.thread is not None or self.p is not None:
            return self
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self._visible_index())
            self.nv = nv
            self.thread = threading.Thread(target=self._loop, args=(nv, h), daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "500"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __enter__(self):
        self.start()
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        import datetime
        self.t1 = time.time()
        self.rows = []
        if self.thread is not None:
            time.sleep(self.period)
            self.stop = True
            self.thread.join(timeout=2)
            nv = self.nv
            bits = [("hw_slowdown", nv.nvmlClocksThrottleReasonHwSlowdown),
                    ("hw_thermal_slowdown", nv.nvmlClocksThrottleReasonHwThermalSlowdown),
                    ("sw_thermal_slowdown", nv.nvmlClocksThrottleReasonSwThermalSlowdown),
                    ("sw_power_cap", nv.nvmlClocksThrottleReasonSwPowerCap)]
            for ts, sm, mx, rs in self.samples:
                if self.t0 - 0.05 <= ts <= self.t1 + 0.05:
                    self.rows.append([str(sm), str(mx)] + ["Active" if rs & b else "Not Active"
                                                           for _, b in bits])
            return
        if self.p is None:
            return
        time.sleep(0.3)   # let the sampler print the last in-region sample
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                continue
            if self.t0 - 0.05 <= ts <= self.t1 + 0.05:
                self.rows.append(f[1:])

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows),
                "sampler": "nvml" if self.thread is not None else "nvidia-smi"}


def fp64_peak_tflops():
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def reduce_max(values, dist, device="cuda"):
    """Per-rank timings -> elementwise max over ranks (every rank gets it)."""
    if dist is None:
        return [float(v) for v in values]
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t]


def family_line(name, v, steps, peak64, hbm):
    """Per kernel family: device ms, algorithmic work and its roofline fraction
    (flop families against the measured fp64 DGEMM peak, byte movers against
    the measured HBM bandwidth)."""
    d = {"ms_per_step": v["ms"] / steps, "gflop_per_step": v["flops"] / steps / 1e9,
         "launches_per_step": v["launches"] / steps}
    if v["ms"] <= 0:
        return d
    t_roof = 0.0     # roofline time: the slower of fp64 peak and HBM for the family's work
    if v["flops"] > 0:
        ach = v["flops"] / (v["ms"] * 1e-3) / 1e12
        d.update({"achieved_tflops": ach, "frac_fp64_peak": ach / peak64 if peak64 else None})
        if peak64:
            t_roof = max(t_roof, v["flops"] / (peak64 * 1e12))
    if v.get("bytes", 0) > 0:
        ach = v["bytes"] / (v["ms"] * 1e-3) / 1e9
        d.update({"achieved_gbs": ach, "frac_hbm": ach / hbm})
        t_roof = max(t_roof, v["bytes"] / (hbm * 1e9))
    if t_roof > 0:
        d["frac_roofline"] = t_roof / (v["ms"] * 1e-3)
    return d


def flush_l2(buf):
    buf.add_(1.0)


def cpu_baseline(A, tree, eps, budget_s=30.0):
    """One full C3 factorization by the CPU oracle (numpy + threaded BLAS)."""
    from oracle import spaqr_oracle as O
    t0 = time.perf_counter()
    O.factorize(A, tree, eps=eps)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"1 full factorization of the same workload by oracle/spaqr_oracle.py "
                      f"({dt:.1f} s, numpy/OpenBLAS threads={os.cpu_count()})",
            "seconds_per_factorization": dt}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    A, tree, eps, b, tol = problem(args.config)
    from oracle import spaqr_oracle as O
    for _ in range(min(args.warmup, 1)):
        t0 = time.perf_counter()
        O.factorize(A, tree, eps=eps)
        step = time.perf_counter() - t0
    times = []
    budget = 200.0
    for k in range(args.steps):
        t0 = time.perf_counter()
        O.factorize(A, tree, eps=eps)
        times.append(time.perf_counter() - t0)
        if sum(times) > budget:
            break
    T = sum(times)
    v = len(times) / T
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "steps_run": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": config_dict(args.config, A, tree, eps, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                             "sample": f"{len(times)} full factorizations by the CPU oracle"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def run_c2(args, rank, world, local, dist):
    """BASELINE config 2: the isolated batched kernels (one step = batched QR +
    Q^T apply of the 4096 QR blocks, then batched threshold RRQR of the 4096
    RRQR blocks at eps 1e-2 and at 1e-4).  value = algorithmic GFLOP/s of the
    step (SURVEY §8d counts) from device time; e2e = the same through the
    host-buffer C-ABI calls (H2D + D2H inside)."""
    from paper_2010_06807_b200.batched import batched_qr, batched_rrqr, config2_inputs
    if args.impl == "reference":
        if rank != 0:
            return
        from oracle import spaqr_oracle as O
        Bs, Cs, Ms = config2_inputs(n_qr=256, n_rrqr=256)
        fl = c2_flops(Bs, Cs, None)
        t0 = time.perf_counter()
        fl_rr = 0.0
        for B, Cc in zip(Bs, Cs):
            V, tau, R = O.house_qr(B)
            O.wy_apply(V, O.larft(V, tau), Cc, True)
        for eps in (1e-2, 1e-4):
            for M in Ms:
                r = O.rrqr_threshold(M, eps)["rank"]
                fl_rr += 4 * 64 * 192 * r - 2 * r * r * (64 + 192) + 4 * r ** 3 / 3
        dt = time.perf_counter() - t0
        v = (fl + fl_rr) / dt / 1e9
        line = {"metric": "config-2 batched QR+apply / RRQR fp64 GFLOP/s", "value": v,
                "unit": "GFLOP/s", "n_gpus": world, "steps": 1, "warmup": 0,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": {"workload": WORKLOADS["C2"], "config": "C2"},
                "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": os.cpu_count(),
                                 "kind": "port", "sample": "256 QR + 2x256 RRQR blocks"},
                "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    import torch
    torch.cuda.set_device(local)
    Bs, Cs, Ms = config2_inputs()
    peak64 = fp64_peak_tflops()
    fl_qr = c2_flops(Bs, Cs, None)
    for _ in range(max(args.warmup, 0)):
        batched_qr(Bs, Cs)
        for eps in (1e-2, 1e-4):
            batched_rrqr(Ms, eps)
    dev = {"qr": 0.0, "rrqr_1e-2": 0.0, "rrqr_1e-4": 0.0}
    fl = {"qr": fl_qr, "rrqr_1e-2": 0.0, "rrqr_1e-4": 0.0}
    wall = 0.0
    ranks = {}
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    with clocks:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            _, _, ms = batched_qr(Bs, Cs)
            dev["qr"] += ms
            for eps in (1e-2, 1e-4):
                rk, _, ms = batched_rrqr(Ms, eps)
                key = "rrqr_1e-2" if eps == 1e-2 else "rrqr_1e-4"
                dev[key] += ms
                fl[key] = float(sum(4 * 64 * 192 * r - 2 * r * r * (64 + 192) + 4 * r ** 3 / 3
                                    for r in rk))
                ranks[key] = [int(rk.min()), int(np.median(rk)), int(rk.max())]
            wall += time.perf_counter() - t0
    torch.cuda.synchronize()
    T = sum(dev.values())
    T, wall = reduce_max([T, wall], dist)
    if rank != 0:
        return
    total = (fl["qr"] + fl["rrqr_1e-2"] + fl["rrqr_1e-4"]) * args.steps * world
    value = total / (T * 1e-3) / 1e9
    kern = {}
    for k in dev:
        ach = fl[k] * args.steps / (dev[k] * 1e-3) / 1e12 if dev[k] else 0.0
        kern[k] = {"ms_per_step": dev[k] / args.steps, "gflop_per_step": fl[k] / 1e9,
                   "achieved_tflops": ach, "frac_fp64_peak": ach / peak64}
    dom = max(dev, key=dev.get)
    in_bytes = 8 * (sum(b.size for b in Bs) + 2 * sum(c.size for c in Cs) + 2 * Ms.size)
    line = {"metric": "config-2 batched QR+apply / RRQR fp64 GFLOP/s", "value": value,
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": T / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS["C2"], "config": "C2", "n_qr": len(Bs),
                       "n_rrqr": int(Ms.shape[0]),
                       "l2": "inputs 0.75 GB per step > 126 MB L2"},
            "kernels": kern, "ranks": ranks,
            "roofline": {"bound": "fp64", "achieved": kern[dom]["achieved_tflops"],
                         "peak": peak64, "unit": "TFLOP/s",
                         "frac": kern[dom]["frac_fp64_peak"], "traffic": None,
                         "kernel_family": dom,
                         "peak_source": "measured cuBLAS DGEMM 8192^3 on this box"},
            "e2e": {"value": total / wall / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(in_bytes), "d2h_bytes_per_step": int(in_bytes // 2)},
            "fp64_peak_tflops_measured": peak64, "clocks": clocks.summary()}
    print(json.dumps(line), flush=True)


def c2_flops(Bs, Cs, _):
    f = 0.0
    for b, c in zip(Bs, Cs):
        m, k = b.shape
        n = c.shape[1]
        f += 2 * m * k * k - 2 * k ** 3 / 3 + 4 * m * n * k - n * k * k
    return f


def main():
    args = parse()
    spawn_ranks(args)
    rank, world, local, dist = dist_setup(args.gpus)
    if args.config == "C2":
        return run_c2(args, rank, world, local, dist)
    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    import torch
    torch.cuda.set_device(local)
    from paper_2010_06807_b200 import factor as FZ
    A, tree, eps, b, tol = problem(args.config)
    peak64 = fp64_peak_tflops()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    l2buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2

    clocks = Clocks(local).start()
    for _ in range(max(args.warmup, 0)):
        FZ.factorize(A, tree, eps=eps, device=local)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    dev_ms, e2e_ms = [], []
    spec_retries = 0
    agg = {}
    launches = 0
    barrier()
    if os.environ.get("SPQ_BENCH_NOGC") == "1":       # diagnostics: are the outliers collector pauses?
        import gc
        gc.collect()
        gc.disable()
    with clocks:
        for _ in range(args.steps):
            flush_l2(l2buf)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            F = FZ.factorize(A, tree, eps=eps, device=local, _marks=True)
            e1.record()
            torch.cuda.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
            dev_ms.append(F.device_ms)
            spec_retries += int(getattr(F, "spec_retries", 0))
            tm = F.device_timings()
            host = tm.pop("host")
            launches += int(host.get("kernels", 0))
            for fam, v in tm.items():
                a = agg.setdefault(fam, {"ms": 0.0, "flops": 0.0, "launches": 0, "bytes": 0.0})
                for key in ("ms", "flops", "launches", "bytes"):
                    a[key] += v.get(key, 0)
            del F
    barrier()
    # solve phase (reported beside the metric): device GMRES on one factorization
    solve = None
    if b is not None:
        from paper_2010_06807_b200.solve import gmres
        F = FZ.factorize(A, tree, eps=eps, device=local)
        gmres(A, b, F, tol=tol)                       # warm (chain graphs, CSR upload)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = gmres(A, b, F, tol=tol)
        ts = time.perf_counter() - t0
        solve = {"gmres_s": ts, "iterations": int(rep.iterations),
                 "final_residual": float(rep.final_residual), "tol": tol,
                 "where": "device (spq_gmres: chains + CSR SpMV + MGS in HBM)"}
        # roofline of the chain applications (row (e)): one application reads the
        # stored payload (V, T, R_ss, R_sn of every record) once -- algorithmic
        # bytes = 8 * payload_scalars -- timed on the library stream
        y = np.random.default_rng(0).standard_normal(A.ncols)
        chain = {}
        for fn in ("apply_qt", "solve_w"):
            getattr(F, fn)(y)
            F._ctx.call("spq_reset_timings")
            reps = 10
            for _ in range(reps):
                getattr(F, fn)(y)
            ms = F.device_timings()["chain"]["ms"] / reps
            gb = 8.0 * int(F.payload_scalars) / 1e9
            chain[fn] = {"device_ms": ms, "payload_gb": gb, "achieved_gbs": gb / (ms * 1e-3),
                         "frac_hbm": gb / (ms * 1e-3) / hbm}
        solve["chain"] = chain
        del F
    T = float(np.sum(dev_ms))
    Te = float(np.sum(e2e_ms))
    T, Te = reduce_max([T, Te], dist)
    if rank != 0:
        return
    units = world * args.steps
    value = units / (T / 1e3)
    e2e = units / (Te / 1e3)
    # roofline of the dominant family
    fams = {k: v for k, v in agg.items() if v["ms"] > 0}
    dom = max(fams, key=lambda k: fams[k]["ms"]) if fams else None
    roof = None
    if dom is not None:
        d = fams[dom]
        t_f = d["flops"] / (peak64 * 1e12) if (peak64 and d["flops"]) else 0.0
        t_b = d.get("bytes", 0.0) / (hbm * 1e9)
        if dom in ("copy", "flags", "chain") or t_b > t_f:
            ach = d["bytes"] / (d["ms"] * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": ach / hbm, "traffic": None, "kernel_family": dom,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        else:
            ach = d["flops"] / (d["ms"] * 1e-3) / 1e12
            roof = {"bound": "tensor" if dom == "wy" else "fp64", "achieved": ach,
                    "peak": peak64, "unit": "TFLOP/s", "frac": ach / peak64, "traffic": None,
                    "kernel_family": dom,
                    "peak_source": "measured cuBLAS DGEMM 8192^3 (torch.matmul fp64) on this box"}
    if roof is not None:
        # DRAM bytes per launch of the same family from the committed ncu launch list
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
            ft = tr["families"][dom]
            roof["traffic"] = ft["dram_bytes_per_launch"]
            roof["traffic_unit"] = "bytes/launch (dram read+write)"
            roof["traffic_source"] = "profiles/ncu_traffic.json (" + tr["source"] + ")"
            # algorithmic bytes per launch of the family, for comparison with traffic
            if d.get("launches"):
                roof["algorithmic_bytes_per_launch"] = d.get("bytes", 0.0) / d["launches"]
        except (OSError, KeyError, ValueError):
            pass
    qr_fams = [f for f in ("qr", "wy", "trsm", "cpqr") if f in fams]
    qflops = sum(fams[f]["flops"] for f in qr_fams)
    qms = sum(fams[f]["ms"] for f in qr_fams)
    bqr = qflops / (qms * 1e-3) / 1e9 if qms else 0.0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": T / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config, A, tree, eps, world),
        "timed_region": "device: mark before spq_load (CSC upload, equilibration, block scatter "
                        "included) -> end of spq_finish; e2e: the public factorize(A_host, tree) "
                        "call",
        "spec_retries": spec_retries,
        "factor_time_s": T / args.steps / 1e3,
        "step_ms": [round(float(x), 3) for x in dev_ms],
        "batched_qr_gflops": bqr,
        "batched_qr_frac_of_fp64_peak": bqr / (peak64 * 1e3) if peak64 else None,
        "fp64_peak_tflops_measured": peak64,
        "kernels": {k: family_line(k, v, args.steps, peak64, hbm) for k, v in fams.items()},
        "roofline": roof,
        "solve": solve,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": csc_bytes(A, tree),
                "d2h_bytes_per_step": 8 * int(A.ncols)},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline and args.config in ("C1", "C3"):
        line["cpu_baseline"] = cpu_baseline(A, tree, eps)
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
