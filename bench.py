#!/usr/bin/env python
"""Benchmark: MTTKRP nnz·R/s and CP-ALS s/iter (fp64) — BASELINE.json metric.

A *step* is one full pass of the hot path on one synthetic
tensor already resident in HBM: splatt_cpd_als_ex = validate, COO->CSF build of every
mode, factor init, `iters` CP-ALS iterations (Hadamard+Cholesky, MTTKRP, solve,
normalise, Gram refresh, fit), finalise.  value = (N_modes * nnz * R * iters) per
second of step time, summed over all ranks' shared work (whole-job throughput).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl reference]

Default workload: c5 (BASELINE.json configs[4]: 4-mode, 150M nonzeros, R=16, 20 iterations),
the largest configuration the metric is stated on ("at 1/2/4/8 B200", BJ:2, :9, :11) that
fits one GPU; c3 (the other one) and c2/c4 via --config.
N>1: one process per GPU.  Under torchrun (WORLD_SIZE set) each rank runs directly;
otherwise `bench.py --gpus N` re-executes itself under torch.distributed.run with N ranks
on 127.0.0.1.  The path is sharded by root slices / equal nonzero ranges
with NCCL all-reduce / all-gather inside the library ("scaling": "strong", fixed tensor).
--impl reference times the CPU oracle (the tier's reference arm) on the host cores.
"""
from __future__ import annotations

import argparse
import contextlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

DEFAULT_CONFIG = "c5"  # BASELINE.json configs[4]: the largest config the metric names at 1/2/4/8 GPUs
METRIC = "MTTKRP nnz·R/s and CP-ALS s/iter (fp64), % HBM roofline"
UNIT = "nnz·R/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def gather_view(st, N, R, t_mttkrp, policy):
    """Rows gathered by the ROOT MTTKRPs (every non-root CSF node: one factor row each) per
    second, against the measured row-gather ceiling (profiles/gather_peak.json)."""
    if policy != "all" or not t_mttkrp:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "gather_peak.json")) as f:
            gp = json.load(f)
    except Exception:
        return None
    rows = sum(s["iters"] * sum(sum(s["csf_nodes"][n][1:N]) for n in range(N)) for s in st)
    rate = rows / t_mttkrp
    row_bytes = 8 * ((R + 3) // 4 * 4)
    peak = gp.get("rows_per_s_by_row_bytes", {}).get(str(row_bytes))
    return {"rows_per_s": rate, "peak_rows_per_s": peak,
            "frac": rate / peak if peak else None, "row_bytes": row_bytes,
            "peak_source": "profiles/gather_peak.json (measured gather microbenchmark)"}


class NvmlClockSampler:
    """NVML sampling (in-process thread) during the timed region: SM clock, max SM clock
    and the clock-event (throttle) reasons, the fields of the recipe's clocks line."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu: int, period_s: float = 0.1):
        self.gpu = gpu
        self.period = period_s
        self.sm, self.mx, self.reasons = [], 0.0, set()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].isdigit() else self.gpu
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            # the max-clock query costs ~3 ms of driver time: once, outside the sampling loop
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
        except Exception:
            return self
        self.stop = threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self.stop.wait(self.period)

    def __exit__(self, *exc):
        if self.ok:
            self.stop.set()
            self.t.join(timeout=5)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": "nvml"}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, period_s: float = 0.2):
        self.gpu = gpu
        self.period_ms = max(100, int(period_s * 1000))
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def algorithmic_units(cfg):
    N = len(cfg["dims"])
    return N * cfg["nnz"] * cfg["rank"] * cfg["iters"]


# Oracle iterations per cpu_baseline sample (about 10-30 s of host work on 16 cores) and per
# reference-arm step (one iteration: each step is a bounded sample of the same workload).
CPU_SAMPLE_ITERS = {"c1": 10, "c2": 10, "c3": 2, "c4": 2, "c4r64": 2, "c5": 2}
REF_SAMPLE_NNZ = 40_000_000


def host_cpu_info():
    """lscpu model / sockets / cores (the oracle's cores are stated)."""
    info = {"logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for ln in out.splitlines():
            if ":" in ln:
                k, v = ln.split(":", 1)
                kv[k.strip()] = v.strip()
        info["model"] = kv.get("Model name")
        for k, name in (("Socket(s)", "sockets"), ("Core(s) per socket", "cores_per_socket"),
                        ("Thread(s) per core", "threads_per_core")):
            if kv.get(k, "").isdigit():
                info[name] = int(kv[k])
    except Exception:
        pass
    info["omp_proc_bind"] = os.environ.get("OMP_PROC_BIND")
    info["omp_num_threads"] = os.environ.get("OMP_NUM_THREADS")
    return info


def _oracle_run(t, cfg, iters):
    import oracle
    t0 = time.perf_counter()
    r = oracle.cpd_als(t.dims, t.ind, t.vals, rank=cfg["rank"], max_iters=iters, tol=0.0,
                       seed=cfg["seed"], timings=True)
    wall = time.perf_counter() - t0
    tm = r["timings"]
    units = len(t.dims) * t.nnz * cfg["rank"] * iters
    return units, tm, wall


def cpu_baseline(t, cfg, iters=None):
    """The oracle as it stands, on the host cores, on a bounded sample of the iterations,
    plus a 1-thread leg on c1 (full run) mirroring the paper's 1-thread column."""
    import oracle
    import synth
    iters = iters or CPU_SAMPLE_ITERS.get(cfg["name"], 2)
    units, tm, wall = _oracle_run(t, cfg, iters)
    step = tm["loop"] + tm["sort"]
    out = {"value": units / step, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
           "sample": f"{cfg['name']} full tensor, {iters} of {cfg['iters']} CP-ALS iterations "
                     f"(+ its per-mode grouping sort); wall {wall:.1f}s",
           "sec_per_iter": tm["loop"] / iters,
           "mttkrp_nnzR_per_s": units / tm["mttkrp"],
           "host": host_cpu_info()}
    nthr = oracle.num_threads()
    try:
        oracle.set_threads(1)
        c1 = dict(synth.config("c1"), name="c1")
        t1 = synth.generate_config("c1")
        u1, tm1, _ = _oracle_run(t1, c1, c1["iters"])
        out["one_thread"] = {"workload": "c1", "iters": c1["iters"],
                             "value": u1 / (tm1["loop"] + tm1["sort"]), "unit": UNIT,
                             "sec_per_iter": tm1["loop"] / c1["iters"]}
    finally:
        oracle.set_threads(nthr)
    return out


def run_reference(args, cfg, t):
    """--impl reference: the CPU oracle (this tier's reference arm), rank 0 only."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    iters = 1
    # Each step is a bounded sample of the workload: one CP-ALS iteration (+ the oracle's
    # per-mode grouping) over the first REF_SAMPLE_NNZ nonzeros (same dims, same generator
    # stream; the full tensor for c1/c2), so that --steps 20 --warmup 5 stays within minutes
    # (c5 in full: ~14 s per step on 16 cores).
    m = min(t.nnz, REF_SAMPLE_NNZ)
    ind = [a[:m] for a in t.ind]
    vals = t.vals[:m]
    units = len(t.dims) * m * cfg["rank"] * iters
    for _ in range(args.warmup):
        oracle.cpd_als(t.dims, ind, vals, rank=cfg["rank"], max_iters=iters, seed=cfg["seed"])
    times = []
    for _ in range(args.steps):
        r = oracle.cpd_als(t.dims, ind, vals, rank=cfg["rank"], max_iters=iters,
                           seed=cfg["seed"], timings=True)
        times.append(r["timings"]["loop"] + r["timings"]["sort"])
    tot = sum(times)
    value = units * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, args.gpus),
        "world_size": world,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(),
                         "kind": "oracle",
                         "sample": (f"{cfg['name']}: first {m} of {t.nnz} nonzeros, {iters} CP-ALS "
                                    "iteration per step (+ per-mode grouping sort)"),
                         "host": host_cpu_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: re-execute under torch.distributed.run with N ranks
    (one process per GPU, rendezvous on 127.0.0.1).  Returns the launcher's exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    log(f"[bench] self-launch: {' '.join(cmd)}")
    return subprocess.call(cmd)


def config_block(cfg, G, policy="all", leaf_tiling="auto"):
    return {"workload": cfg["name"], "dims": list(cfg["dims"]), "nnz": cfg["nnz"],
            "rank": cfg["rank"], "iters": cfg["iters"], "seed": cfg["seed"],
            "csf_policy": policy, "leaf_tiling": leaf_tiling,
            "parallelism": (f"root-mode partitioned x{G} (P1/P2 per mode)" if G > 1 else "single GPU"),
            "l2": "inputs larger than L2 (COO + per-mode CSFs >> 126 MB); no explicit flush"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--iters", type=int, default=None, help="override CP-ALS iterations")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--clocks", default="nvml", choices=["nvml", "smi", "off"],
                    help="clock sampler during the timed region (nvml: in-process thread)")
    ap.add_argument("--clock-period", type=float, default=0.1,
                    help="seconds between clock samples")
    ap.add_argument("--policy", default="all", choices=["all", "one", "two"],
                    help="CSF allocation policy (SPLATT_CSF_*)")
    ap.add_argument("--leaf-tiling", default="auto",
                    help="ROOT MTTKRP leaf tiling above this fraction of L2 (0 = off; default "
                         "auto = the library's: half-L2 tiles in runs of >= 10 iterations)")
    ap.add_argument("--partition", default="auto", choices=["auto", "nnz", "slices"],
                    help="multi-GPU split: per-mode auto, equal nonzero ranges (P2), whole slices (P1)")
    ap.add_argument("--exchange", default="collective", choices=["collective", "peer"],
                    help="multi-GPU factor-row exchange: NCCL all-gather after the solve (default), "
                         "or the solve kernel storing its rows into the peers' matrices over NVLink")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(args))
    if args.impl == "reference" and rank != 0:
        return  # the reference arm runs on rank 0 only; the other ranks exit without work
    # the oracle legs (reference arm, cpu_baseline) spread their OpenMP threads over the
    # host's cores; libgomp reads this when the oracle library loads
    os.environ.setdefault("OMP_PROC_BIND", "spread")

    import synth
    cfg = dict(synth.config(args.config))
    cfg["name"] = args.config
    if args.iters:
        cfg["iters"] = args.iters
    t0 = time.perf_counter()
    t = synth.generate_config(args.config)
    log(f"[bench] generated {args.config}: dims={t.dims} nnz={t.nnz} in "
        f"{time.perf_counter() - t0:.1f}s")

    if args.impl == "reference":
        run_reference(args, cfg, t)
        return

    import torch
    import torch.distributed as dist
    import paper_1812_05961_b200 as sb

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but {torch.cuda.device_count()} "
                         "visible GPUs")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    stream = torch.cuda.Stream(local)
    ctx = sb.Context(local, stream=stream)
    if args.leaf_tiling != "auto":
        ctx.set_leaf_tiling(float(args.leaf_tiling))
    if world > 1:
        ctx.set_comm()
        ctx.set_partition(args.partition)
        ctx.set_exchange(args.exchange)

    N = len(t.dims)
    R, iters = cfg["rank"], cfg["iters"]
    with torch.cuda.stream(stream):
        ind = [torch.from_numpy(a.view(np.int32)).cuda(local) for a in t.ind]
        vals = torch.from_numpy(t.vals).cuda(local)
    torch.cuda.synchronize(local)

    host_call_s = []
    # Caller-owned device outputs, allocated once (a repeated-solve caller's pattern): the
    # timed region holds the library call, not torch allocator traffic.
    dev_out = {"factors": [torch.empty((int(d), R), dtype=torch.float64, device=f"cuda:{local}")
                           for d in t.dims],
               "lam": torch.empty(R, dtype=torch.float64, device=f"cuda:{local}")}

    def step(stats=True):
        t0 = time.perf_counter()
        try:
            r = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=iters, tol=0.0,
                           seed=cfg["seed"], ctx=ctx, stats=stats, policy=args.policy,
                           out=dev_out)
            return {"stats": r["stats"], "fit": r["fit"]}
        finally:
            host_call_s.append(time.perf_counter() - t0)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(local)
    if world > 1:
        dist.barrier()

    runs = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    sampler = {"nvml": NvmlClockSampler, "smi": ClockSampler}.get(args.clocks)
    with (sampler(local, args.clock_period) if sampler else contextlib.nullcontext()) as clk:
        torch.cuda.synchronize(local)
        if world > 1:
            dist.barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            runs.append(step())
        ev1.record(stream)
        torch.cuda.synchronize(local)
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        pin_ind = [torch.from_numpy(a.view(np.int32)).pin_memory() for a in t.ind]
        pin_val = torch.from_numpy(t.vals).pin_memory()
        h_ind = [p.numpy() for p in pin_ind]
        h_val = pin_val.numpy()
        h_out = {"factors": [torch.empty((int(d), R), dtype=torch.float64).pin_memory().numpy()
                             for d in t.dims],
                 "lam": torch.empty(R, dtype=torch.float64).pin_memory().numpy()}
        e_times = []
        for k in range(max(1, args.steps // 2) + 1):
            torch.cuda.synchronize(local)
            a = time.perf_counter()
            r = sb.cpd_als(h_ind, h_val, t.dims, rank=R, max_iters=iters, seed=cfg["seed"],
                           ctx=ctx, out=h_out, policy=args.policy)
            b = time.perf_counter()
            if k > 0:
                e_times.append(b - a)
        emax = max(e_times) if world == 1 else e_times
        et = float(np.mean(e_times))
        if world > 1:
            tt = torch.tensor([et], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            et = float(tt.item())
        h2d = t.nnz * (4 * N + 8)
        d2h = sum(int(d) for d in t.dims) * R * 8 + R * 8
        e2e = {"value": algorithmic_units(cfg) / et, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "sec_per_step": et,
               "note": "public API sb.cpd_als with pinned host COO in, pinned host factors/lambda "
                       "out; H2D/D2H inside the timed call (wall clock around the synchronous call)"}
        del emax

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ------------------------------------------------------------- summarise
    st = [r["stats"] for r in runs]
    t_mttkrp = sum(s["t_mttkrp"] for s in st)
    alg_bytes = sum(s["mttkrp_alg_bytes"] for s in st)
    min_bytes = sum(s["mttkrp_min_bytes"] for s in st)
    launches = sum(s["mttkrp_launches"] for s in st)
    peak, peak_src = peaks()
    achieved = alg_bytes / t_mttkrp / 1e9 if t_mttkrp > 0 else 0.0
    # DRAM bytes and L1TEX wavefront load per ROOT launch from the committed ncu capture of
    # this config (profiles/mttkrp_traffic.json; ncu cannot run inside a timed bench)
    traffic, ncu_rec = None, {}
    tf = os.path.join(ROOT, "profiles", "mttkrp_traffic.json")
    if os.path.exists(tf) and args.policy == "all":
        try:
            with open(tf) as f:
                ncu_rec = json.load(f).get(f"{args.config}:G{world}") or {}
            traffic = ncu_rec.get("dram_bytes_per_launch")
        except Exception:
            traffic, ncu_rec = None, {}
    avg_launch_s = t_mttkrp / max(1, launches)
    units = algorithmic_units(cfg) * args.steps
    value = units / (ms * 1e-3)
    loop = [s["t_loop"] for s in st]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, world, args.policy, args.leaf_tiling),
        "cpals_sec_per_iter": statistics.mean(loop) / iters,
        "mttkrp_nnzR_per_s": N * t.nnz * R * iters * args.steps / t_mttkrp if t_mttkrp else None,
        "breakdown_s_per_step": {k: sum(s[k] for s in st) / args.steps for k in
                                 ("t_build", "t_mttkrp", "t_inverse", "t_ata", "t_norm", "t_fit",
                                  "t_comm", "t_loop", "t_call", "t_host_sync", "t_aux_inverse",
                                  "t_aux_fit")},
        "host_syncs_per_step": sum(s["host_syncs"] for s in st) / args.steps,
        "host_call_ms": 1e3 * statistics.mean(host_call_s[-args.steps:]),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": ((f"mttkrp_root2_kernel<N={N}> ROOT traversal (second generation)"
                                 if N == 4 else f"mttkrp_csf_kernel<N={N}> ROOT traversal")
                                if args.policy == "all"
                                else f"mttkrp_csf_kernel<N={N}> ROOT/INTERNAL/LEAF ({args.policy})"), "peak_source": peak_src,
                     "alg_bytes_per_launch": alg_bytes / max(1, launches),
                     # SURVEY.md §7 hard part 3: the compulsory-traffic view beside the
                     # north star's every-gather-at-HBM count (tree, referenced rows and
                     # output once per launch).
                     "min_bytes_per_launch": min_bytes / max(1, launches),
                     "frac_compulsory": (min_bytes / t_mttkrp / 1e9 / peak) if t_mttkrp else None,
                     # the bound that actually binds: the L1TEX row-gather rate (measured
                     # ceiling of the gather primitive, profiles/gather_peak.json)
                     "gather": gather_view(st, N, R, t_mttkrp, args.policy),
                     "avg_launch_ms": 1e3 * t_mttkrp / max(1, launches),
                     "launches": launches,
                     # three views of the same launches, side by side: algorithmic bytes
                     # (every gather at HBM, the north star's roofline), the physical DRAM
                     # bytes ncu measured, and the L1TEX data-pipe load that actually binds
                     "views": {
                         "alg_frac_of_hbm": achieved / peak,
                         "dram_frac_of_hbm": (traffic / avg_launch_s / 1e9 / peak
                                              if traffic and avg_launch_s > 0 else None),
                         "dram_over_compulsory": (traffic / (min_bytes / max(1, launches))
                                                  if traffic and min_bytes else None),
                         "l2_hit_pct": ncu_rec.get("l2_hit_rate_pct"),
                         "l1tex_wavefront_pct": ncu_rec.get("l1tex_wavefront_pct"),
                         "ncu_source": ncu_rec.get("source"),
                     }},
        "comm": {"backend": "nccl" if world > 1 else None,
                 "nranks": int(st[0].get("nranks", 1)) if st else None,
                 "exchange": ("peer stores from the solve kernel" if st and st[0].get("exchange")
                              else "nccl all-gather") if world > 1 else None},
        "gpu_launches": sum(s["kernel_launches"] for s in st),
        "clocks": clk.summary() if clk else None,
        "e2e": e2e,
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(t, cfg)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
