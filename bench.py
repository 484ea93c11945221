#!/usr/bin/env python
"""Benchmark of the Exp-ParaDiag hot path (BASELINE.json metric: space-time
DOF-iterations/s per sweep; achieved HBM GB/s vs B200 peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl reference]

A step is one Exp-ParaDiag sweep of the whole hot path on the resident c5 workload
(BASELINE.json:11; the largest config, it fits one GPU): stage 3 (N-hat = V N(V u-hat) for
every slice), then the fused residual + ||r||^2 + alpha-circulant preconditioner + update
(stages 1, 2), the norm reduction and the device->host read of the residual norm that the
convergence test needs.  K steps are timed with CUDA events on the plan's stream between
barrier + synchronize, max over ranks.  Inputs (8.6 GB per space-time array) exceed the
126 MB L2, so no flush is needed.

--impl reference times the CPU oracle (oracle/, naive long-double sums) on host cores, on
a bounded sample of the same workload.

N > 1 (torchrun): one c5 problem distributed over the ranks (SURVEY §8e, strong scaling):
mode slabs for the fused time-local kernel, time slabs for stage 3, two NCCL all-to-alls
and one allreduce per sweep.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL prints its version banner to stdout at communicator init (NCCL_DEBUG unset / VERSION):
# keep stdout to the one JSON line
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"

# fp64 FMA throughput of this pool's B200 (not in MEASURED_PEAKS.json): a DFMA loop measured
# 34.19 TFLOP/s (profiles/r01_probe_fp64_hbm.txt, tools/probe_fp64.cu); nominal 148 SMs x 64
# DFMA/clk x 2 x 1.965 GHz = 37.2 TFLOP/s
FP64_PEAK_TFLOPS = 34.19


def k1_kernel(cfg, lay) -> str:
    """The K1 kernel the library launches for this plan (csrc/k_time.cuh use_wp / use_ring): the
    warp-per-pair kernel for Nt = 256 Picard sweeps, else the ring
    when the mode slab holds whole tiles, at Nt = 128 / 256 always and at Nt = 16 / 32 / 64
    with at least 16 tiles per SM, unless EXPD_K1V picks a variant; else the TMA-fed kernel."""
    tile = {16: 64, 32: 64, 64: 32, 128: 16, 256: 8}.get(cfg.nt)
    npairs = lay["mode_len"] // 2
    if not tile or npairs % tile:
        return "k_time_tma"
    v = os.environ.get("EXPD_K1V")
    if v in ("2562", "1282", "2561", "5123"):
        return "k_time_ring" if v == "5123" else "k_time_tma"
    # the warp-per-pair kernel: Nt = 256 Picard sweeps (ETD1 / ETD2 / IF; csrc/k_time.cuh use_wp)
    if cfg.nt == 256 and cfg.q and cfg.scheme in (0, 1, 2) and not getattr(cfg, "is_complex", False):
        return "k_time_wp"
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count if torch.cuda.is_available() else 148
    return "k_time_ring" if cfg.nt >= 128 or npairs // tile >= 16 * sms else "k_time_tma"


def dst_flops_per_line_pair(M: int) -> float:
    """Algorithmic fp64 flops of one DST-I transform of two real lines of length M-1
    ("4 DST-I via half-length complex FFTs at ~25-30 flop/point/axis"): the
    split-radix count of the complex FFT of length M, 4 M log2 M - 6 M, plus the sinft
    pre-processing, Hermitian unpack and prefix sum, 12 flops per complex point:
    (4 log2 M + 6) M, i.e. 25 flops per real point per axis at M = 2048."""
    import math

    return (4.0 * math.log2(M) + 6.0) * M


BYTES_PER_DOF = {  # algorithmic fp64 bytes per space-time dof
    "k1_linear": 16,      # read U-hat, write U-hat
    "k1_nonlinear": 24,   # read U-hat, read N-hat, write U-hat
    "k1_complex": 32,     # complex dof (NEXT-4): read U-hat (re, im), write U-hat (re, im)
    "stage3": 16,         # read U-hat slice, write N-hat slice
}


def workload_label(cfg) -> str:
    if getattr(cfg, "is_complex", False):
        scheme = "BDF2" if cfg.scheme == 3 else "exp. Euler"
        return (f"{cfg.name}: {cfg.dim}D n={cfg.n} Nt={cfg.nt} complex a={cfg.a}+{cfg.a_im}i c={cfg.c}+{cfg.c_im}i "
                f"{scheme} fixed-point sweep (Schroedinger, PAPER.md:983/1064; NEXT-4)")
    src = {"c1": ":7", "c2": ":8", "c3": ":9", "c4": ":10", "c5": ":11"}.get(cfg.name)
    return (f"{cfg.name}: {cfg.dim}D n={cfg.n} Nt={cfg.nt} "
            f"{ {0: 'exp. Euler' if not cfg.q else 'ETD1', 1: 'ETD2', 2: 'IF/IMEX', 3: 'BDF2'}[cfg.scheme] } "
            f"{'Picard' if cfg.q else 'fixed-point'} sweep" + (f" (BASELINE.json{src})" if src else ""))


def oracle_dsts_per_slice(cfg) -> float:
    """Real-DST-equivalent transforms per time slice in one oracle sweep: residual (A = V E V:
    2; ETD adds the Phi products: 2 each), Step (b) (DST + IDST of the real and imaginary
    parts of the DFT'd slice: 4).  A complex DST is two real ones."""
    if getattr(cfg, "is_complex", False):
        return 8.0
    res = 2.0 + (2.0 if cfg.q and cfg.scheme == 0 else 0.0) + (4.0 if cfg.q and cfg.scheme == 1 else 0.0)
    return res + 4.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--dist1", action="store_true",
                    help="N = 1: run the distributed schedule (1-rank NCCL communicator) instead")
    ap.add_argument("--solver", default="sweep", choices=["sweep", "gmres"],
                    help="sweep: one fixed-point / Picard sweep per step; gmres: one Arnoldi step of "
                         "left-preconditioned GMRES per step (linear configs, e.g. c4; SURVEY §8(d.3))")
    ap.add_argument("--peer", action="store_true",
                    help="N > 1, nonlinear: stage 3 loads / stores its rows through peer memory (CUDA IPC) "
                         "instead of the NCCL all-to-alls (Plan.enable_peer_stores)")
    ap.add_argument("--launch-check", action="store_true",
                    help="only check the multi-rank launch (gloo without a GPU): ranks, world size, one allreduce")
    return ap.parse_args()


def free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args) -> int:
    """--gpus N > 1 without a torchrun environment: start N ranks of this script on this node
    (one process per GPU, rendezvous on 127.0.0.1) and return their exit status."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def launch_check(args) -> int:
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if ws > 1:
        dist.init_process_group(backend, init_method="env://")
    dev = torch.device(f"cuda:{local}") if backend == "nccl" else torch.device("cpu")
    t = torch.ones(1, device=dev)
    if ws > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": ws, "backend": backend if ws > 1 else "none",
                          "allreduce_sum": float(t.item()), "world_size_ok": ws == args.gpus}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [x.strip() for x in l.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# CPU oracle baseline (oracle/ as it stands; rank 0, N = 1 only)
# ------------------------------------------------------------------------------------------
REF_ROWS = 2048  # rows per CPU-baseline sample (about one whole x-axis pass of a c5 slice)


def oracle_sample_step(cfg, u_rows):
    """One bounded sample of the oracle's sweep: the x-axis DST-I (plain O(n) long-double
    sums per output; the sine table is built once per n) of REF_ROWS rows of a slice.  The
    oracle's sweep applies oracle_dsts_per_slice(cfg) DSTs per time slice, each dim axis passes
    over the slice's n^{dim-1} rows, plus O(Nt) DFT sums per point (< 3 % of its work at c5):
    one sample is REF_ROWS / (dsts dim n^{dim-1} Nt) of a sweep, i.e. that fraction of N_st
    DOF-iterations."""
    import oracle

    oracle.dst_x_rows(oracle.spec(cfg), u_rows)
    rows_per_slice = cfg.n ** (cfg.dim - 1)
    return cfg.nst * u_rows.shape[0] / (oracle_dsts_per_slice(cfg) * cfg.dim * rows_per_slice * cfg.nt)


def oracle_sweep(cfg):
    """One WHOLE oracle sweep (orc_residual + orc_precond: stages 1 and 2 with the nonlinear
    terms, exactly what an oracle Picard / fixed-point iteration computes per sweep) on a
    seeded state; returns (DOF-iter/s, seconds)."""
    import oracle
    import synth

    s = oracle.spec(cfg)
    u0 = synth.initial_condition(cfg)
    U = synth.random_spacetime(cfg, seed=1, scale=0.3)
    t0 = time.perf_counter()
    R, _ = oracle.residual(s, u0, U)
    oracle.precond(s, R)
    dt = time.perf_counter() - t0
    return cfg.nst / dt, dt


def host_cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(cfg, sweep_cfgs=("c2", "c3")):
    """The oracle as it stands on this host's cores (rank 0, N = 1): whole oracle sweeps of
    the configs the oracle finishes in seconds (c2, c3), plus the bounded sample of the
    benchmarked config (a scaled addendum: a whole c5 oracle sweep takes minutes)."""
    import numpy as np

    import oracle
    import synth

    oracle.build()
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    sweeps = {}
    for name in sweep_cfgs:
        rate, sec = oracle_sweep(synth.CONFIGS[name])
        sweeps[name] = {"value": rate, "unit": "DOF-iter/s", "seconds": sec,
                        "workload": workload_label(synth.CONFIGS[name])}
    u = np.random.default_rng(0).standard_normal((REF_ROWS, cfg.n))
    oracle_sample_step(cfg, u)  # warm-up (library load, OpenMP pool, sine table)
    t0 = time.perf_counter()
    dofs, done = 0.0, 0
    while done < 3 or time.perf_counter() - t0 < 5.0:
        dofs += oracle_sample_step(cfg, u)
        done += 1
    dt = time.perf_counter() - t0
    head = sweep_cfgs[-1]
    return {"value": sweeps[head]["value"], "unit": "DOF-iter/s", "cores": int(os.environ["OMP_NUM_THREADS"]),
            "cpu_model": host_cpu_model(), "kind": "oracle",
            "sample": f"one whole oracle sweep (orc_residual + orc_precond, long double, naive O(n) sine and O(Nt) "
                      f"DFT sums) of {head} ({sweeps[head]['seconds']:.1f} s); c2 and the {cfg.name} sample below",
            "sweeps": sweeps,
            f"{cfg.name}_sample": {"value": dofs / dt, "unit": "DOF-iter/s", "seconds": dt,
                                   "sample": f"{done} x oracle x-axis DST-I of {REF_ROWS} rows of a {cfg.name} slice = "
                                             f"{REF_ROWS}/({oracle_dsts_per_slice(cfg):.0f} dim n^(dim-1) Nt) of an "
                                             f"oracle sweep each (scaled by that work ratio)"}}


def run_reference(args):
    import synth

    ws, rank, local = dist_env()
    cfg = synth.CONFIGS[args.config]
    if rank != 0:
        return 0
    import numpy as np

    import oracle

    cores = os.cpu_count() or 1
    if ws > 1:  # torchrun pins OMP_NUM_THREADS=1 per rank; rank 0 alone runs the oracle here
        os.environ["OMP_NUM_THREADS"] = str(cores)
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    oracle.build()
    u = np.random.default_rng(0).standard_normal((REF_ROWS, cfg.n))
    for _ in range(args.warmup):
        oracle_sample_step(cfg, u)
    t0 = time.perf_counter()
    dofs = 0.0
    for _ in range(args.steps):
        dofs += oracle_sample_step(cfg, u)
    dt = time.perf_counter() - t0
    value = dofs / dt
    line = {
        "impl": "reference", "metric": "space-time DOF-iterations/s per Exp-ParaDiag sweep", "value": value,
        "unit": "DOF-iter/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / max(args.steps, 1), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f80 (long double accumulation)", "data": "synthetic",
        "config": {"workload": workload_label(cfg)},
        "cpu_baseline": {"value": value, "unit": "DOF-iter/s", "cores": int(os.environ["OMP_NUM_THREADS"]),
                         "kind": "oracle",
                         "cpu_model": host_cpu_model(),
                         "sample": f"each step: oracle x-axis DST-I of {REF_ROWS} rows of a {cfg.name} slice = "
                                   f"{REF_ROWS}/({oracle_dsts_per_slice(cfg):.0f} dim n^(dim-1) Nt) of an oracle "
                                   f"sweep (scaled by that work ratio)"},
        "e2e": {"value": value, "unit": "DOF-iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# the GPU path
# ------------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2603_04350_b200 import Comm, Plan, Problem
    from paper_2603_04350_b200 import build as pbuild

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if rank == 0:
        pbuild.build()
    if ws > 1:
        dist.barrier()

    cfg = synth.CONFIGS[args.config]
    prob = Problem.from_config(cfg)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    comm = None
    if ws > 1 or args.dist1:
        saved = os.dup(1)  # NCCL's init banner goes to stdout: keep stdout to the JSON line
        os.dup2(2, 1)
        try:
            comm = Comm(rank, ws, local)
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    plan = Plan(prob, device=local, stream=stream, comm=comm)
    peer = bool(args.peer and ws > 1 and cfg.q)
    if peer:
        plan.enable_peer_stores()
    lay = plan.layout
    u0 = torch.from_numpy(synth.initial_condition(cfg)).to(dev)
    plan.load_state(u0, None)
    plan.set_profiling(True)
    nl = len(cfg.q) > 0
    cx = cfg.is_complex
    esz = 16 if cx else 8  # bytes per state entry (complex128 / float64)

    def step():
        plan.sweep()
        return plan.sweep_norm2()  # convergence-test scalar (device -> host, syncs)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    ev0.record(stream)
    ms_nl, ms_k1, norms, passes = [], [], [], []
    for _ in range(args.steps):
        norms.append(step())
        a, b = plan.sweep_stage_ms()
        ms_nl.append(a)
        ms_k1.append(b)

    ev1.record(stream)
    torch.cuda.synchronize(dev)
    ck = clocks.stop()
    if nl and comm is None and cfg.dim == 2:
        # stage-3 families: the same captured sweep with an event between every pass (kept
        # out of the timed region: ~50 extra graph nodes cost ~1 % of a sweep)
        plan.set_profiling(2)
        for _ in range(max(3, min(args.steps, 10))):
            step()
            passes.append(plan.sweep_pass_ms())
        plan.set_profiling(1)
    ms = ev0.elapsed_time(ev1)
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    ms_step = ms / args.steps
    value = cfg.nst * args.steps / (ms * 1e-3)  # one problem over all ranks (strong scaling)

    pk = peaks()
    hbm_peak = pk["hbm_gbs"] if pk else 6650.0
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if pk else "fallback (B200_PROFILING.md)"
    # this rank's share: K1 on its mode slab (nt x mode_len padded entries, of which the
    # n^dim real modes are counted), stage 3 on its time slab
    share = lay["mode_len"] / lay["npad"]
    k1_bytes = BYTES_PER_DOF["k1_complex" if cx else ("k1_nonlinear" if nl else "k1_linear")] * cfg.nst * share
    s3_slices = (cfg.nt - 1) if ws == 1 else lay["nt_local"]
    s3_bytes = BYTES_PER_DOF["stage3"] * cfg.N * s3_slices if nl else 0
    k1_ms = statistics.mean(ms_k1)
    s3_ms = statistics.mean(ms_nl) if nl else 0.0
    k1_gbs = k1_bytes / (k1_ms * 1e-3) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = prof.get(f"{cfg.name}:k1", None)
    except Exception:
        pass
    try:
        k1_ncu = (json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get("counters") or {}).get(
            f"{cfg.name}:k1")
    except Exception:
        k1_ncu = None
    k1_roof = {"bound": "hbm", "kernel": f"{k1_kernel(cfg, lay)} (K1: residual + ||r||^2 + alpha-circulant "
                                        "preconditioner + update, one HBM pass)", "ncu": k1_ncu,
               "achieved": k1_gbs, "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
               "frac": k1_gbs / hbm_peak, "traffic": traffic,
               "algorithmic_bytes_per_launch": k1_bytes, "launch_ms": k1_ms, "launches_per_step": 1}
    kernels = {"k1": k1_roof, "stage3_ms": s3_ms,
               "stage3_gbs": (s3_bytes / (s3_ms * 1e-3) / 1e9) if s3_ms > 0 else None}
    # north_star's quantity: "achieved fraction of the HBM roofline (bytes moved per iteration
    # over peak bandwidth)" -- the whole sweep's algorithmic bytes (40 B/dof
    # for a nonlinear sweep, 16 for a linear one) over the step's device time
    sweep_bytes = k1_bytes + s3_bytes
    sweep_gbs = sweep_bytes / (ms_step * 1e-3) / 1e9
    sweep_traffic = None
    try:
        tp = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        sweep_traffic = tp.get(f"{cfg.name}:sweep")
    except Exception:
        pass
    roofline = {"bound": "hbm", "scope": "whole sweep (north_star: bytes moved per iteration over peak bandwidth)",
                "kernel": (f"sweep = stage 3 (k_line passes: x-IDST, fused y [V, N(u), V], x-DST) + K1 "
                           f"({k1_kernel(cfg, lay)}) + norm reduction" if nl
                           else f"sweep = K1 ({k1_kernel(cfg, lay)}) + norm reduction"),
                "achieved": sweep_gbs, "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
                "frac": sweep_gbs / hbm_peak, "traffic": sweep_traffic,
                "traffic_note": "ncu dram read+write bytes of one whole sweep (profiles/ncu_traffic.json)",
                "algorithmic_bytes_per_step": sweep_bytes,
                "bytes_per_dof": BYTES_PER_DOF["k1_complex" if cx else ("k1_nonlinear" if nl else "k1_linear")]
                + (BYTES_PER_DOF["stage3"] if nl else 0),
                "ms_per_step": ms_step}
    if passes:
        # stage-3 kernel families, timed live in full sweeps right after the timed region: CUDA
        # events recorded on the plan's stream between consecutive passes of stage 3 inside the
        # captured sweep (expd_sweep_pass_ms), summed per family, averaged over the sweeps
        M = cfg.n + 1
        s3 = cfg.nt - 1                                               # slices per sweep
        pairs = (cfg.n + 1) // 2                                      # line pairs per slice
        f_t = dst_flops_per_line_pair(M) * pairs                      # one axis transform / slice
        f_nl = 2 * f_t + 3.0 * 2 * M * pairs                          # [V, N, V], cubic N / slice
        fam = {}
        try:
            tprof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        except Exception:
            tprof = {}
        persistent = passes[-1]["x_launches"] == 0 and passes[-1]["fused_launches"] >= 1
        fams = ((("stage3_persistent", "fused_ms", "fused_launches", 2 * f_t + f_nl, s3),) if persistent else
                (("line_x", "x_ms", "x_launches", f_t, 2 * s3), ("line_y_nl", "fused_ms", "fused_launches", f_nl, s3)))
        for label, key, nkey, flops, slices in fams:
            ms_sweep = statistics.mean(p_[key] for p_ in passes)
            nlaunch = passes[-1][nkey]
            tf = flops * slices / (ms_sweep * 1e-3) / 1e12
            kname = {"line_x": "k_line (line_x: x-axis DST-I)", "line_y_nl": "k_line (line_y_nl: fused y [V, N(u), V])",
                     "stage3_persistent": "k_stage3p (persistent stage 3: x-IDST -> fused y [V, N(u), V] -> x-DST, "
                                          "intermediate in an L2-resident ring)"}[label]
            fam[label] = {"bound": "alu", "kernel": kname,
                          "achieved": tf, "peak": FP64_PEAK_TFLOPS,
                          "peak_source": "measured DFMA loop (profiles/r01_probe_fp64_hbm.txt)", "unit": "TFLOP/s",
                          "frac": tf / FP64_PEAK_TFLOPS, "traffic": tprof.get(f"{cfg.name}:{label}"),
                          "traffic_note": ("ncu dram bytes of the one launch per sweep" if persistent else
                                           f"ncu dram bytes of one launch ({slices / max(nlaunch, 1):.0f} slices)"),
                          "hbm_gbs": 16.0 * cfg.N * slices / (ms_sweep * 1e-3) / 1e9 if persistent else None,
                          "ncu": (tprof.get("counters") or {}).get(f"{cfg.name}:{label}"),
                          "algorithmic_flops_per_launch": flops * slices / max(nlaunch, 1),
                          "launch_ms": ms_sweep / max(nlaunch, 1), "launches_per_step": nlaunch,
                          "slices_per_step": slices, "ms_per_step": ms_sweep,
                          "timing": "CUDA events between the passes of full sweeps run right after the timed region"}
        kernels.update(fam)
        # the dominant kernel of the step by device time
        cand = [(k1_ms, k1_roof)] + [(v["ms_per_step"], v) for v in fam.values()]
        kernels["dominant"] = max(cand, key=lambda x: x[0])[1]["kernel"]
    else:
        kernels["dominant"] = k1_roof["kernel"]

    # e2e: the full solve through the C-ABI call with HOST buffers (pinned u0 and U): the
    # library copies u0 in, solves from the zero guess, and streams the solution out (the
    # final inverse DST chunk by chunk, each chunk's device-to-host copy overlapping the next
    # chunk's transform); distributed runs keep device buffers plus explicit copies
    e2e = None
    if not args.no_e2e:
        u0_h = torch.from_numpy(synth.initial_condition(cfg)).pin_memory()
        U_h = torch.empty((lay["nt_local"],) + cfg.shape, dtype=prob.dtype).pin_memory()
        u0_d = torch.empty_like(u0_h, device=dev)
        U_d = torch.empty((lay["nt_local"],) + cfg.shape, dtype=prob.dtype, device=dev)
        plan.set_profiling(False)
        plan.set_zero_guess(True)
        host_io = comm is None
        tot_ms, tot_sweeps = 0.0, 0
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize(dev)
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            if host_io:
                _, rep = plan.fixed_point_solve(u0_h, U_h, tol=cfg.tol, maxit=100)
            else:
                u0_d.copy_(u0_h, non_blocking=True)
                _, rep = plan.fixed_point_solve(u0_d, U_d, tol=cfg.tol, maxit=100)
                U_h.copy_(U_d, non_blocking=True)
            a1.record(stream)
            torch.cuda.synchronize(dev)
            if i > 0:  # first solve is warm-up
                tot_ms += a0.elapsed_time(a1)
                tot_sweeps += rep["sweeps"]
        if ws > 1:
            t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot_ms = float(t.item())
        e2e = {"value": cfg.nst * tot_sweeps / (tot_ms * 1e-3), "unit": "DOF-iter/s",
               "h2d_bytes_per_step": u0_h.numel() * esz * ws, "d2h_bytes_per_step": cfg.nst * esz,
               "what": f"full fixed-point solve per step ({rep['sweeps']} sweeps, {rep['iterations']} iterations, "
                       f"rel residual {rep['rel_residual']:.2e}) through the C-ABI call with host buffers: H2D of u0, "
                       f"setup DST, the sweeps (from the zero guess: the first sweep's stage 3 is skipped, N-hat of "
                       f"U = 0 being exactly 0), the final IDST streamed to the pinned host U (overlapped D2H)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline(cfg)
        except Exception as e:  # pragma: no cover
            cpu = {"error": str(e)}

    launches = plan.sweep_kernel_launches() * args.steps
    line = {
        "metric": "space-time DOF-iterations/s per Exp-ParaDiag sweep", "value": value, "unit": "DOF-iter/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128" if cx else "f64", "data": "synthetic",
        "config": {"workload": workload_label(cfg),
                   "n_st": cfg.nst, "alpha": cfg.alpha,
                   "l2": f"inputs {cfg.nst * esz / 1e9:.1f} GB per space-time array "
                         f"{'>>' if cfg.nst * esz > 126e6 else '<'} 126 MB L2"
                         f"{' (no flush needed)' if cfg.nst * esz > 126e6 else ' (L2-resident: not a roofline number)'}",
                   "parallelism": "single GPU" if ws == 1 else
                   f"{ws} GPUs: mode slabs (K1) / time slabs (stage 3), "
                   f"{'peer-memory row loads / stores' if peer else 'NCCL all-to-all'} + allreduce"},
        "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": ck,
        "residual_norm_last": float(np.sqrt(norms[-1])) if norms else None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if comm is not None:
        comm.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_gmres(args):
    """--solver gmres: a step is one Arnoldi step j of left-preconditioned GMRES:
    the K1 operator pass w = Q_alpha^{-1} Q v_j (16 B/dof) and CGS2 -- multi-dot over j+1 basis
    vectors, fused w -= V h + second multi-dot, fused w -= V h2 + ||w||^2 (8(3j+5) B/dof) --
    SURVEY §8(d.3): 16 + 8(3j+5) B/dof.  K steps = one GMRES(K) cycle run with tol 0 from U = 0,
    each step's device time taken by CUDA events on the plan's stream around its kernels
    (expd_solver_step_ms); the whole solve (setup, K steps with their host Givens round trips,
    x += V y, final IDST) is also timed end to end."""
    import torch
    import torch.distributed as dist

    import synth
    from paper_2603_04350_b200 import Comm, Plan, Problem
    from paper_2603_04350_b200 import build as pbuild

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if rank == 0:
        pbuild.build()
    if ws > 1:
        dist.barrier()
    cfg = synth.CONFIGS[args.config]
    if cfg.q:
        raise SystemExit("--solver gmres: linear configs only (GMRES is for npoly == 0)")
    prob = Problem.from_config(cfg)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    comm = Comm(rank, ws, local) if ws > 1 else None
    K = args.steps
    plan = Plan(prob, device=local, stream=stream, comm=comm, krylov_vectors=K + 1)
    lay = plan.layout
    cx = cfg.is_complex
    esz = 16 if cx else 8
    u0 = torch.from_numpy(synth.initial_condition(cfg)).to(dev)
    U = torch.zeros((lay["nt_local"],) + cfg.shape, dtype=prob.dtype, device=dev)
    plan.set_profiling(True)
    for _ in range(max(1, args.warmup // 3)):
        U.zero_()
        plan.gmres_solve(u0, U, tol=0.0, restart=K, maxit=K)
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    U.zero_()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    ev0.record(stream)
    _, rep = plan.gmres_solve(u0, U, tol=0.0, restart=K, maxit=K)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    ck = clocks.stop()
    steps_ms = plan.solver_step_ms()
    solve_ms = ev0.elapsed_time(ev1)
    dev_ms = sum(steps_ms)
    if ws > 1:
        t = torch.tensor([dev_ms, solve_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, solve_ms = (float(x) for x in t.tolist())
    pk = peaks()
    hbm_peak = pk["hbm_gbs"] if pk else 6650.0
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if pk else "fallback (B200_PROFILING.md)"
    share = lay["mode_len"] / lay["npad"]
    dof_bytes = esz * cfg.nst * share  # one space-time vector of this rank, in bytes
    per_step = [(16 + 8 * (3 * j + 5)) / 8 * dof_bytes for j in range(1, len(steps_ms) + 1)]
    gbs = sum(per_step) / (dev_ms * 1e-3) / 1e9
    value = cfg.nst * len(steps_ms) / (dev_ms * 1e-3)
    roofline = {"bound": "hbm", "scope": "GMRES Arnoldi steps j = 1..K (SURVEY §8(d.3): 16 + 8(3j+5) B/dof)",
                "kernel": f"{k1_kernel(cfg, lay)} (RM_QOP: w = Q_alpha^{{-1}} Q v_j) + k_multi_dot + 2 x k_axpy_dot "
                          "(CGS2, ||w||^2)",
                "achieved": gbs, "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s", "frac": gbs / hbm_peak,
                "traffic": None, "algorithmic_bytes_per_step": per_step,
                "step_ms": steps_ms}
    line = {
        "metric": "space-time DOF-iterations/s per Exp-ParaDiag GMRES (Arnoldi) step", "value": value,
        "unit": "DOF-iter/s", "n_gpus": ws, "steps": len(steps_ms), "warmup": args.warmup,
        "ms_per_step": dev_ms / max(len(steps_ms), 1), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128" if cx else "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.dim}D n={cfg.n} Nt={cfg.nt} GMRES({K}) Arnoldi steps, tol 0 "
                               f"(BASELINE.json{ {'c2': ':8', 'c4': ':10'}.get(cfg.name, '') })",
                   "n_st": cfg.nst, "alpha": cfg.alpha,
                   "l2": f"basis vectors {cfg.nst * esz / 1e9:.2f} GB each vs 126 MB L2"},
        "roofline": roofline,
        "e2e_solve_ms": solve_ms, "e2e_note": "the whole GMRES(K) solve on resident data incl. setup DSTs, the "
                                             "host Givens round trip per step, x += V y and the final IDST",
        "clocks": ck, "hist": rep["hist"], "iterations": rep["iterations"],
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if comm is not None:
        comm.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    env_ws = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and env_ws is None:
        return self_launch(args)
    if int(env_ws or 1) != args.gpus:
        print(f"bench.py: WORLD_SIZE={env_ws} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.launch_check:
        return launch_check(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.solver == "gmres":
        return run_gmres(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
