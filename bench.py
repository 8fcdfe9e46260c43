#!/usr/bin/env python3
"""FMM hot-path benchmark (BASELINE.json metric: "P2P+M2L interactions/s and FMM ms/step at
N=1M; achieved % of FP32 peak").

A step = one whole FMM evaluation (tree build, dual traversal, upward, M2L, P2P, downward) of
BASELINE config C2: N = 1 048 576 bodies uniform in [-1,1]^3, q in (0,1/N], p = 6, n_crit = 64,
theta = 0.5, FP32 P2P / FP64 expansions, potential + acceleration. Synthetic data from the
reference's xorshift64* generator.

  value   interactions/s = (P2P body pairs + M2L cell pairs) per step / device step time, with
          the bodies resident in HBM before the timed region (CUDA events on the FMM stream);
  e2e     the same metric through the C-ABI with host buffers: H2D of the bodies, the step,
          and D2H of phi + acceleration (input order) inside the timed region;
  roofline  the P2P kernel's throughput (20 flops per body pair) against the peak of the pipe
            it runs on (FP32 for --precision fp32, FP64 for the fp64 parity mode);
  cpu_baseline  the reference's own CPU FMM (oracle/_ref, its scheduler) on the host cores.

`--impl reference` times the reference's CPU FMM (oracle/_ref) with all host threads.
Multi-GPU (torchrun): ranks run the sharded step; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # BASELINE.json configs (name -> generator config, n, p, n_crit, theta)
    "C1": (1, 16384, 4, 64, 0.5),
    "C2": (2, 1 << 20, 6, 64, 0.5),
    "C3": (3, 1 << 20, 6, 64, 0.5),
    "C4": (4, 1 << 24, 8, 128, 0.4),
    "C5": (5, 1 << 22, 10, 64, 0.5),
}
METRIC = "P2P+M2L interactions/s and FMM ms/step at N=1M; achieved % of FP32 peak"
UNIT = "interactions/s"
FLOPS_PER_PAIR = 20  # potential + acceleration


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = {}
    if os.path.exists(path):
        with open(path) as f:
            peaks = json.load(f)
    return peaks


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML polled every ~2 ms
    from a thread (the handle is opened before the region starts), nvidia-smi -lms as fallback."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int = 0):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, set of reasons)
        self._stop = threading.Event()
        self._proc = None
        self._nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._bits = {"hw_slowdown": pynvml.nvmlClocksThrottleReasonHwSlowdown,
                          "hw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                          "sw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonSwThermalSlowdown,
                          "sw_power_cap": pynvml.nvmlClocksThrottleReasonSwPowerCap}
        except Exception:
            self._nv = None

    def _poll_nvml(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                self.samples.append((float(sm), float(self._max), {k for k, v in self._bits.items() if r & v}))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._poll_nvml, daemon=True)
            self._t.start()
            return self
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read_smi, daemon=True)
            self._t.start()
        except Exception:
            self._proc = None
        return self

    def _read_smi(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6 and parts[0].replace(".", "").isdigit():
                self.samples.append((float(parts[0]), float(parts[1]),
                                     {self.NAMES[k] for k in range(4) if parts[2 + k] == "Active"}))

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1)
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = sorted(set().union(*[s[2] for s in self.samples]))
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nv is not None else "nvidia-smi"}


def flush_l2(buf):
    if buf is not None:
        buf.zero_()


DIST = {1: "uniform [-1,1]^3, q in (0,1/N]", 2: "uniform [-1,1]^3, q in (0,1/N]",
        3: "Plummer sphere (scale radius 1, r <= 100), q = 1/N", 4: "uniform [-1,1]^3, q in (0,1/N]",
        5: "unit sphere surface (normalised Gaussian), q in [-1,1]/N"}
L2_NOTE = ("flushed between steps by a 256 MB write (device buffer on the GPU arm, host buffer on "
           "the CPU reference arm); > 126 MB L2")


def workload_config(cfg_name, n, world=1, strong=False):
    """The `config` object, identical for the GPU arm and the CPU reference arm."""
    gen, n_cfg, p, n_crit, theta = CONFIGS[cfg_name]
    cfg = {"workload": f"{cfg_name}: N={n} {DIST[gen]}, p={p}, n_crit={n_crit}, theta={theta}, "
                       "potential+acceleration (reference: potential)",
           "n_bodies": n, "order": p, "n_crit": n_crit, "theta": theta, "l2": L2_NOTE,
           "seed": 1}
    if world > 1:
        cfg["parallelism"] = (f"dp{world}: target leaves sharded by cost-balanced Morton range, NCCL "
                              "all-gather of owned multipoles" + (" (strong scaling: N fixed)" if strong else ""))
    else:
        cfg["parallelism"] = "single GPU"
    return cfg


def _ref_bodies(gen, n):
    """BASELINE bodies from the oracle's restated generator (bit-identical to
    fmm_generate_bodies, tests/test_oracle.py): the reference arm never loads libfmm_b200.so."""
    import oracle
    return oracle.Oracle().generate_baseline_bodies(gen, n, 1)


def _ref_interactions(ref, bodies, n_crit, p, theta):
    t = ref.build_tree(bodies, n_crit, p)
    c = t.cells()
    m, pp = t.traverse(theta)
    nb = (c.body_end - c.body_begin).astype(np.int64)
    return int((nb[pp[:, 0]] * nb[pp[:, 1]]).sum()), len(m)


def _host_flush(buf):
    buf += 1  # 256 MB write: the CPU arm's counterpart of the GPU arm's L2 flush


STAGES = ("build", "upward", "traversal+m2l+p2p", "downward")


def cpu_reference(gen, n, p, n_crit, theta, steps=1, warmup=0, single_core=False):
    """The reference CPU FMM (oracle/_ref: the unmodified sources) at the config's N.
    All cores: its scheduler with nproc-1 workers + the helping master (scheduler.cpp:62-72),
    Q = RunConfig's default (engine.hpp:32-35). Optional 1 core: inline traversal with Q = inf
    on a thread pinned to one core. Per-stage medians (engine.cpp:69-106)."""
    import oracle
    ref = oracle.Reference()
    bodies = _ref_bodies(gen, n)
    n_pairs, n_m2l = _ref_interactions(ref, bodies, n_crit, p, theta)
    inter = n_pairs + n_m2l
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    threads = max(1, cores - 1)
    q = max(n // 100, 64)
    flush = np.zeros(256 << 20, np.uint8)
    for _ in range(warmup):
        ref.step(bodies, n_crit, p, theta, q, threads)
    totals, stages = [], []
    for _ in range(max(1, steps)):
        _host_flush(flush)
        t0 = time.perf_counter()
        st, _ = ref.step(bodies, n_crit, p, theta, q, threads)
        totals.append(time.perf_counter() - t0)
        stages.append(st)
    sec = float(np.median(totals))
    out = {"value": inter / sec, "ms_per_step": sec * 1e3, "cores": cores, "threads": threads + 1,
           "interactions_per_step": inter, "p2p_body_pairs": n_pairs, "m2l_pairs": n_m2l,
           "stage_ms": dict(zip(STAGES, (1e3 * np.median(np.array(stages), 0)).tolist())),
           "sample": f"full config N={n}: reference scheduler, {threads} workers + master on {cores} host "
                     f"cores, Q={q}, median of {len(totals)} step(s)"}
    try:
        import platform
        out["cpu_model"] = next((ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo")
                                 if ln.startswith("model name")), platform.processor())
    except Exception:
        pass
    if single_core:
        import threading
        res = {}

        def pinned():
            cpu = sorted(os.sched_getaffinity(0))[0]
            os.sched_setaffinity(0, {cpu})  # this thread only (Linux: pid 0 = calling thread)
            t0 = time.perf_counter()
            st, _ = ref.step(bodies, n_crit, p, theta, 1 << 30, 0)
            res["s"] = time.perf_counter() - t0
            res["st"] = st

        th = threading.Thread(target=pinned)
        th.start()
        th.join()
        out["single_core"] = {"ms_per_step": res["s"] * 1e3, "value": inter / res["s"], "cores": 1,
                              "stage_ms": dict(zip(STAGES, (1e3 * np.asarray(res["st"])).tolist())),
                              "setting": "inline traversal, Q=inf, thread pinned to one core, 1 step"}
    return out


def run_reference(args, cfg_name):
    """--impl reference: the reference's own CPU FMM (oracle/_ref) on the host cores, at the
    config's full N (C4/C5: a bounded sample, see --ref-n); rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    if not oracle.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfmmref.so not built"}))
        return 0
    gen, n_full, p, n_crit, theta = CONFIGS[cfg_name]
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    n = args.ref_n or (n_full if n_full <= (1 << 20) else (1 << 20))
    res = cpu_reference(gen, n, p, n_crit, theta, steps=args.steps, warmup=min(args.warmup, 1),
                        single_core=not args.no_single_core)
    cfg = workload_config(cfg_name, n_full, world, strong=cfg_name == "C4")
    line = {"metric": METRIC, "impl": "reference", "value": res["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": min(args.warmup, 1),
            "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE generator: reference xorshift64*, seed 1)", "config": cfg,
            "interactions_per_step": res["interactions_per_step"], "stage_ms": res["stage_ms"],
            "cpu_baseline": {"value": res["value"], "unit": UNIT, "cores": res["cores"],
                             "kind": "reference", "sample": res["sample"]},
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "cpu_model": res.get("cpu_model"), "single_core": res.get("single_core"),
            "warmup_note": "CPU arm: at most 1 warm-up step (no device state to warm)"}
    if n != n_full:
        line["sampled_n"] = n
    print(json.dumps(line))
    return 0


def run_sharded(args, fb, torch, world, rank, local):
    """torchrun, one rank per GPU. The step is the library's fmm_evaluate_sharded: every rank
    builds the (bit-identical) tree, traverses its targets, computes its own cells' multipoles and
    all-gathers them with the library's own NCCL communicator (fmm_comm_init; the exchange runs
    under the P2P kernel), then M2L / P2P / L2L / L2P for its Morton range of target leaves.
    torch.distributed only bootstraps: it ships the NCCL unique id and takes max-over-ranks.
    Strong scaling (default): N fixed at the config's N at every world size."""
    import torch.distributed as dist
    os.environ.setdefault("NCCL_DEBUG", "INFO")  # the driver checks the communicator's rank count
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    gen, n_cfg, p, n_crit, theta = CONFIGS[args.config]
    strong = args.scaling == "strong"
    n = n_cfg if strong else n_cfg * world
    bodies = fb.generate_bodies(gen, n, 1)
    ctx = fb.Context(order=p, n_crit=n_crit, theta=theta, precision=args.precision, device=local, with_acc=True)
    uid = [fb.fmm.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ctx.comm_init(uid[0], rank, world)
    d_bodies = torch.from_numpy(bodies).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ctx.set_bodies_device(d_bodies.data_ptr(), n)
    n_m2l_problem = None
    for w in range(args.warmup):
        ctx.evaluate_sharded()
        if w == 0:  # the first step traverses in full (and plans): the problem's M2L pairs
            n_m2l_problem = int(ctx.tree_info().n_m2l)
    torch.cuda.synchronize()
    times, launches, stage_acc = [], 0, {}
    keys = ("build_ms", "traverse_ms", "upward_ms", "m2l_ms", "p2p_ms", "downward_ms", "exchange_ms",
            "p2p_kernel_ms", "m2l_kernel_ms")
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            info = ctx.evaluate_sharded()
            t = ctx.stage_times()
            times.append(t.total_ms)
            launches += t.kernel_launches
            for k in keys:
                stage_acc[k] = stage_acc.get(k, 0.0) + getattr(t, k)
    torch.cuda.synchronize()
    dist.barrier()
    total = torch.tensor([float(np.sum(times))], device="cuda")
    dist.all_reduce(total, op=dist.ReduceOp.MAX)
    ms_per_step = total.item() / args.steps
    tinfo = ctx.tree_info()
    own_p2p = torch.tensor([float(tinfo.p2p_body_pairs)], device="cuda", dtype=torch.float64)
    dist.all_reduce(own_p2p)
    p2p_total = int(own_p2p.item())
    inter = p2p_total + n_m2l_problem  # M2L pairs of shared targets counted once
    mine = {"rank": rank, "body_range": [int(info.body_begin), int(info.body_end)],
            "own_leaves": int(info.own_leaves), "own_cells": int(info.own_cells),
            "p2p_body_pairs": int(tinfo.p2p_body_pairs), "n_m2l_rank": int(tinfo.n_m2l),
            "stage_ms": {k: v / args.steps for k, v in stage_acc.items()}}
    per_rank = [None] * world
    dist.all_gather_object(per_rank, mine)

    e2e = None
    if not args.no_e2e:
        # through the library per rank and step: H2D of the rank's 1/world share from pinned
        # memory + NCCL all-gather of the shares (fmm_set_bodies_shard), the sharded step, D2H of
        # the own results and their input indices (fmm_get_owned_results); max over ranks
        chunk = (n + world - 1) // world
        b0, b1 = min(n, rank * chunk), min(n, (rank + 1) * chunk)
        h_in = torch.from_numpy(np.ascontiguousarray(bodies[b0:b1])).pin_memory()
        ts, nres = [], 0
        dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.set_bodies_shard_ptr(h_in.data_ptr(), b1 - b0, n)
            sinfo = ctx.evaluate_sharded()
            phi, acc, idx = ctx.owned_results(sinfo)
            ts.append(time.perf_counter() - t0)
            nres = len(phi)
        assert np.isfinite(phi).all()
        e2e_ms = torch.tensor([float(np.mean(ts)) * 1e3], device="cuda")
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": inter / (e2e_ms.item() * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms.item(),
               "h2d_bytes_per_step": int((b1 - b0) * 32), "d2h_bytes_per_step": int(nres * (32 + 8)),
               "path": "fmm_set_bodies_shard (H2D share + NCCL all-gather) + fmm_evaluate_sharded + "
                       "fmm_get_owned_results", "per": "rank 0's copies; time = max over ranks"}
    if rank == 0:
        peaks = load_peaks()
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        fp32 = args.precision == "fp32"
        peak = sms * (128 if fp32 else 64) * 2 * sm_max * 1e6 / 1e12
        worst_p2p = max(r["stage_ms"]["p2p_kernel_ms"] for r in per_rank)
        achieved = FLOPS_PER_PAIR * p2p_total / (worst_p2p * 1e-3) / 1e12 / world
        line = {"metric": METRIC, "value": inter / (ms_per_step * 1e-3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if strong else "weak", "vs_baseline": None,
                "dtype": "f32 P2P / f64 expansions" if fp32 else "f64",
                "data": "synthetic (BASELINE generator: reference xorshift64*, seed 1)",
                "config": workload_config(args.config, n, world, strong), "precision": args.precision,
                "interactions_per_step": inter, "p2p_body_pairs": p2p_total, "m2l_pairs": n_m2l_problem,
                "roofline": {"bound": "fp32" if fp32 else "fp64", "achieved": achieved, "peak": peak,
                             "unit": "TFLOP/s per GPU", "frac": achieved / peak, "traffic": None,
                             "kernel": "k_p2p_fp32_ws" if fp32 else "k_p2p_fp64", "flops_per_unit": FLOPS_PER_PAIR,
                             "timing": "all ranks' P2P pairs x 20 flops / the slowest rank's P2P kernel "
                                       "(CUDA events, in the step) / world"},
                "per_rank": per_rank, "e2e": e2e,
                "cpu_baseline": None, "cpu_baseline_note": "the CPU baseline is timed at N=1 only (rank 0)",
                "clocks": clk.summary(), "gpu_launches": launches,
                "nccl": {"comm": "library-owned (fmm_comm_init, NCCL loaded at run time)",
                         "collective": "ncclAllGather of owned multipoles, one per step"}}
        print(json.dumps(line))
    ctx.close()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded (torchrun) path even at world size 1 (tests the NCCL flow on one GPU)")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2", choices=list(CONFIGS))
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="multi-GPU: strong = the config's N at every world size; weak = N x world")
    ap.add_argument("--ref-n", type=int, default=0,
                    help="CPU reference N (default: the config's N up to 2^20; C4/C5 sample 2^20)")
    ap.add_argument("--no-single-core", action="store_true",
                    help="reference arm: skip the 1-core (Q=inf, pinned) step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fp64-mode", action="store_true",
                    help="skip the FP64 parity-mode leg (reported as fp64_mode in the line)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, args.config)

    import torch
    import paper_1203_0889_b200 as fb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.sharded:
        return run_sharded(args, fb, torch, world, rank, local)
    return run_single(args, fb, torch, local)


def time_steps(ctx, torch, flush, steps, clk=None):
    """K evaluate() steps, L2 flushed before each; per-step CUDA-event times from the library."""
    step_ms, p2p_ms, m2l_ms, launches, stage_acc = [], [], [], 0, {}
    torch.cuda.synchronize()
    for _ in range(steps):
        flush_l2(flush)
        torch.cuda.synchronize()
        ctx.evaluate()
        t = ctx.stage_times()
        step_ms.append(t.total_ms)
        p2p_ms.append(t.p2p_kernel_ms)
        m2l_ms.append(t.m2l_kernel_ms)
        launches += t.kernel_launches
        for k in ("build_ms", "traverse_ms", "upward_ms", "m2l_ms", "p2p_ms", "downward_ms"):
            stage_acc[k] = stage_acc.get(k, 0.0) + getattr(t, k)
    torch.cuda.synchronize()
    return step_ms, p2p_ms, m2l_ms, launches, {k: v / steps for k, v in stage_acc.items()}


def serialised_kernel_times(ctx, torch, flush, reps):
    """Roofline pass (outside the timed steps): stages serialised so that the P2P and M2L
    kernels each run alone (in the default overlap the L2L levels share the SMs with P2P and the
    P2P work list with M2L)."""
    p2p, m2l = [], []
    ctx.set_overlap(0)
    for _ in range(reps):
        flush_l2(flush)
        torch.cuda.synchronize()
        ctx.evaluate()
        t = ctx.stage_times()
        p2p.append(t.p2p_kernel_ms)
        m2l.append(t.m2l_kernel_ms)
    ctx.set_overlap(1)
    return float(np.mean(p2p)), float(np.mean(m2l))


M2L_FLOPS = {4: 335, 6: 1469, 8: 4699, 10: 12455}  # SURVEY.md section 8(d), per M2L pair


def m2l_flops_per_pair(p):
    """2 C(p+5, 6) (one FMA per folded term) + the D-table recurrence
    over the n_coef(p) derivatives of degree <= p-1 (multi_index.cpp:59-85, ~10 flops each)."""
    from math import comb
    return M2L_FLOPS.get(p, 2 * comb(p + 5, 6) + 10 * (p * (p + 1) * (p + 2) // 6))


def run_single(args, fb, torch, local):
    gen, n, p, n_crit, theta = CONFIGS[args.config]
    bodies = fb.generate_bodies(gen, n, 1)
    ctx = fb.Context(order=p, n_crit=n_crit, theta=theta, precision=args.precision, device=local,
                     with_acc=True)
    d_bodies = torch.from_numpy(bodies).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    ctx.set_bodies_device(d_bodies.data_ptr(), n)
    # default stage order: the upward pass runs on a second stream concurrently with the
    # traversal; the P2P work list beside M2L; L2L beside P2P
    for _ in range(args.warmup):
        ctx.evaluate()
    info = ctx.tree_info()
    inter = int(info.p2p_body_pairs) + int(info.n_m2l)
    with ClockSampler(local) as clk:
        step_ms, p2p_ms, m2l_ms, launches, stage_ms = time_steps(ctx, torch, flush, args.steps)
    ms_per_step = float(np.sum(step_ms)) / args.steps
    value = inter / (ms_per_step * 1e-3)
    p2p_kernel, m2l_kernel = serialised_kernel_times(ctx, torch, flush, max(3, min(args.steps, 10)))

    # roofline: the P2P kernel (dominant at C2), 20 flops per body pair, against the peak of the
    # pipe it runs on
    peaks = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    fp32 = args.precision == "fp32"
    fp32_peak = sms * 128 * 2 * sm_max * 1e6 / 1e12
    fp64_peak = sms * 64 * 2 * sm_max * 1e6 / 1e12
    pipe_peak = fp32_peak if fp32 else fp64_peak
    p2p_name = "k_p2p_fp32_ws" if fp32 else "k_p2p_fp64"
    achieved = FLOPS_PER_PAIR * info.p2p_body_pairs / (p2p_kernel * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        key = f"{args.config}/{args.precision}"
        if key in tj.get("by_config", {}):
            traffic = tj["by_config"][key]["dram_bytes_per_launch"]
    except Exception:
        traffic = None
    # M2L: FP64 pipe (flops per pair: SURVEY.md section 8d) and its algorithmic HBM bytes
    # (one source multipole row per pair + one local row per target), CUDA events, alone
    ncoef = p * (p + 1) * (p + 2) // 6
    m2l_fpp = m2l_flops_per_pair(p)
    m2l_tf = m2l_fpp * info.n_m2l / (m2l_kernel * 1e-3) / 1e12
    m2l_bytes = 8 * ncoef * (info.n_m2l + info.ncells)
    m2l_kname = "k_m2l_reg<%d>" % p if p <= 6 else ("k_m2l_flat<%d>" if p >= 10 else "k_m2l_big2<%d>") % p
    roofline_m2l = {"bound": "fp64", "achieved": m2l_tf, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": m2l_tf / fp64_peak, "kernel": m2l_kname, "flops_per_unit": m2l_fpp,
                    "unit_of_work": "M2L cell pair", "kernel_ms": m2l_kernel,
                    "source_bytes_per_s_algorithmic": m2l_bytes / (m2l_kernel * 1e-3),
                    "bytes_note": "8 n_coef bytes per pair (source row) + per cell (local row); the "
                                  "multipoles of C1-C3 (<= 29 MB) are L2-resident, so this rate is "
                                  "served by L2, not HBM; HBM peak %.0f GB/s" % float(peaks.get("hbm_gbs", 6446.6)),
                    "peak_source": f"derived: {sms} SMs x 64 FP64 lanes x 2 x {sm_max:.0f} MHz (DFMA "
                                   "microbenchmark 60 lane-ops/clk/SM, profiles/r1_microbench_pipes.txt)"}

    # FP64 parity mode (the reference's precision): same workload, its own context and steps
    fp64_mode = None
    if fp32 and not args.no_fp64_mode:
        c64 = fb.Context(order=p, n_crit=n_crit, theta=theta, precision="fp64", device=local, with_acc=True)
        c64.set_bodies_device(d_bodies.data_ptr(), n)
        for _ in range(3):
            c64.evaluate()
        k64 = max(3, min(args.steps, 10))
        s64, p64, _, _, st64 = time_steps(c64, torch, flush, k64)
        ms64 = float(np.mean(s64))
        a64 = FLOPS_PER_PAIR * info.p2p_body_pairs / (float(np.mean(p64)) * 1e-3) / 1e12
        fp64_mode = {"ms_per_step": ms64, "value": inter / (ms64 * 1e-3), "unit": UNIT, "steps": k64,
                     "stage_ms": st64, "p2p_kernel": "k_p2p_fp64", "p2p_kernel_ms": float(np.mean(p64)),
                     "p2p_frac_of_fp64_peak": a64 / fp64_peak}
        c64.close()

    # e2e through the C-ABI with host buffers (pinned), H2D + step + D2H in the timed region
    e2e = None
    if not args.no_e2e:
        h_in = torch.from_numpy(bodies).pin_memory()
        h_phi = torch.empty(n, dtype=torch.float64).pin_memory()
        h_acc = torch.empty(3 * n, dtype=torch.float64).pin_memory()
        import ctypes as C
        lib = ctx.lib
        dp = C.POINTER(C.c_double)
        ptr = lambda tns: C.cast(tns.data_ptr(), dp)  # noqa: E731
        for _ in range(2):
            lib.fmm_set_bodies(ctx.h, ptr(h_in), n)
            lib.fmm_evaluate(ctx.h)
            lib.fmm_get_results(ctx.h, ptr(h_phi), ptr(h_acc), 1)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc = lib.fmm_set_bodies(ctx.h, ptr(h_in), n)
            rc |= lib.fmm_evaluate(ctx.h)
            rc |= lib.fmm_get_results(ctx.h, ptr(h_phi), ptr(h_acc), 1)
            ts.append(time.perf_counter() - t0)
            assert rc == 0, lib.fmm_last_error(ctx.h)
        e2e_ms = float(np.mean(ts)) * 1e3
        e2e = {"value": inter / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(n * 32), "d2h_bytes_per_step": int(n * 8 * 4),
               "path": "fmm_set_bodies(host) + fmm_evaluate + fmm_get_results(host, input order)"}

    # extra (not the headline): the same e2e calls from two host threads on two contexts, so one
    # evaluation's PCIe copies run under the other's kernels (independent evaluations, e.g. a
    # parameter sweep; the serial e2e above stays the reported figure)
    if e2e is not None and n <= (1 << 22):
        try:
            import threading
            ctx2 = fb.Context(order=p, n_crit=n_crit, theta=theta, precision=args.precision, device=local,
                              with_acc=True)
            bufs = [(h_in, h_phi, h_acc),
                    (torch.from_numpy(bodies).pin_memory(), torch.empty(n, dtype=torch.float64).pin_memory(),
                     torch.empty(3 * n, dtype=torch.float64).pin_memory())]
            per = max(2, (args.steps + 1) // 2)
            rcs = [0, 0]

            def worker(i, c, k):
                torch.cuda.set_device(local)
                a, b, d = bufs[i]
                for _ in range(k):
                    rcs[i] |= lib.fmm_set_bodies(c.h, ptr(a), n)
                    rcs[i] |= lib.fmm_evaluate(c.h)
                    rcs[i] |= lib.fmm_get_results(c.h, ptr(b), ptr(d), 1)

            worker(1, ctx2, 2)  # warm the second context
            torch.cuda.synchronize()
            th = [threading.Thread(target=worker, args=(i, c, per)) for i, c in enumerate((ctx, ctx2))]
            t0 = time.perf_counter()
            for t in th:
                t.start()
            for t in th:
                t.join()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            assert rcs == [0, 0]
            assert np.array_equal(bufs[0][1].numpy(), bufs[1][1].numpy()), "pipelined contexts disagree"
            e2e["pipelined_two_contexts"] = {
                "value": inter * 2 * per / dt, "unit": UNIT, "ms_per_step": dt * 1e3 / (2 * per), "steps": 2 * per,
                "note": "two host threads, two contexts, same calls as e2e; copies of one evaluation overlap "
                        "the kernels of the other; no L2 flush between steps (extra, not the headline)"}
            ctx2.close()
        except Exception as e:  # the extra never blocks the line
            e2e["pipelined_two_contexts"] = {"value": None, "note": f"failed: {e}"}

    # CPU baseline: the unmodified reference (oracle/_ref) at the same N, all host cores, 1 step
    cpu = None
    if not args.no_cpu_baseline:
        try:
            import oracle
            if oracle.reference_available() and n <= (1 << 20):
                r = cpu_reference(gen, n, p, n_crit, theta, steps=1)
                cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
                       "sample": r["sample"], "ms_per_step": r["ms_per_step"], "stage_ms": r["stage_ms"]}
            elif oracle.reference_available():
                nr = 1 << 20
                r = cpu_reference(gen, nr, p, n_crit, theta, steps=1)
                cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
                       "sample": f"N={nr} sample of the {args.config} distribution (full N would take "
                                 f"minutes per step): " + r["sample"],
                       "ms_per_step": r["ms_per_step"], "stage_ms": r["stage_ms"]}
            else:
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                       "sample": "oracle/_ref not built"}
        except Exception as e:  # the baseline never blocks the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 P2P / f64 expansions" if fp32 else "f64",
        "data": "synthetic (BASELINE generator: reference xorshift64*, seed 1)",
        "config": workload_config(args.config, n), "precision": args.precision,
        "interactions_per_step": inter, "p2p_body_pairs": int(info.p2p_body_pairs),
        "m2l_pairs": int(info.n_m2l), "p2p_pairs_per_s": info.p2p_body_pairs / (ms_per_step * 1e-3),
        "m2l_pairs_per_s": info.n_m2l / (ms_per_step * 1e-3),
        "stage_ms": stage_ms, "p2p_kernel_ms": p2p_kernel, "m2l_kernel_ms": m2l_kernel,
        "roofline": {"bound": "fp32" if fp32 else "fp64", "achieved": achieved, "peak": pipe_peak,
                     "unit": "TFLOP/s", "frac": achieved / pipe_peak, "traffic": traffic,
                     "traffic_unit": f"bytes per launch (dram read + write, ncu, {args.config} "
                                     f"{args.precision}; profiles/ncu_traffic.json)",
                     "kernel": p2p_name, "flops_per_unit": FLOPS_PER_PAIR,
                     "unit_of_work": "target-source body pair (n_t * n_s per P2P leaf pair)",
                     "timing": "CUDA events around the P2P launch in a serialised pass after the timed "
                               "steps (the kernel runs alone), L2 flushed",
                     "peak_source": f"derived: {sms} SMs x {128 if fp32 else 64} {'FP32' if fp32 else 'FP64'} "
                                    f"lanes x 2 x {sm_max:.0f} MHz (sm_max_mhz of MEASURED_PEAKS.json, which "
                                    "has no FP32/FP64 figure; microbenchmarks: FFMA2 126-128, DFMA 60 "
                                    "lane-ops/clk/SM). Flop convention: 20 per pair (SURVEY 8d), rsqrt = 2 "
                                    "flops in both precisions"},
        "roofline_m2l": roofline_m2l, "fp64_mode": fp64_mode,
        "e2e": e2e, "cpu_baseline": cpu, "clocks": clk.summary(),
        "gpu_launches": launches, "tree": {"ncells": info.ncells, "nleaves": info.nleaves,
                                           "depth": info.depth},
    }
    print(json.dumps(line))
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
