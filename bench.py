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


def run_reference(args, cfg_name):
    """--impl reference: the reference's own CPU FMM (oracle/_ref, scheduler with all host
    threads) on a bounded sample of the workload; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    if not oracle.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfmmref.so not built"}))
        return 0
    gen, n_full, p, n_crit, theta = CONFIGS[cfg_name]
    res = cpu_reference_sample(gen, n_full, p, n_crit, theta, args.ref_sample, steps=args.steps,
                               warmup=args.warmup)
    line = {"metric": METRIC, "impl": "reference", "value": res["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE generator, seeded)",
            "config": res["config"],
            "cpu_baseline": {"value": res["value"], "unit": UNIT, "cores": res["cores"],
                             "kind": "reference", "sample": res["sample"]},
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def cpu_reference_sample(gen, n_full, p, n_crit, theta, n_sample, steps=1, warmup=0):
    """The reference CPU FMM (build + upward + scheduled traversal/kernels + downward) on a
    same-distribution sample of n_sample bodies; interactions/s = (P2P pairs + M2L pairs)/s."""
    import oracle
    import paper_1203_0889_b200.fmm as fb
    ref = oracle.Reference()
    n = min(n_sample, n_full)
    bodies = fb.generate_bodies(gen, n, 1)
    cores = os.cpu_count() or 1
    threads = max(1, cores - 1)  # the master also executes tasks (scheduler.cpp:62-72)
    # interaction counts of this sample (reference traversal)
    t = ref.build_tree(bodies, n_crit, p)
    c = t.cells()
    m, pp = t.traverse(theta)
    nb = (c.body_end - c.body_begin).astype(np.int64)
    inter = int((nb[pp[:, 0]] * nb[pp[:, 1]]).sum()) + len(m)
    del t
    q = max(n // 100, 64)  # RunConfig default queue threshold (engine.hpp:32-35)
    for _ in range(warmup):
        ref.step(bodies, n_crit, p, theta, q, threads)
    times = []
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        ref.step(bodies, n_crit, p, theta, q, threads)
        times.append(time.perf_counter() - t0)
    sec = float(np.mean(times))
    return {"value": inter / sec, "ms_per_step": sec * 1e3, "cores": cores,
            "sample": f"N={n} bodies of the same distribution (p={p}, n_crit={n_crit}, theta={theta}), "
                      f"reference scheduler with {threads} workers + master, {len(times)} step(s), "
                      f"{inter} interactions/step",
            "config": {"workload": f"C{gen}: same distribution/p/n_crit/theta as the GPU arm; reference CPU "
                                   f"FMM timed on a bounded N={n} sample (interactions/s)",
                       "n_bodies": n, "order": p, "n_crit": n_crit, "theta": theta}}


def run_sharded(args, fb, torch, world, rank, local):
    """torchrun, one rank per GPU: weak scaling, N = 2^20 * world bodies of the config's
    distribution held by every rank; target leaves sharded by cost-balanced Morton range; the
    owned multipoles all-gathered with NCCL over NVLink (the step's only data-path exchange)."""
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    gen, n1, p, n_crit, theta = CONFIGS[args.config]
    n = n1 * world
    bodies = fb.generate_bodies(gen, n, 1)
    ctx = fb.Context(order=p, n_crit=n_crit, theta=theta, precision=args.precision, device=local, with_acc=True)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)  # NCCL and the FMM kernels share one stream
    d_bodies = torch.from_numpy(bodies).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    class Buf:
        def __init__(self, k):
            self.t = torch.empty(int(k), dtype=torch.float64, device="cuda")
            self.ptr = self.t.data_ptr()

    def all_gather(recv, send):
        dist.all_gather_into_tensor(recv.t, send.t)

    def step():
        ctx.set_bodies_device(d_bodies.data_ptr(), n)
        return fb.fmm.sharded_step(ctx, rank, world, all_gather, Buf)

    for w in range(args.warmup):
        step()
        if w == 0:  # the first step traverses in full (and plans): the problem's unique M2L pairs
            n_m2l_problem = int(ctx.tree_info().n_m2l)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    launches = 0
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0.record(stream)
            info = step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            launches += ctx.stage_times().kernel_launches
    torch.cuda.synchronize()
    dist.barrier()
    total = torch.tensor([float(np.sum(times))], device="cuda")
    dist.all_reduce(total, op=dist.ReduceOp.MAX)
    ms_per_step = total.item() / args.steps
    tinfo = ctx.tree_info()
    own_p2p = torch.tensor([float(tinfo.p2p_body_pairs)], device="cuda", dtype=torch.float64)
    dist.all_reduce(own_p2p)
    inter = int(own_p2p.item()) + n_m2l_problem  # M2L pairs of shared targets counted once

    # e2e through the public API, per rank and step: H2D of this rank's 1/world share of the
    # bodies from pinned memory, NCCL all-gather of the shares over NVLink (every rank builds the
    # full tree), the sharded step, and D2H of the results this rank owns (its contiguous
    # tree-order body range, read from the context's result buffers); max over ranks
    e2e = None
    if not args.no_e2e:
        chunk = n // world  # n = 2^20 * world
        h_in = torch.from_numpy(np.ascontiguousarray(bodies[rank * chunk:(rank + 1) * chunk])).pin_memory()
        d_part = torch.empty_like(h_in, device="cuda")
        h_phi = torch.empty(n, dtype=torch.float64).pin_memory()  # own range <= n
        h_acc = torch.empty((n, 3), dtype=torch.float64).pin_memory()

        class _Dev:  # zero-copy torch view of a context result buffer
            def __init__(self, ptr, shape):
                self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f8", "data": (ptr, False),
                                                 "version": 3, "strides": None}

        ts = []
        dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d_part.copy_(h_in, non_blocking=True)
            dist.all_gather_into_tensor(d_bodies, d_part)
            sinfo = step()
            b0, b1 = int(sinfo.body_begin), int(sinfo.body_end)
            pphi, pacc = ctx.results_device()
            d_phi = torch.as_tensor(_Dev(pphi, (n,)), device="cuda")
            d_acc = torch.as_tensor(_Dev(pacc, (n, 3)), device="cuda")
            h_phi[:b1 - b0].copy_(d_phi[b0:b1], non_blocking=True)
            h_acc[:b1 - b0].copy_(d_acc[b0:b1], non_blocking=True)
            torch.cuda.current_stream().synchronize()
            ts.append(time.perf_counter() - t0)
        assert np.isfinite(h_phi[:b1 - b0].numpy()).all()
        e2e_ms = torch.tensor([float(np.mean(ts)) * 1e3], device="cuda")
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": inter / (e2e_ms.item() * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms.item(),
               "h2d_bytes_per_step": int(chunk * 32), "d2h_bytes_per_step": int((b1 - b0) * 32),
               "per": "rank 0 (each rank copies its own share; bodies all-gathered over NVLink: "
                      f"{int(n * 32)} bytes per rank)"}
    if rank == 0:
        line = {"metric": METRIC, "value": inter / (ms_per_step * 1e-3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "f32 P2P / f64 expansions" if args.precision == "fp32" else "f64",
                "data": "synthetic (BASELINE generator, seed 1)",
                "config": {"workload": f"{args.config} distribution, N={n} (2^20 per GPU), p={p}, n_crit={n_crit}, "
                                       f"theta={theta}, potential+acceleration",
                           "n_bodies": n, "order": p, "n_crit": n_crit, "theta": theta, "precision": args.precision,
                           "parallelism": f"dp{world}: target leaves sharded by cost-balanced Morton range, "
                                          "NCCL all-gather of owned multipoles",
                           "l2": "flushed (256 MB write) between steps"},
                "interactions_per_step": inter, "e2e": e2e, "cpu_baseline": None, "clocks": clk.summary(),
                "gpu_launches": launches, "own_body_range_rank0": [int(info.body_begin), int(info.body_end)]}
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
    ap.add_argument("--ref-sample", type=int, default=262144)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
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
    dist = None

    gen, n, p, n_crit, theta = CONFIGS[args.config]
    bodies = fb.generate_bodies(gen, n, 1)
    ctx = fb.Context(order=p, n_crit=n_crit, theta=theta, precision=args.precision, device=local,
                     with_acc=True)
    d_bodies = torch.from_numpy(bodies).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    ctx.set_bodies_device(d_bodies.data_ptr(), n)
    # default stage order: the upward pass runs on a second stream concurrently with the
    # traversal; M2L, P2P and the downward pass follow on one stream (P2P timed alone)

    for _ in range(args.warmup):
        ctx.evaluate()
    info = ctx.tree_info()
    inter = int(info.p2p_body_pairs) + int(info.n_m2l)

    step_ms, p2p_ms, m2l_ms, launches = [], [], [], 0
    stage_acc = {}
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
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
    # roofline pass (outside the timed steps): stages serialised so that the P2P kernel runs
    # alone (in the default overlap the L2L levels share the SMs with it)
    p2p_alone = []
    ctx.set_overlap(0)
    for _ in range(max(3, min(args.steps, 10))):
        flush_l2(flush)
        torch.cuda.synchronize()
        ctx.evaluate()
        p2p_alone.append(ctx.stage_times().p2p_kernel_ms)
    ctx.set_overlap(1)
    total_ms = float(np.sum(step_ms))
    if dist:
        tt = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    value = inter * world / (ms_per_step * 1e-3)

    # roofline: the P2P kernel, FP32 pipe (20 flops per body pair), CUDA events around its
    # launch in the serialised pass (the kernel runs alone)
    peaks = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    fp32 = args.precision == "fp32"
    lanes = 128 if fp32 else 64  # FP32 / FP64 lanes per SM (FFMA2 126, DFMA 60 ops/clk/SM measured)
    pipe_peak = sms * lanes * 2 * sm_max * 1e6 / 1e12  # TFLOP/s
    p2p_name = "k_p2p_fp32_ws" if fp32 else "k_p2p_fp64"
    p2p_kernel = float(np.mean(p2p_alone))
    achieved = FLOPS_PER_PAIR * info.p2p_body_pairs / (p2p_kernel * 1e-3) / 1e12
    # DRAM bytes per launch of the same kernel from the committed ncu --set full capture
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        key = f"{args.config}/{args.precision}"
        if key in tj.get("by_config", {}):
            traffic = tj["by_config"][key]["dram_bytes_per_launch"]
        elif key == "C2/fp32":
            traffic = tj[p2p_name]["dram_bytes_per_launch"]
    except Exception:
        traffic = None

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
        if dist:
            dist.barrier()
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
        if dist:
            tt = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        e2e = {"value": inter * world / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(n * 32), "d2h_bytes_per_step": int(n * 8 * 4)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            import oracle
            if oracle.reference_available():
                r = cpu_reference_sample(gen, n, p, n_crit, theta, args.ref_sample)
                cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
                       "sample": r["sample"]}
            else:
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                       "sample": "oracle/_ref not built"}
        except Exception as e:  # the baseline never blocks the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 P2P / f64 expansions"
            if args.precision == "fp32" else "f64",
            "data": "synthetic (BASELINE C2 generator: reference xorshift64*, seed 1+rank)",
            "config": {"workload": f"{args.config}: N={n} uniform [-1,1]^3, p={p}, n_crit={n_crit}, "
                                   f"theta={theta}, potential+acceleration",
                       "n_bodies": n, "order": p, "n_crit": n_crit, "theta": theta,
                       "precision": args.precision, "l2": "flushed (256 MB write) between steps",
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "interactions_per_step": inter, "p2p_body_pairs": int(info.p2p_body_pairs),
            "m2l_pairs": int(info.n_m2l), "p2p_pairs_per_s": info.p2p_body_pairs / (ms_per_step * 1e-3),
            "m2l_pairs_per_s": info.n_m2l / (ms_per_step * 1e-3),
            "stage_ms": {k: v / args.steps for k, v in stage_acc.items()},
            "p2p_kernel_ms": p2p_kernel, "m2l_kernel_ms": float(np.mean(m2l_ms)),
            "roofline": {"bound": "fp32" if fp32 else "fp64", "achieved": achieved, "peak": pipe_peak,
                         "unit": "TFLOP/s", "frac": achieved / pipe_peak, "traffic": traffic,
                         "traffic_unit": f"bytes per launch (dram read + write, ncu, {args.config} "
                                         f"{args.precision}; profiles/ncu_traffic.json)",
                         "kernel": p2p_name, "flops_per_unit": FLOPS_PER_PAIR,
                         "timing": "CUDA events around the P2P launch in a serialised pass after the timed steps (the kernel runs alone), L2 flushed",
                         "peak_source": f"derived: {sms} SMs x {lanes} {'FP32' if fp32 else 'FP64'} lanes x 2 x "
                                        f"{sm_max:.0f} MHz (sm_max_mhz of MEASURED_PEAKS.json; "
                                        + ("FFMA2 microbenchmark measured 126-128 lane-ops/clk/SM)" if fp32 else
                                           "DFMA microbenchmark measured 60 lane-ops/clk/SM)")},
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk.summary(),
            "gpu_launches": launches, "tree": {"ncells": info.ncells, "nleaves": info.nleaves,
                                               "depth": info.depth},
        }
        print(json.dumps(line))
    ctx.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
