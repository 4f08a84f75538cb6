#!/usr/bin/env python
"""Throughput of one REXII step (S1..S5, all poles) on B200 — the bench contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--variant dz]
    python bench.py --impl reference ...      # the oracle (CPU) as the reference arm

Workload (default, BASELINE.json configs[1]): 2-D linear SWE on a 512 x 512 periodic grid,
one REXII step of tau = 1 at tol = 1e-8 (h = 0.5, M = 4558, 4583 poles), Gaussian scenario
initial data (eq:GAUSSIANSCENARIO), fp64. A "step" = one rexi_apply.
Metric: pole·gridpoint solves per second = n_poles * D^2 / step time (whole job).
For N > 1 the poles are split over the ranks (rexi_apply_partial) and one NCCL all-reduce
sums the three fields: the total work is fixed ("scaling": "strong").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (D, tau, tol, scenario, BASELINE.json configs index)
    "c1": (64, 0.02, 1e-12, "gaussian", 0),
    "c2": (512, 1.0, 1e-8, "gaussian", 1),
    "c3": (1024, 0.1, 1e-12, "gaussian", 2),
    "c4": (4096, 1.0, 1e-12, "gaussian", 3),
}
METRIC = "REXI pole·gridpoint solves/s"
UNIT = "pole·gp/s"
# fp64 peak derived from unit counts and clocks: 148 SMs x 64 DFMA
# lanes/clk x 2 flop x 1.965 GHz (clocks.max.sm, B200_PROFILING.md).
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
FP64_PIPE_PEAK_OPS = 148 * 64 * 1.965e9


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--variant", default="pfhx", choices=["pfhx", "pfhr", "pfh", "pf", "dz", "dz3", "uv"])
    ap.add_argument("--h", default="0.5", help="Gaussian spacing h, or 'auto' (NEXT-2 h_for_tol)")
    ap.add_argument("--tuning", default=None,
                    help="pole kernel tuning 'modes_per_thread,poles_per_iter,min_blocks' (default: plan's)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: functional check only)")
    ap.add_argument("--dist", action="store_true",
                    help="use the process-group path (apply_distributed + all-reduce) even at world size 1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def scenario(name, D):
    from paper_2008_11607_b200 import inputs
    return {"gaussian": inputs.gaussian_scenario, "white": inputs.white_noise}[name](D)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ["uuid", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, uuid):
        self.uuid = (uuid or "").lower().replace("gpu-", "")
        self.rows = []
        self.proc = None
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            if self.uuid and self.uuid not in parts[0].lower():
                continue
            self.rows.append((time.time(), parts))

    def mark(self):
        self.marks.append(time.time())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows or len(self.marks) < 2:
            return None
        t0, t1 = self.marks[0], self.marks[-1]
        sel = [r for t, r in self.rows if t0 - 0.05 <= t <= t1 + 0.05] or [r for _, r in self.rows[-3:]]

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in sel if num(r[1]) is not None]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in sel:
            for i, n in enumerate(names):
                if r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": num(sel[0][2]), "reasons": sorted(reasons), "samples": len(sel),
                "power_w_max": max((num(r[3]) or 0.0) for r in sel)}


# ----------------------------------------------------------------------------- CPU oracle
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_rate(D, tau, tol, scen, seconds, threads=0):
    """Time the oracle (as it stands) on a bounded sample of the workload: all poles on a
    deterministic sample of Fourier modes (per-mode work is identical across modes).
    threads > 0 sets the oracle's OpenMP thread count for this call (restored after).
    Returns (pole·gp/s, cores, sample description, n_poles, seconds)."""
    from oracle import coeffs as C
    from oracle import lrsw
    from paper_2008_11607_b200 import inputs
    prev = lrsw.num_threads(0)
    cores = lrsw.num_threads(threads)
    h = 0.5
    M = C.M_lrsw(D, tau, h, tol)
    n, al, c1, c2, g = C.rexii_terms(h, M).half()
    f = scenario(scen, D)
    # spectral input by the oracle's own naive DFT (one-off, not part of the timed sample)
    F = lrsw.spectral_fields(*f)
    S = 64 if threads != 1 else 8
    rate = None
    desc = ""
    try:
        while True:
            ml, mk = inputs.sample_modes(D, S)
            fm = F[ml, mk, :]
            t0 = time.perf_counter()
            lrsw.rexii_pole_sum(D, tau, fm, ml, mk, al, c1, c2, g)
            dt = time.perf_counter() - t0
            rate = len(ml) * len(g) / dt
            desc = (f"{len(ml)} sampled Fourier modes x all {len(g)} poles (dense 3x3 LU per mode, "
                    f"2 solves per pole) of the {D}^2 step on {cores} thread(s); {dt:.1f} s")
            if dt >= seconds or S >= D * D:
                break
            S = min(D * D, int(S * max(2.0, min(16.0, seconds / max(dt, 1e-3) * 1.2))))
    finally:
        lrsw.num_threads(prev)
    return rate, cores, desc, len(g), dt


def run_reference(args):
    """--impl reference: the oracle timed on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    D, tau, tol, scen, cidx = CONFIGS[args.config]
    per_step = max(0.2, min(2.0, 120.0 / max(1, args.steps + args.warmup)))
    rate, cores, desc, n_poles, dt = oracle_rate(D, tau, tol, scen, per_step)
    from oracle import coeffs as C
    from oracle import lrsw
    from paper_2008_11607_b200 import inputs
    M = C.M_lrsw(D, tau, 0.5, tol)
    n, al, c1, c2, g = C.rexii_terms(0.5, M).half()
    # each step: the same bounded sample (modes chosen above), timed
    S = max(1, int(rate * per_step / n_poles))
    ml, mk = inputs.sample_modes(D, S)
    F = lrsw.spectral_fields(*scenario(scen, D))
    fm = F[ml, mk, :]
    for _ in range(args.warmup):
        lrsw.rexii_pole_sum(D, tau, fm, ml, mk, al, c1, c2, g)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        lrsw.rexii_pole_sum(D, tau, fm, ml, mk, al, c1, c2, g)
    T = time.perf_counter() - t0
    value = args.steps * len(ml) * n_poles / T
    sample = (f"each step: {len(ml)} sampled Fourier modes x all {n_poles} poles of the {D}^2 "
              f"tau={tau} step (dense per-mode LU, naive), {T / args.steps:.3f} s")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            # measured wall time of one timed step (a bounded sample of the workload)
            "ms_per_step": 1e3 * T / args.steps,
            # the whole D^2 step at this rate: an extrapolation, not a measurement
            "full_step_ms_extrapolated": 1e3 * n_poles * D * D / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: LRSW {D}x{D}, tau={tau}, tol={tol}, h=0.5, "
                                   f"{n_poles} poles, {scen} scenario (BASELINE configs[{cidx}])"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def nccl_summary(path):
    """The communicator lines of this rank's NCCL INFO log (echoed to stderr): init, nranks,
    transport (NVLS / P2P), so the run shows which communicator the all-reduce used."""
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError:
        return None
    sys.stderr.write(text)
    keys = ("Init COMPLETE", "nranks", "NVLS", "P2P", "comm 0x", "Channel")
    lines = [ln.split("NCCL INFO", 1)[-1].strip() for ln in text.splitlines() if any(k in ln for k in keys)]
    return {"log": path, "lines": len(text.splitlines()), "init": lines[:12]}


# ----------------------------------------------------------------------------- native arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist_on = world > 1 or args.dist
    nccl_log = None
    if dist_on and args.backend == "nccl":
        # communicator evidence: NCCL's INIT lines (rank, nranks, channels / NVLS) go to a file
        # (NCCL's default is stdout, which must keep the one JSON line); they are echoed to
        # stderr and summarised in the line's "comm" object at the end
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if "NCCL_DEBUG_FILE" not in os.environ:
            import tempfile
            nccl_log = os.path.join(tempfile.gettempdir(), f"rexi_bench_nccl.{os.getpid()}.log")
            os.environ["NCCL_DEBUG_FILE"] = nccl_log
    import torch
    import torch.distributed as dist
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    if args.backend == "gloo":
        # functional check of the multi-rank control flow on fewer GPUs than ranks (host-side
        # all-reduce, no kernel waits on another rank); its timings are not bench numbers
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if dist_on:
        if args.backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_2008_11607_b200 import rexi
    from paper_2008_11607_b200.distributed import apply_distributed, pole_partition

    D, tau, tol, scen, cidx = CONFIGS[args.config]
    h_arg = "auto" if args.h == "auto" else float(args.h)
    plan = rexi.Plan(D, tau, tol=tol, h=h_arg, device=local, variant=args.variant)
    if args.tuning:
        plan.set_tuning(*[int(x) for x in args.tuning.split(",")])
    info = plan.info
    n_poles = info["n_poles"]
    pb, pe = pole_partition(n_poles, world, rank)
    f_host = [np.ascontiguousarray(x) for x in scenario(scen, D)]
    f = [torch.from_numpy(x).to(dev) for x in f_host]
    out = torch.empty((3, D, D), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > L2
    stream = torch.cuda.current_stream(dev)

    def step(timers=None):
        if dist_on:
            apply_distributed(plan, *f, out=out, timers=timers)
        else:
            plan.apply(*f, out=(out[0], out[1], out[2]))

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    uuid = None
    try:
        uuid = str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        pass
    clocks = ClockSampler(uuid)
    clocks.start()
    time.sleep(0.3)
    plan.timing_enable(False)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    rank_timers = []                       # per step: (start, partial done, all-reduce done)
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    for i in range(args.steps):
        flush.zero_()                      # L2 flush between timed steps, outside the events
        ev[i][0].record(stream)
        step(rank_timers if dist_on else None)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    clocks.mark()
    if dist_on:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms_local = sum(step_ms)
    # kernel-timing pass: the same K steps again, with the library's CUDA events around the pole
    # kernel (or the fused step) on its stream. Kept out of the timed steps above: two event
    # records per step cost ~6 us of a 23 us C1 step (tools/time_step_events.py), 0.4 % at C2.
    plan.timing_enable(True)
    plan.timing_read()
    ev_k = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        ev_k[i][0].record(stream)
        step()
        ev_k[i][1].record(stream)
    torch.cuda.synchronize()
    ms_local_k = sum(a.elapsed_time(b) for a, b in ev_k)
    pole_ms, pole_launches, launches = plan.timing_read()
    plan.timing_enable(False)
    # per-step time = max over ranks of that step; the statistic is the median
    t = torch.tensor(step_ms + [ms_local], dtype=torch.float64, device=dev)
    if dist_on:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t = t.tolist()
    step_max = t[:-1]
    ms_median = statistics.median(step_max)
    ms_mean = sum(step_max) / len(step_max)
    ms_total = t[-1]
    time.sleep(0.25)
    clocks.stop()
    clk = clocks.summary()

    # fp64-pipe peak of this GPU, measured now (the roofline denominator)
    peak_ops, _ = rexi.fp64_peak(local, reps=5)
    peak_tflops = 2.0 * peak_ops / 1e12

    # per-rank breakdown (S3 pole kernel, rexi_apply_partial, S4 all-reduce)
    pole_avg_s = (pole_ms / 1e3) / max(1, pole_launches)
    mine = {"rank": rank, "poles": [pb, pe], "pole_kernel_ms": pole_avg_s * 1e3,
            "step_ms_median": statistics.median(step_ms), "fp64_peak_tflops": peak_tflops}
    if rank_timers:
        part = [a.elapsed_time(b) for a, b, _ in rank_timers]
        ar = [b.elapsed_time(c) for _, b, c in rank_timers]
        mine["apply_partial_ms"] = statistics.median(part)
        mine["allreduce_ms"] = statistics.median(ar)
    ranks = [mine]
    if dist_on:
        ranks = [None] * world
        dist.all_gather_object(ranks, mine)

    # ---- end to end through the public API with host buffers (pinned), copies inside
    pinned_in = [torch.from_numpy(x).pin_memory() for x in f_host]
    pinned_out = [torch.empty((D, D), dtype=torch.float64).pin_memory() for _ in range(3)]
    e2e_steps = max(3, min(args.steps, 50))

    def e2e_step():
        if dist_on:
            for d_, h_ in zip(f, pinned_in):
                d_.copy_(h_, non_blocking=True)
            apply_distributed(plan, *f, out=out)
            for c in range(3):
                pinned_out[c].copy_(out[c], non_blocking=True)
            torch.cuda.synchronize()
        else:
            plan.apply_host(*pinned_in, out=pinned_out)

    def timed(fn, reps):
        fn()
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        te = torch.tensor([dt], dtype=torch.float64, device=dev)
        if dist_on:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return float(te.item())

    # one synchronous rexi_apply_host call per step: copies serialised with the step
    single_s = timed(e2e_step, e2e_steps)
    e2e_mode = "rexi_apply_host per step (copies serialised with the step)"
    e2e_s, e2e_n = single_s, e2e_steps
    if world == 1:
        # a stream of independent problems through rexi_apply_host_batch: problem i+1's inputs
        # and problem i-1's outputs cross PCIe while problem i is computed
        B = max(3, min(e2e_steps, int(2e9 // (48 * D * D))))
        bin_ = [torch.from_numpy(np.ascontiguousarray(np.broadcast_to(x, (B, D, D)))).pin_memory()
                for x in f_host]
        bout = [torch.empty((B, D, D), dtype=torch.float64).pin_memory() for _ in range(3)]
        plan.apply_host_batch(*[x[:2] for x in bin_], out=[x[:2] for x in bout])
        batch_s = timed(lambda: plan.apply_host_batch(*bin_, out=bout), 1)
        if not np.array_equal(bout[0][-1].numpy(), pinned_out[0].numpy()):
            raise RuntimeError("rexi_apply_host_batch result differs from rexi_apply_host")
        e2e_mode = (f"rexi_apply_host_batch over {B} problems (copies of neighbouring problems "
                    f"overlap each step)")
        e2e_s, e2e_n = batch_s, B
        del bin_, bout

    units = n_poles * D * D                           # pole·gridpoints per step, whole job
    value = units / (ms_median / 1e3)
    # roofline of the dominant kernel (the pole kernel) on this rank: algorithmic flops of the
    # kernel's route (DESIGN.md 6.1 recount) x the pole·gridpoints of one launch / its time
    rank_units = (pe - pb) * D * D
    per_s = rank_units / pole_avg_s if pole_avg_s > 0 else None
    achieved = info["flops_per_pole_mode"] * per_s / 1e12 if per_s else None
    pipe_frac = info["fp64_ops_per_pole_mode"] * per_s / peak_ops if per_s else None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_median,
            "ms_per_step_mean": ms_mean, "ms_timed_region": ms_total,
            "statistic": "median over the timed steps of the per-step max over ranks (CUDA events)",
            "steps_per_s": 1e3 / ms_median,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: LRSW {D}x{D}, tau={tau}, tol={tol}, "
                                   f"h={info['h']:.4g}, M={info['M']}, {n_poles} poles, {scen} scenario "
                                   f"(BASELINE configs[{cidx}])",
                       "variant": args.variant, "tuning": args.tuning or "default",
                       "l2": "flushed between timed steps (256 MB write)",
                       "parallelism": f"poles split over {world} GPU(s)"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_tflops,
                         "unit": "TFLOP/s", "frac": (achieved / peak_tflops) if achieved else None,
                         "traffic": None,
                         "traffic_note": "DRAM bytes per launch are an ncu quantity (profiles/r02*_summary.md); "
                                         "not measurable inside this run",
                         "kernel": ("pole_kernel_r2x (S2+S3)" if os.environ.get("REXI_R2X_BULK", "1") == "0"
                                    or (args.tuning and args.tuning.replace(" ", "") != "8,8,2")
                                    else "pole_kernel_r2x_bulk (S2+S3)") if args.variant == "pfhx"
                                   else "pole_kernel",
                         "flops_per_pole_mode": info["flops_per_pole_mode"],
                         "fp64_ops_per_pole_mode": info["fp64_ops_per_pole_mode"],
                         "peak_source": "measured in this run: rexi_fp64_peak (DFMA, register operands, "
                                        "best of 5), x 2 flop per DFMA",
                         "peak_derived": FP64_PEAK_TFLOPS,
                         # SURVEY.md 8(d)'s per-unit figure (the paper's Helmholtz route, ~200 flops
                         # per pole-gridpoint): > 1 means the kernel's route executes fewer flops
                         "frac_survey_route_200": (200.0 * per_s / 1e12 / peak_tflops) if per_s else None,
                         "fp64_pipe_frac": pipe_frac,
                         "kernel_ms_avg": pole_avg_s * 1e3,
                         "kernel_share_of_step": (pole_ms / ms_local_k) if ms_local_k > 0 else None,
                         "kernel_timing": "CUDA events on the kernel's stream around every pole-kernel "
                                          "(or fused-step) launch, in a second pass of the same K "
                                          "steps (L2 flushed likewise) after the timed one"},
            "clocks": clk,
            "e2e": {"value": units * e2e_n / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": 3 * D * D * 8, "d2h_bytes_per_step": 3 * D * D * 8,
                    "ms_per_step": 1e3 * e2e_s / e2e_n, "mode": e2e_mode,
                    "single_call_ms_per_step": 1e3 * single_s / e2e_steps},
            "gpu_launches": launches,   # repo kernels launched in the K steps (kernel-timing pass count)
        }
        if dist_on:
            line["ranks"] = ranks
            line["comm"] = {"backend": args.backend, "nranks": dist.get_world_size(),
                            "collective": "all_reduce(sum, fp64) of the 3 real fields, once per step",
                            "bytes_per_step": 3 * D * D * 8,
                            "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))
                            if args.backend == "nccl" else None}
            if nccl_log:
                line["comm"]["nccl_init"] = nccl_summary(nccl_log)
        if world == 1 and not args.no_cpu_baseline:
            rate, cores, desc, _, _ = oracle_rate(D, tau, tol, scen, args.cpu_seconds)
            rate1, _, desc1, _, _ = oracle_rate(D, tau, tol, scen, min(5.0, args.cpu_seconds / 2), threads=1)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": desc, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                                    "value_1core": rate1, "sample_1core": desc1}
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
