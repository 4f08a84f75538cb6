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
def oracle_rate(D, tau, tol, scen, seconds, threads=0):
    """Time the oracle (as it stands) on a bounded sample of the workload: all poles on a
    deterministic sample of Fourier modes (per-mode work is identical across modes).
    Returns (pole·gp/s, cores, sample description, n_poles)."""
    from oracle import coeffs as C
    from oracle import lrsw
    from paper_2008_11607_b200 import inputs
    cores = lrsw.num_threads(threads)
    h = 0.5
    M = C.M_lrsw(D, tau, h, tol)
    n, al, c1, c2, g = C.rexii_terms(h, M).half()
    f = scenario(scen, D)
    # spectral input by the oracle's own naive DFT (one-off, not part of the timed sample)
    F = lrsw.spectral_fields(*f)
    S = 64
    rate = None
    desc = ""
    while True:
        ml, mk = inputs.sample_modes(D, S)
        fm = F[ml, mk, :]
        t0 = time.perf_counter()
        lrsw.rexii_pole_sum(D, tau, fm, ml, mk, al, c1, c2, g)
        dt = time.perf_counter() - t0
        rate = len(ml) * len(g) / dt
        desc = (f"{len(ml)} sampled Fourier modes x all {len(g)} poles (dense 3x3 LU per mode, "
                f"2 solves per pole) of the {D}^2 step; {dt:.1f} s")
        if dt >= seconds or S >= D * D:
            break
        S = min(D * D, int(S * max(2.0, min(16.0, seconds / max(dt, 1e-3) * 1.2))))
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
            "ms_per_step": 1e3 * n_poles * D * D / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: LRSW {D}x{D}, tau={tau}, tol={tol}, h=0.5, "
                                   f"{n_poles} poles, {scen} scenario (BASELINE configs[{cidx}])"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- native arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    if args.backend == "gloo":
        # functional check of the multi-rank control flow on fewer GPUs than ranks (host-side
        # all-reduce, no kernel waits on another rank); its timings are not bench numbers
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
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

    def step():
        if world > 1:
            apply_distributed(plan, *f, out=out)
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
    plan.timing_enable(True)
    plan.timing_read()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    for i in range(args.steps):
        flush.zero_()                      # L2 flush between timed steps, outside the events
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    clocks.mark()
    if world > 1:
        dist.barrier()
    ms_local = sum(a.elapsed_time(b) for a, b in ev)
    pole_ms, pole_launches, launches = plan.timing_read()
    plan.timing_enable(False)
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    time.sleep(0.25)
    clocks.stop()
    clk = clocks.summary()

    # ---- end to end through the public API with host buffers (pinned), copies inside
    pinned_in = [torch.from_numpy(x).pin_memory() for x in f_host]
    pinned_out = [torch.empty((D, D), dtype=torch.float64).pin_memory() for _ in range(3)]
    e2e_steps = max(3, min(args.steps, 50))

    def e2e_step():
        if world > 1:
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
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        te = torch.tensor([dt], dtype=torch.float64, device=dev)
        if world > 1:
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
    value = units * args.steps / (ms_total / 1e3)
    # roofline of the dominant kernel (the pole kernel) on this rank
    rank_units = (pe - pb) * D * D
    pole_avg_s = (pole_ms / 1e3) / max(1, pole_launches)
    achieved = info["flops_per_pole_mode"] * rank_units / pole_avg_s / 1e12 if pole_avg_s > 0 else None
    pipe_frac = (info["fp64_ops_per_pole_mode"] * rank_units / pole_avg_s / FP64_PIPE_PEAK_OPS
                 if pole_avg_s > 0 else None)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "pole_kernel_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get(f"{args.config}_{args.variant}")
        except Exception:
            traffic = None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
            "steps_per_s": args.steps / (ms_total / 1e3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: LRSW {D}x{D}, tau={tau}, tol={tol}, "
                                   f"h={info['h']:.4g}, M={info['M']}, {n_poles} poles, {scen} scenario "
                                   f"(BASELINE configs[{cidx}])",
                       "variant": args.variant, "tuning": args.tuning or "default", "l2": "flushed between timed steps (256 MB write)",
                       "parallelism": f"poles split over {world} GPU(s)"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None,
                         "traffic": traffic, "kernel": "pole_kernel",
                         "flops_per_pole_mode": info["flops_per_pole_mode"],
                         # SURVEY.md 8(d)'s per-unit figure is the paper's route (~200 flops per
                         # pole-gridpoint); the kernel's exact rearrangements execute fewer, so the
                         # roofline uses the kernel's own count and this is reported beside it
                         "paper_route_flops_per_pole_mode": 200.0,
                         "paper_route_equiv_tflops": (200.0 * rank_units / pole_avg_s / 1e12
                                                      if pole_avg_s > 0 else None),
                         "fp64_pipe_frac": pipe_frac,
                         "kernel_ms_avg": pole_avg_s * 1e3,
                         "kernel_share_of_step": (pole_ms / ms_local) if ms_local > 0 else None,
                         "peak_note": "derived: 148 SM x 64 fp64 FMA/clk x 2 x 1.965 GHz"},
            "clocks": clk,
            "e2e": {"value": units * e2e_n / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": 3 * D * D * 8, "d2h_bytes_per_step": 3 * D * D * 8,
                    "ms_per_step": 1e3 * e2e_s / e2e_n, "mode": e2e_mode,
                    "single_call_ms_per_step": 1e3 * single_s / e2e_steps},
            "gpu_launches": launches,
        }
        if world == 1 and not args.no_cpu_baseline:
            rate, cores, desc, _, _ = oracle_rate(D, tau, tol, scen, args.cpu_seconds)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": desc}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
