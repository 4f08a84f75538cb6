"""Pole ("time") parallelism across GPUs.

The N+1 poles of the half-sum are independent and cost the same, so rank r of P
evaluates the contiguous block [r (N+1) / P, (r+1)(N+1) / P) through
``rexi_apply_partial`` (forward FFT, its poles, inverse FFT + Re — the inverse
transform and Re are real-linear, so they commute with the sum), and ONE
all-reduce (sum, fp64) over NCCL/NVLink combines the three real fields
(option b of SURVEY.md 8(e): 3 D^2 doubles instead of 3 D^2 complex).
"""
from __future__ import annotations


def pole_partition(n_poles, world_size, rank):
    """Contiguous block of rank `rank`; block sizes differ by at most one pole."""
    if world_size < 1 or not (0 <= rank < world_size):
        raise ValueError("bad rank / world size")
    return (n_poles * rank) // world_size, (n_poles * (rank + 1)) // world_size


def _event(out):
    """A timing event recorded on the current stream of out's device (None on CPU)."""
    import torch
    if not (hasattr(out, "is_cuda") and out.is_cuda):
        return None
    e = torch.cuda.Event(enable_timing=True)
    e.record(torch.cuda.current_stream(out.device))
    return e


def pole_parallel_step(partial_fn, n_poles, out, group=None, timers=None):
    """Generic S3 + S4: ``partial_fn(begin, end, out)`` writes this rank's partial result
    into ``out`` (a tensor holding the three fields); then one all-reduce(sum).

    ``timers`` (optional list): appends (start, partial done, all-reduce done) CUDA events
    recorded on the current stream (the all-reduce's completion is ordered into it)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    b, e = pole_partition(n_poles, world, rank)
    e0 = _event(out) if timers is not None else None
    partial_fn(b, e, out)
    e1 = _event(out) if timers is not None else None
    if dist.is_initialized():
        # also at world size 1 (the collective then runs as NCCL's single-rank copy)
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    if timers is not None and e0 is not None:
        timers.append((e0, e1, _event(out)))
    return out


def apply_distributed(plan, eta, u, v, out=None, group=None, timers=None):
    """One REXII step with the poles split over the ranks of `group` (one GPU per rank).

    ``out`` (optional) is a contiguous (3, D, D) float64 CUDA tensor; returns it."""
    import torch
    if out is None:
        out = torch.empty((3, plan.D, plan.D), dtype=torch.float64, device=eta.device)

    def partial(b, e, buf):
        plan.apply_partial(b, e, eta, u, v, out=(buf[0], buf[1], buf[2]))

    return pole_parallel_step(partial, plan.n_poles, out, group, timers)


def run_distributed(plan, steps, eta, u, v, group=None, spectral=False):
    """`steps` REXII steps in place (S6, T_final = steps * tau) with every step's poles split
    over the ranks of `group`. Returns (eta, u, v).

    spectral=False: per step one pole-parallel `apply_distributed` (S1, the rank's poles, S5,
    all-reduce of the three real fields), the summed fields becoming the next step's input.
    spectral=True (spectral-resident, NEXT-4): S1 once; per step every rank evaluates its poles
    on the shared Hermitian spectrum (rexi_poles_real), the ranks all-reduce the spectrum's rows
    l = 0 .. D/2 (per field; the same bytes as the real fields) and rebuild the other rows by
    Hermitian symmetry (rexi_hermitian_mirror) — the next step's input; S5 once at the end. The
    real part of each step is the Hermitian projection the R2C kernel applies, so
    this equals the physical-space loop up to rounding, without two FFTs per step."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if not spectral:
        buf = torch.empty((3, plan.D, plan.D), dtype=torch.float64, device=eta.device)
        for _ in range(int(steps)):
            apply_distributed(plan, eta, u, v, out=buf, group=group)
            eta.copy_(buf[0])
            u.copy_(buf[1])
            v.copy_(buf[2])
        return eta, u, v
    b, e = pole_partition(plan.n_poles, world, rank)
    fhat = plan.forward(eta, u, v)
    acc = torch.empty_like(fhat)
    half = plan.D // 2 + 1
    for _ in range(int(steps)):
        plan.poles_real(fhat, b, e, acc=acc)
        if dist.is_initialized():
            for c in range(3):
                dist.all_reduce(acc[c, :half], op=dist.ReduceOp.SUM, group=group)
        plan.hermitian_mirror(acc)
        fhat, acc = acc, fhat
    plan.inverse(fhat, out=(eta, u, v))
    return eta, u, v
