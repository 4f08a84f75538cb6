"""Example: pole-parallel REXII steps over the GPUs of one node (one process per GPU, NCCL).

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 examples/lrsw_multi_gpu.py [D] [tau] [steps]

Every rank builds the same plan (term count from the paper's rule for tol 1e-12), evaluates its
contiguous block of the poles (the terms are independent) and the ranks sum their
partial results with one NCCL all-reduce per step; the state stays in Fourier space between steps
(distributed.run_distributed(spectral=True)). Rank 0 prints the per-step time (max over ranks,
CUDA events) and the energy drift. Runs with one process too (the NCCL communicator then has one
rank)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2008_11607_b200 import inputs, rexi  # noqa: E402
from paper_2008_11607_b200.distributed import pole_partition, run_distributed  # noqa: E402

D = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rank, world = dist.get_rank(), dist.get_world_size()

plan = rexi.Plan(D, tau, tol=1e-12, device=local)
b, e = pole_partition(plan.n_poles, world, rank)
state = [torch.from_numpy(x.copy()).to(dev) for x in inputs.gaussian_scenario(D)]
energy0 = sum(float((x * x).sum()) for x in state)
run_distributed(plan, 1, *[x.clone() for x in state], spectral=True)   # warm-up (graphs, NCCL)
dist.barrier()
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
run_distributed(plan, steps, *state, spectral=True)
t1.record()
torch.cuda.synchronize()
ms = torch.tensor([t0.elapsed_time(t1) / steps], device=dev)
dist.all_reduce(ms, op=dist.ReduceOp.MAX)
energy = sum(float((x * x).sum()) for x in state)
if rank == 0:
    units = plan.n_poles * D * D
    print(f"D={D} tau={tau} poles={plan.n_poles} ranks={world} (rank 0: poles [{b}, {e})): "
          f"{ms.item():.3f} ms/step, {units / (ms.item() / 1e3):.3e} pole-gridpoint solves/s; "
          f"after T = {steps * tau:g}: energy drift {abs(energy - energy0) / energy0:.2e}")
dist.destroy_process_group()
