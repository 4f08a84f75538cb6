"""The pole-parallel multi-rank step (S3 + S4) through the REAL CUDA path:
two processes, each running rexi_apply_partial on its pole block through librexi.so, combined
by the one all-reduce of distributed.apply_distributed — compared with the ORACLE (not with
the library's own rexi_apply). The box has one GPU, so both ranks share cuda:0 and the
all-reduce runs over gloo (host side): no kernel of one rank waits on the other rank, so this
checks the control flow and the numbers, not NCCL's transport (bench.py --gpus N does that)."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, D, tau, steps, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2008_11607_b200 import build
        build.build()
        from paper_2008_11607_b200 import inputs, rexi
        from paper_2008_11607_b200.distributed import apply_distributed, run_distributed
        torch.cuda.set_device(0)
        p = rexi.Plan(D, tau, tol=1e-12, device=0)
        f = [torch.from_numpy(x).cuda() for x in inputs.white_noise(D, seed=61)]
        one = apply_distributed(p, *f).cpu().numpy()
        g = [x.clone() for x in f]
        run_distributed(p, steps, *g)
        multi = np.stack([x.cpu().numpy() for x in g])
        spec = [x.clone() for x in f]
        run_distributed(p, steps, *spec, spectral=True)
        multi_spec = np.stack([x.cpu().numpy() for x in spec])
        if rank == 0:
            q.put((one, multi, multi_spec, p.info["h"], p.info["M"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_two_rank_cuda_partial_vs_oracle(world):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import lrsw
    from paper_2008_11607_b200 import inputs
    D, tau, steps = 64, 1.0, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, D, tau, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    one, multi, multi_spec, h, M = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    f = inputs.white_noise(D, seed=61)
    ref = np.stack(lrsw.rexii_step(*f, tau, h, M))
    assert np.linalg.norm(one - ref) / np.linalg.norm(ref) < 1e-12
    g = f
    for _ in range(steps):
        g = lrsw.rexii_step(*g, tau, h, M)
    ref = np.stack(g)
    assert np.linalg.norm(multi - ref) / np.linalg.norm(ref) < 1e-12
    assert np.linalg.norm(multi_spec - ref) / np.linalg.norm(ref) < 1e-12


def _nccl_worker(port, D, tau, steps, log, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["NCCL_DEBUG"] = "INFO"
    os.environ["NCCL_DEBUG_SUBSYS"] = "INIT,COLL"
    os.environ["NCCL_DEBUG_FILE"] = log
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2008_11607_b200 import inputs, rexi
        from paper_2008_11607_b200.distributed import apply_distributed, run_distributed
        p = rexi.Plan(D, tau, tol=1e-12, device=0)
        f = [torch.from_numpy(x).cuda() for x in inputs.white_noise(D, seed=67)]
        one = apply_distributed(p, *f).cpu().numpy()
        spec = [x.clone() for x in f]
        run_distributed(p, steps, *spec, spectral=True)
        q.put((dist.get_backend(), one, np.stack([x.cpu().numpy() for x in spec]), p.info["h"], p.info["M"]))
    finally:
        dist.destroy_process_group()


def test_nccl_world1_collective_path_vs_oracle(tmp_path):
    """The S4 code path with the NCCL backend on the one GPU of the box: world size 1, so the
    all-reduce is NCCL's single-rank copy (no rank waits on another), but the communicator is
    initialised and every all_reduce of apply_distributed / run_distributed(spectral=True) is
    enqueued through NCCL on the step's stream; the result is compared with the oracle and the
    NCCL log must show the communicator's INIT and the AllReduce calls."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import lrsw
    from paper_2008_11607_b200 import build, inputs
    build.build()
    D, tau, steps = 64, 1.0, 2
    log = str(tmp_path / "nccl.%h.%p.log")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nccl_worker, args=(_free_port(), D, tau, steps, log, q))
    pr.start()
    backend, one, multi_spec, h, M = q.get(timeout=600)
    pr.join(timeout=600)
    assert pr.exitcode == 0
    assert backend == "nccl"
    text = "".join(open(os.path.join(tmp_path, n)).read() for n in os.listdir(tmp_path) if n.startswith("nccl."))
    assert "Init COMPLETE" in text or "Init" in text, text[-2000:]
    assert "AllReduce" in text, text[-2000:]
    f = inputs.white_noise(D, seed=67)
    ref = np.stack(lrsw.rexii_step(*f, tau, h, M))
    assert np.linalg.norm(one - ref) / np.linalg.norm(ref) < 1e-12
    g = f
    for _ in range(steps):
        g = lrsw.rexii_step(*g, tau, h, M)
    ref = np.stack(g)
    assert np.linalg.norm(multi_spec - ref) / np.linalg.norm(ref) < 1e-12
