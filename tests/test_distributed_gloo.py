"""Host logic of the pole-parallel multi-GPU step (S4) on CPU with the gloo
backend, world size 2 (and 3): the pole partition and the one all-reduce compose to the
single-process oracle result. The per-rank compute here is the oracle's partial pole sum
(tests may use the oracle); on GPUs it is rexi_apply_partial."""
import os
import socket

import numpy as np
import pytest

from paper_2008_11607_b200.distributed import pole_partition


def test_pole_partition_covers_and_balances():
    for n in (1, 7, 47, 604, 4583, 36432):
        for P in (1, 2, 3, 4, 8):
            if P > n:
                continue
            ranges = [pole_partition(n, P, r) for r in range(P)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        pole_partition(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, D, tau, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import coeffs as C
        from oracle import lrsw
        from paper_2008_11607_b200 import inputs
        from paper_2008_11607_b200.distributed import pole_parallel_step
        f = inputs.white_noise(D)
        M = C.M_lrsw(D, tau, 0.5, 1e-12)
        n, al, c1, c2, g = C.rexii_terms(0.5, M).half()
        F = lrsw.spectral_fields(*f)
        ml, mk = lrsw.all_modes(D)

        def partial(b, e, out):
            acc = lrsw.rexii_pole_sum(D, tau, F[ml, mk], ml, mk, al[b:e], c1[b:e], c2[b:e], g[b:e])
            A = np.zeros((D, D, 3), complex)
            A[ml, mk] = acc
            for c in range(3):
                out[c] = torch.from_numpy(lrsw.idft2_real(A[..., c]))

        out = torch.zeros((3, D, D), dtype=torch.float64)
        pole_parallel_step(partial, len(g), out)
        if rank == 0:
            q.put(out.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_pole_parallel_allreduce_matches_single(world, oracle_lib):
    import multiprocessing as mp
    from oracle import lrsw
    from paper_2008_11607_b200 import inputs
    D, tau = 16, 1.0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, D, tau, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    from oracle import coeffs as C
    M = C.M_lrsw(D, tau, 0.5, 1e-12)
    ref = lrsw.rexii_step(*inputs.white_noise(D), tau, 0.5, M)
    err = np.linalg.norm(got - np.stack(ref)) / np.linalg.norm(np.stack(ref))
    assert err < 1e-14
