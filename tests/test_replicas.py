"""Multi-GPU = replicas only: the N > 1 host logic of bench.py, run as world_size-2
`gloo` process groups on CPU (the driver's N-GPU runs use the same functions over NCCL)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    el_ms = [120.0, 150.0][rank]          # device time of this rank's K steps

    def reduce_max(x):
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    el_max, value = bench.aggregate_ranks(el_ms, 5, world, reduce_max)
    seed = bench.replica_seed(0, rank)
    _, u0, _ = synth.problem_inputs(2, seed, 63)
    q.put((rank, el_max, value, seed, float(np.abs(u0).sum())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, m0, v0, s0, a0), (r1, m1, v1, s1, a1) = out
    assert m0 == m1 == 150.0                       # job time = max over ranks
    assert v0 == v1 == pytest.approx(2 * 5 / 0.150)   # all ranks' steps / max time (weak scaling)
    assert s0 != s1 and a0 != a1                   # independent problems per replica
