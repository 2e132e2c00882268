"""Multi-process path on CPU: bench.py --gpus N runs N independent replicas
(the solve does not shard); its whole-job numbers are the MAX of the step
and loop times over ranks and the SUM of iterations. Exercised here with
world_size 2 over gloo."""
import os
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, cg, its = bench.combine_ranks(100.0 + rank, 1.0 + 2 * rank, 10 + rank, world, "cpu")
    q.put((rank, ms, cg, its))
    dist.barrier()
    dist.destroy_process_group()


def test_combine_ranks_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, ms, cg, its in out:
        assert ms == 101.0 and cg == 3.0 and its == 21.0


def test_combine_ranks_single():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.combine_ranks(5.0, 2.0, 7, 1, "cpu") == (5.0, 2.0, 7.0)
