"""bench.py's N > 1 path ("replicas only") on CPU with the gloo
backend, world_size 2: the whole-job value counts every rank's points and
divides by the slowest rank's time (max over ranks)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    local_ms = [40.0, 50.0][rank]  # rank 1 is the slowest
    value, max_ms = bench.job_value(1_000_000, 5, local_ms, dist, "cpu")
    dist.barrier()
    q.put((rank, value, max_ms))
    dist.destroy_process_group()


def test_job_value_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, value, max_ms in res:
        assert max_ms == 50.0
        assert value == pytest.approx(1_000_000 * 5 * 2 / 0.050)


def test_job_value_single():
    import bench
    v, ms = bench.job_value(10, 2, 4.0)
    assert ms == 4.0 and v == pytest.approx(10 * 2 / 0.004)
