"""Multi-rank plumbing of bench.py on CPU (gloo, world_size 2): the path is
replicated per GPU (no data-path collective); the only
cross-rank operation is the max-over-ranks of the device time."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch.distributed as tdist
    import bench
    tdist.init_process_group("gloo", init_method="env://", rank=rank, world_size=ws)
    local_ms = 10.0 + 5.0 * rank
    m = bench.reduce_max(local_ms)
    rate = bench.whole_job_rate(ws, 1000, m)
    q.put((rank, m, rate, bench.dist_info()))
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.timeout(120)
def test_reduce_max_and_whole_job_rate_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    for rank, m, rate, info in res:
        assert m == 15.0                     # slowest rank
        assert rate == 2 * 1000 / 15e-3      # whole-job units / slowest time
        assert info == (2, rank, rank)
