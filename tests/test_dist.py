"""CPU, world_size 2 over gloo: rank sharding and the max-over-ranks timing
reduction used by bench.py (no GPU; the data path has no collective)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_03636_b200 import dist as hd
    from paper_2110_03636_b200 import acopf
    seeds = hd.shard(rank, 3)
    systems = [acopf.generate(40, 7, s) for s in seeds]
    m = hd.allmax(10.0 * (rank + 1), world)
    tot = hd.allsum(len(systems), world)
    q.put((rank, seeds, m, tot, float(systems[0].r_y[0])))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_sharding_and_max_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in range(2))
    for p in procs:
        p.join(timeout=30)
    (r0, s0, m0, t0, v0), (r1, s1, m1, t1, v1) = res
    assert set(s0).isdisjoint(s1)
    assert m0 == m1 == 20.0
    assert t0 == t1 == 6
    assert v0 != v1
