"""CPU, world_size 2 over gloo: the sharding bench.py uses (dist.setup /
shard_seeds / allmax / allsum / gather_objects), checked against the
one-GPU batch (no GPU; the data path has no collective)."""
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
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2110_03636_b200 import acopf
    from paper_2110_03636_b200 import dist as hd
    w, r, _ = hd.setup("gloo")
    strong = hd.shard_seeds(7, w, r, scaling="strong")      # 7 systems over 2 ranks
    weak = hd.shard_seeds(3, w, r, scaling="weak")
    systems = [acopf.generate(40, 7, s) for s in strong]
    m = hd.allmax(10.0 * (r + 1), w)
    tot = hd.allsum(len(systems), w)
    gathered = hd.gather_objects([float(x.r_y[0]) for x in systems], w)
    hd.barrier(w)
    q.put((r, strong, weak, m, tot, gathered))
    import torch.distributed as dist
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
    (r0, s0, w0, m0, t0, g0), (r1, s1, w1, m1, t1, g1) = res
    from paper_2110_03636_b200 import acopf
    from paper_2110_03636_b200 import dist as hd
    # strong: contiguous blocks whose union is exactly the one-GPU batch
    assert s0 + s1 == hd.shard_seeds(7, 1, 0) == list(range(7, 14))
    assert (len(s0), len(s1)) == (4, 3)
    # weak: disjoint full batches
    assert len(w0) == len(w1) == 3 and set(w0).isdisjoint(w1)
    assert m0 == m1 == 20.0
    assert t0 == t1 == 7
    # the systems the ranks solved are the one-GPU batch's systems
    one = [float(x.r_y[0]) for x in acopf.batch(40, 7, seed=7)]
    assert g0 == g1 and g0[0] + g0[1] == one


def test_shard_range_covers_batch():
    from paper_2110_03636_b200 import dist as hd
    for n in (1, 7, 256):
        for g in (1, 2, 3, 4, 8):
            parts = [hd.shard_range(n, g, r) for r in range(g)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1
