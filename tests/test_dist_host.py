"""Host logic of the distributed LDL^T (paper_2605_13736_b200.dist, SURVEY §8(f)
NEXT-4) on CPU: the 1-D block-cyclic panel map covers every panel exactly once,
and the collectives wrapper (gloo, world_size 2, CPU tensors) broadcasts and
sums as the panel loop needs.  The device arithmetic is covered by
tests/test_gpu_dist.py."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_13736_b200 import dist as pdist


@pytest.mark.parametrize("N,world", [(1, 1), (64, 2), (700, 2), (1000, 3), (8192, 8)])
def test_block_cyclic_map_covers_every_panel_once(N, world):
    npanel = -(-N // pdist.DB)
    owned = [pdist.local_panels(npanel, r, world) for r in range(world)]
    flat = sorted(sum(owned, []))
    assert flat == list(range(npanel))
    for r in range(world):
        assert all(pdist.panel_owner(g, world) == r for g in owned[r])
    spans = [pdist.panel_span(g, N) for g in range(npanel)]
    assert spans[0][0] == 0 and sum(w for _, w in spans) == N
    assert all(spans[g][0] + spans[g][1] == spans[g + 1][0] for g in range(npanel - 1))
    assert all(1 <= w <= pdist.DB for _, w in spans)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = pdist._Comm()
    t = torch.full((5,), float(rank + 1), dtype=torch.float64)
    c.allsum(t)
    b = torch.arange(3, dtype=torch.float64) * (10 if rank == 1 else 0)
    c.bcast(b, 1)
    if rank == 0:
        q.put((t.tolist(), b.tolist(), c.world, c.stage))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_comm_two_rank_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, b, world, stage = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert t == [3.0] * 5 and b == [0.0, 10.0, 20.0] and world == 2 and stage
