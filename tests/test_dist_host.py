"""N > 1 host logic on CPU (gloo, world_size 2): the bench's max-over-ranks timing and the
reference arm's rank-0-only rule (replicas, no data-path collective)."""
import os
import socket

import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    import torch.distributed as tdist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    t = bench.max_over_ranks(10.0 + 5.0 * rank)  # rank 1 is the slow one

    class Args:  # the reference arm returns nothing on ranks != 0
        workload = "cfg1"
        steps = 1
        warmup = 0

    ref = bench.run_reference(Args, rank, world) if rank != 0 else "skipped"
    q.put((rank, t, ref))
    tdist.barrier()
    tdist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = {r: (t, ref) for r, t, ref in out}
    assert got[0][0] == 15.0 and got[1][0] == 15.0  # every rank sees the max
    assert got[1][1] is None  # only rank 0 runs the reference arm


def test_max_over_ranks_single_process():
    import bench

    assert bench.max_over_ranks(3.5) == 3.5
