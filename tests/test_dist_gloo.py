"""Multi-process (world_size 2, gloo, CPU) coverage of the row-sharded path's host logic:
NCCL-id sharing, max-over-ranks timing, and the row partition + stage/all-gather/unpack
layout the library uses, with the oracle standing in for each
rank's rows (test-only)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import bipb_inputs as g
        import oracle
        import paper_1301_5885_b200 as bp
        from paper_1301_5885_b200 import dist as bd
        uid = bd.share_uid(lambda: bytes(range(128)), rank, world)
        assert uid == bytes(range(128))
        t = bd.max_over_ranks(10.0 + rank, world)
        assert t == 10.0 + world - 1
        p = g.sphere_problem(2, 4.0, g.helix_charges())  # N = 320
        u = g.random_vector(2 * p.n, 4)
        r0, r1 = bp.bipb_partition(p.n, world, rank)
        yi, yin = oracle.matvec_rows(p, u, np.arange(r0, r1))
        npad = -(-p.n // world)
        st = torch.from_numpy(bd.stage_rows(yi, yin, npad))
        gathered = [torch.zeros_like(st) for _ in range(world)]
        dist.all_gather(gathered, st)
        y = bd.unpack_gathered(torch.cat(gathered).numpy(), p.n, world)
        ref = oracle.matvec(p, u)
        q.put((rank, float(np.max(np.abs(y - ref))), None))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_shard_allgather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, err, exc in res:
        assert exc is None, exc
        assert err == 0.0  # rows are computed independently: bitwise identical to the full product
