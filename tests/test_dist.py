"""CPU (gloo, world_size 2): the N>1 host path -- partition + the single
end-of-run combine -- with the oracle standing in for each rank's device
sieve.  Also checks that the sharded result equals the unsharded one."""
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


def _worker(rank, world, port, L, R, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port
    from paper_2310_17746_b200 import dist as wsdist
    from paper_2310_17746_b200.wheelsieve import Checks
    port_ = Port()

    def local_fn(lo, hi):
        r = port_.range(lo, hi)
        return Checks(r["count"], r["sum"], r["xor"], r["largest"])

    c = wsdist.sharded_count(L, R, rank, world, local_fn=local_fn, segment_slots=1 << 12)
    m = wsdist.max_over_ranks(float(rank))
    s = wsdist.sum_over_ranks(rank + 1)
    q.put((rank, c.count, c.sum, c.xor, c.largest, m, s))
    dist.destroy_process_group()


@pytest.mark.parametrize("L,R", [(0, 3_000_001), (10**12, 10**12 + 2_000_003), (1, 30)])
def test_sharded_count_gloo(port, L, R):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, p, L, R, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    ref = port.range(L, R)
    for rank, count, s, x, lg, m, sm in res:
        assert (count, s, x, lg) == (ref["count"], ref["sum"], ref["xor"], ref["largest"])
        assert m == world - 1 and sm == world * (world + 1) // 2
