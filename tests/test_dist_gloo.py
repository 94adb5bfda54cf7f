"""Multi-rank (world_size 2, gloo, CPU) test of the sharded-run merge.

Each rank takes its replica shard of one run (replica_offset/replicas_total
semantics: trajectory g = point * replicas_total + replica), computes that
shard's exact moments (here with the oracle standing in for the GPU kernel,
which needs a device), and merges with paper_1010_2438_b200.dist.
allreduce_stats.  The merged moments must equal the unsharded run's
exactly, including sumsq carries across the 64-bit word boundary."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import workloads as w
    from paper_1010_2438_b200.dist import allreduce_stats, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        desc, sweep = w.config("C3")[0], w.mm_sweep(3, 2)
        R_local = 5
        off, R_tot = shard_range(R_local, rank)
        P = len(sweep["values"])
        g = [p * R_tot + off + r for p in range(P) for r in range(R_local)]
        res = oracle.simulate(desc, R_tot, 10.0, 0.5, 1, sweep=sweep, g_list=g, want_traj=False)
        c = torch.from_numpy(res["count"].copy())
        s = torch.from_numpy(res["sum"].copy())
        q2 = torch.from_numpy(res["sumsq"].view(np.int64).copy())
        allreduce_stats(c, s, q2)
        # carry check: two ranks each adding 2^64 - 1 in the low word
        big = torch.tensor([[-1, 0]], dtype=torch.int64)
        allreduce_stats(torch.zeros(1, dtype=torch.int64), torch.zeros(1, dtype=torch.int64), big)
        if rank == 0:
            q.put((c.numpy(), s.numpy(), q2.numpy(), big.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_merge_equals_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    c, s, q2, big = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    import oracle
    import workloads as w
    whole = oracle.simulate(w.config("C3")[0], 10, 10.0, 0.5, 1, sweep=w.mm_sweep(3, 2), want_traj=False)
    assert (c == whole["count"]).all()
    assert (s == whole["sum"]).all()
    assert (q2.view(np.uint64) == whole["sumsq"]).all()
    # (2^64 - 1) * 2 = 2^65 - 2 -> lo = 2^64 - 2, hi = 1
    assert big.view(np.uint64)[0, 0] == 2**64 - 2 and big[0, 1] == 1
