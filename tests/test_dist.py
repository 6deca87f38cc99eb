"""The data-parallel exchange (R11) with world_size 2 over gloo on CPU:
each rank holds its own sensitivities c^(r); the all-reduce merges them to the mean;
every rank then runs libgact's greedy allocator and obtains identical bits, equal to the
oracle's allocation on the merged vector; a disagreement is detected."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import oracle
    import paper_2206_11357_b200 as gact
    import synth
    from paper_2206_11357_b200 import dist as gdist
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        specs = synth.workload_specs("resnet50")
        D = np.array([s.numel for s in specs], dtype=np.int64)
        c_local = synth.sensitivities(specs, seed=7, rank=rank + 1)
        c = gdist.merge_sensitivities(c_local)
        B = int(4 * D.sum())
        bits = gact.allocate_bits(c, D, B)
        gdist.assert_same_allocation(bits)
        # the oracle on the merged vector (computed here from both ranks' inputs)
        both = [synth.sensitivities(specs, seed=7, rank=r + 1) for r in range(world)]
        merged = sum(both) / world
        rc, ref = oracle.allocate_bits(merged, D, [1, 2, 4, 8], B)
        # a deliberately different allocation on rank 1 must be caught
        caught = False
        try:
            gdist.assert_same_allocation(bits if rank == 0 else bits[::-1].copy())
        except RuntimeError:
            caught = True
        q.put((rank, c.tolist(), bits.tolist(), rc, ref.tolist(), float(np.max(np.abs(c - merged) / merged)), caught))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, "error", repr(e)))


@pytest.mark.timeout(300)
def test_two_rank_merge_and_allocation():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res = sorted(res, key=lambda r: r[0])
    for r in res:
        assert r[1] != "error", r
    (_, c0, b0, rc0, ref0, err0, caught0), (_, c1, b1, rc1, ref1, err1, caught1) = res
    assert c0 == c1                      # identical merged vector on both ranks
    assert b0 == b1                      # identical allocation
    assert rc0 == 0 and b0 == ref0       # == the oracle's allocation of the merged vector
    assert err0 < 1e-12 and err1 < 1e-12
    assert caught0 and caught1           # disagreement detected on every rank
