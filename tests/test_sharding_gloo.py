"""Multi-rank host logic of the sharded H_eff apply on CPU:
world_size 2 with the gloo backend. Each rank takes its slab of L with the
product's `slice_environment`, computes its output slab (here with the oracle,
since there is no GPU: test infrastructure), and the slabs are all-gathered
in rank order; the result must equal the unsharded apply bitwise (the per-row
summation order is shard independent)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2512_23917_b200.sharding import shard_bounds, slice_environment
        inp = synth.heff_inputs(12, 2, 5, "c128", 77, "heisenberg")
        Ls = slice_environment(inp["L"], world, rank)
        lo, hi = shard_bounds(12, world, rank)
        part = oracle.heff(Ls.numpy(), inp["W1"].numpy(), inp["W2"].numpy(), inp["R"].numpy(),
                           inp["psi"].numpy(), threads=1)
        t = torch.from_numpy(np.ascontiguousarray(part))
        gathered = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        full = torch.cat(gathered, dim=0).numpy()
        if rank == 0:
            ref = oracle.heff(*(inp[k].numpy() for k in ("L", "W1", "W2", "R", "psi")), threads=1)
            q.put((bool(np.array_equal(full, ref)), (lo, hi), full.shape))
    finally:
        dist.destroy_process_group()


def test_sharded_apply_gloo_world2():
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ok, bounds, shape = q.get(timeout=10)
    assert ok and bounds == (0, 6) and shape == (12, 2, 2, 12)


def test_shard_bounds():
    from paper_2512_23917_b200.sharding import shard_bounds
    assert [shard_bounds(4096, 8, r) for r in (0, 7)] == [(0, 512), (3584, 4096)]
    with pytest.raises(ValueError):
        shard_bounds(10, 4, 0)
