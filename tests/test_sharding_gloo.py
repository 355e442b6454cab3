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


def _handle_worker(rank, world, port, q):
    """Host logic of the peer-memory gather setup: IPC handles exchanged with
    all_gather_object (gloo here, the same call over NCCL on the GPU box),
    pointer tables built in rank order with this rank's own buffers."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_23917_b200.sharding import peer_pointer_table
        mine = ((b"F%d" % rank + bytes(62), 4096 * rank), (b"G%d" % rank + bytes(62), 64 * rank))
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        opened = []

        def opener(h, off):   # stands in for tci_ipc_open: a distinct fake pointer per (handle, offset)
            p = (1 << 40) + int(h[1:2].decode()) * (1 << 32) + (1 << 20) * (h[:1] == b"G") + off
            opened.append(p)
            return p
        own = (7000 + rank, 9000 + rank)
        fulls, flags, op = peer_pointer_table(rank, allh, own, opener)
        q.put((rank, fulls, flags, op, opened))
    finally:
        dist.destroy_process_group()


def test_peer_gather_handle_exchange_gloo_world3():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_handle_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = {}
    for _ in range(world):
        r, fulls, flags, op, opened = q.get(timeout=10)
        res[r] = (fulls, flags, op, opened)
    for r in range(world):
        fulls, flags, op, opened = res[r]
        assert len(fulls) == len(flags) == world
        assert fulls[r] == 7000 + r and flags[r] == 9000 + r          # own buffers, unmapped
        for i in range(world):
            if i != r:                                                 # peer i's mapping + its offset
                assert fulls[i] == (1 << 40) + i * (1 << 32) + 4096 * i
                assert flags[i] == (1 << 40) + i * (1 << 32) + (1 << 20) + 64 * i
        assert sorted(op) == sorted(opened) and len(op) == 2 * (world - 1)


def _agree_worker(rank, world, port, q, fail_stage):
    """PeerGatherHeff setup when one rank fails (IPC export or mapping): every
    rank must raise at the same point (agreement by all-reduce MIN) instead of
    leaving the others blocked in the handle exchange; mapped handles are closed."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2512_23917_b200 as tci
        from paper_2512_23917_b200.sharding import PeerGatherHeff
        closed = []

        def fake_handle(ptr):
            if fail_stage == "export" and rank == 1:
                raise RuntimeError("no IPC on this rank")
            return (b"H%d" % rank + bytes(62), 0)

        def fake_open(h, off):
            if fail_stage == "map" and rank == 1:
                raise RuntimeError("cannot map")
            return 4096 + int(h[1:2].decode())
        tci.tci_ipc_handle, tci.tci_ipc_open = fake_handle, fake_open
        tci.tci_ipc_close = lambda p: closed.append(p)

        def exchange(obj):
            allo = [None] * world
            dist.all_gather_object(allo, obj)
            return allo

        def agree(ok):
            t = torch.tensor([1 if ok else 0], dtype=torch.int32)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            return bool(t.item())
        L = torch.zeros(4, 2, 3, dtype=torch.complex128)
        W = torch.zeros(2, 2, 2, 2, dtype=torch.complex128)
        R = torch.zeros(4, 2, 4, dtype=torch.complex128)
        try:
            PeerGatherHeff(None, L, W, W, R, world, rank, exchange=exchange, agree=agree)
            q.put((rank, "no error", closed))
        except RuntimeError as e:
            q.put((rank, str(e), closed))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("stage", ["export", "map"])
def test_peer_gather_setup_failure_agreement_gloo(stage):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, q, stage)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, "a rank hung or crashed"
    res = dict((r, (msg, closed)) for r, msg, closed in (q.get(timeout=10) for _ in range(2)))
    word = "export" if stage == "export" else "mapping"
    assert all(word in res[r][0] for r in (0, 1)), res
    if stage == "map":
        assert res[0][1] == [4097] * 2 and res[1][1] == []    # rank 0 unmapped what it had opened
