"""Peer-memory all-gather of the sharded H_eff output (tci_heff_apply_gather;
SURVEY 8(e)), on one GPU: P ranks are emulated by P contexts,
each on its own stream, whose "peer" buffers are the other contexts' device
buffers (the pointer tables tci_gather_register takes; on a multi-GPU box they
come from CUDA IPC mappings). The steps run concurrently on the streams, so
the flag barriers and the remote stores of the Ozaki CRT epilogue (or the
push kernel of the DMMA path) are exercised exactly as across GPUs. Every
rank's gathered buffer must equal the unsharded apply bitwise (per-element
summation order does not depend on the shard), and sampled rows the oracle."""
import numpy as np
import pytest
import torch

import paper_2512_23917_b200 as tci
import synth
from conftest import rel_frob
from paper_2512_23917_b200.sharding import PeerGatherHeff, slice_environment

pytestmark = pytest.mark.gpu


def _run(chi, d, D, P, algo, steps=3, seed=91):
    inp = synth.heff_inputs(chi, d, D, "c128", seed, "heisenberg", device="cuda")
    L, W1, W2, R, psi = (inp[k] for k in ("L", "W1", "W2", "R", "psi"))
    code = {"ozaki": tci.TCI_GEMM_OZAKI_INT8, "dmma3m": tci.TCI_GEMM_DMMA_3M}[algo]
    ref_ctx = tci.Context(0)
    ref_ctx.set_gemm_algorithm(code)
    ref = ref_ctx.heff_apply(L, W1, W2, R, psi)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [tci.Context(0, streams[r]) for r in range(P)]
    for c in ctxs:
        c.set_gemm_algorithm(code)
    fulls = [torch.full((chi, d, d, chi), float("nan"), dtype=torch.complex128, device="cuda") for _ in range(P)]
    flags = [torch.zeros(P, dtype=torch.int32, device="cuda") for _ in range(P)]
    table = ([f.data_ptr() for f in fulls], [g.data_ptr() for g in flags])
    shs = [PeerGatherHeff(ctxs[r], slice_environment(L, P, r), W1, W2, R, P, r, peers=table, full=fulls[r],
                          flags=flags[r]) for r in range(P)]
    # one plain slab apply per rank first: every chain kernel is loaded before
    # a barrier spins (CUDA lazy loading cannot load a kernel on this device
    # while another stream's barrier kernel waits for it -- only the emulation
    # shares one device; across GPUs each rank loads on its own)
    for r in range(P):
        ctxs[r].heff_apply(shs[r].L, W1, W2, R, psi)
    torch.cuda.synchronize()
    for _ in range(steps):
        for r in range(P):
            shs[r].apply(psi)          # enqueued on rank r's stream; the ranks run concurrently
    torch.cuda.synchronize()
    status = [c.gather_status() for c in ctxs]
    launches = [c.launch_count() for c in ctxs]
    for c in ctxs + [ref_ctx]:
        c.close()
    return inp, ref, fulls, flags, status, launches


@pytest.mark.parametrize("P", [2, 4])
def test_peer_gather_ozaki_fused_epilogue(oracle_mod, P):
    """chi = 1024 (config 2 shape): both GEMMs take the Ozaki path per rank, so
    the gather rides in the CRT epilogue's remote stores."""
    chi = 1024
    inp, ref, fulls, flags, status, launches = _run(chi, 2, 5, P, "ozaki")
    assert status == [0] * P
    for r in range(P):
        assert torch.equal(fulls[r], ref), f"rank {r} gathered buffer differs from the unsharded apply"
        assert flags[r].cpu().tolist() == [6] * P          # 3 steps x (entry + exit) epochs
    rows = [0, chi // P - 1, chi // P, chi - 1]
    n = {k: v.cpu().numpy() for k, v in inp.items()}
    want = oracle_mod.heff_rows(n["L"], n["W1"], n["W2"], n["R"], n["psi"], rows)
    got = fulls[P - 1].cpu().numpy()[rows]
    assert rel_frob(got, want) <= 1e-12


@pytest.mark.parametrize("P", [2, 3])
def test_peer_gather_dmma_push(P):
    """DMMA GEMM4 (and chi not a tile multiple): the slab is pushed to the
    peers by the copy kernel after the chain."""
    chi = 96 * P
    inp, ref, fulls, flags, status, launches = _run(chi, 2, 5, P, "dmma3m", steps=2)
    assert status == [0] * P
    for r in range(P):
        assert torch.equal(fulls[r], ref)
        assert flags[r].cpu().tolist() == [4] * P


def test_peer_gather_single_rank_is_plain_apply():
    inp = synth.heff_inputs(40, 2, 5, "c128", 5, "heisenberg", device="cuda")
    ctx = tci.Context(0)
    sh = PeerGatherHeff(ctx, inp["L"], inp["W1"], inp["W2"], inp["R"], 1, 0)
    out = sh.apply(inp["psi"])
    ref = ctx.heff_apply(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"])
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    ctx.close()


def test_peer_gather_errors():
    ctx = tci.Context(0)
    f = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(tci.TciError):
        ctx.gather_register(9, 0, [f.data_ptr()] * 9, [f.data_ptr()] * 9)     # > 8 ranks
    with pytest.raises(tci.TciError):
        ctx.gather_register(2, 2, [f.data_ptr()] * 2, [f.data_ptr()] * 2)     # rank out of range
    # registered buffer mismatch
    inp = synth.heff_inputs(16, 2, 5, "c128", 5, "heisenberg", device="cuda")
    fulls = [torch.empty(16, 2, 2, 16, dtype=torch.complex128, device="cuda") for _ in range(2)]
    ctx.gather_register(2, 0, [x.data_ptr() for x in fulls], [f.data_ptr(), f.data_ptr()])
    other = torch.empty_like(fulls[0])
    with pytest.raises(tci.TciError):
        ctx.heff_apply_gather(slice_environment(inp["L"], 2, 0), inp["W1"], inp["W2"], inp["R"], inp["psi"], other)
    ctx.close()
    # IPC handle of a torch allocation: 64 bytes + the offset inside its allocation
    x = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    h, off = tci.tci_ipc_handle(x.data_ptr() + 4096)
    assert len(h) == 64 and off >= 4096


def test_lanes_streaming_applies():
    """tci_copy_async / tci_lane_record / tci_lane_wait: a stream of applies
    with double-buffered device inputs (each step's inputs copied on lane 1
    while the previous step computes, results copied out on lane 2) returns
    exactly the per-step results of plain synchronous applies."""
    ctx = tci.Context(0)
    chi, steps = 48, 5
    KEYS = ("L", "W1", "W2", "R", "psi")
    hosts = [synth.heff_inputs(chi, 2, 5, "c128", 200 + i, "heisenberg") for i in range(steps)]
    hosts = [{k: v.pin_memory() for k, v in h.items()} for h in hosts]
    refs = [ctx.heff_apply(*(h[k].cuda() for k in KEYS)).cpu() for h in hosts]
    bufs = [{k: torch.empty_like(v, device="cuda") for k, v in hosts[0].items()} for _ in range(2)]
    outs = [torch.empty(chi, 2, 2, chi, dtype=torch.complex128, device="cuda") for _ in range(2)]
    houts = [torch.empty(chi, 2, 2, chi, dtype=torch.complex128).pin_memory() for _ in range(steps)]
    IN, DONE, OUT = 0, 2, 4

    def load(i, b):
        ctx.lane_wait(1, DONE + b)
        for k in KEYS:
            ctx.copy_async(hosts[i][k], bufs[b][k], 1)
        ctx.lane_record(1, IN + b)
    torch.cuda.synchronize()
    load(0, 0)
    for i in range(steps):
        b = i % 2
        if i + 1 < steps:
            load(i + 1, 1 - b)
        ctx.lane_wait(0, IN + b)
        ctx.lane_wait(0, OUT + b)
        ctx.heff_apply(*(bufs[b][k] for k in KEYS), out=outs[b])
        ctx.lane_record(0, DONE + b)
        ctx.lane_wait(2, DONE + b)
        ctx.copy_async(outs[b], houts[i], 2)
        ctx.lane_record(2, OUT + b)
    ctx.lane_wait(0, OUT + (steps - 1) % 2)
    ctx.synchronize()
    torch.cuda.synchronize()
    for i in range(steps):
        assert torch.equal(houts[i], refs[i]), f"step {i}"
    with pytest.raises(tci.TciError):
        ctx.lane_record(3, 0)
    with pytest.raises(tci.TciError):
        ctx.lane_wait(0, 16)
    ctx.close()


def test_peer_gather_bench_workload_p2():
    """The bench workload (chi = 4096, d = 2, D = 5, Ozaki) gathered over
    emulated peer memory by two ranks: bitwise the unsharded apply."""
    inp, ref, fulls, flags, status, launches = _run(4096, 2, 5, 2, "ozaki", steps=1, seed=6)
    assert status == [0, 0]
    for r in range(2):
        assert torch.equal(fulls[r], ref)
    del inp, ref, fulls
    torch.cuda.empty_cache()
