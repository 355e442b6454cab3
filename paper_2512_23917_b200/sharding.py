"""Output-leg sharding of H_eff.psi across ranks.

Rank r owns the contiguous slab b in [lo_r, hi_r) of the output's slowest
bond; it holds L[:, :, lo_r:hi_r] and the full psi, W1, W2, R, computes its
out slab with tci_heff_apply and the slabs are concatenated in rank order by
one all-gather (tci_allgather, NCCL) -- which yields the full row-major
output without a post-permute because b is the slowest leg. The per-element
summation order does not depend on the shard, so the gathered result is
bitwise equal to the unsharded one.

Host-side logic only; the compute is the C ABI.
"""
from __future__ import annotations

from typing import Tuple


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous equal slabs of the leg of extent n (all-gather needs equal counts)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"rank {rank} of {world}")
    if n % world:
        raise ValueError(f"leg extent {n} is not divisible by {world} ranks")
    s = n // world
    return rank * s, (rank + 1) * s


def slice_environment(L, world: int, rank: int):
    """L[a, w, b] -> this rank's contiguous L[:, :, lo:hi] (setup, not per step)."""
    lo, hi = shard_bounds(L.shape[2], world, rank)
    return L[:, :, lo:hi].contiguous()


class ShardedHeff:
    """One rank of the sharded apply: out_full = allgather(heff(L_r, W1, W2, R, psi))."""

    def __init__(self, ctx, L_slice, W1, W2, R, world: int, rank: int, out_full=None):
        import torch
        self.ctx, self.world, self.rank = ctx, world, rank
        self.L, self.W1, self.W2, self.R = L_slice, W1, W2, R
        chi_lo = L_slice.shape[2]
        d = W1.shape[2]
        chi_ro = R.shape[2]
        dev = L_slice.device
        self.out = torch.empty((chi_lo, d, d, chi_ro), dtype=L_slice.dtype, device=dev)
        if world > 1:
            self.full = out_full if out_full is not None else torch.empty(
                (chi_lo * world, d, d, chi_ro), dtype=L_slice.dtype, device=dev)
        else:
            self.full = self.out

    def apply(self, psi):
        self.ctx.heff_apply(self.L, self.W1, self.W2, self.R, psi, out=self.out)
        if self.world > 1:
            self.ctx.allgather(self.out, self.full)
        return self.full


def peer_pointer_table(rank: int, handles, own, opener):
    """Pointer tables for tci_gather_register from the exchanged IPC handles.

    handles: per rank (rank order) ((full_handle, full_offset), (flag_handle,
    flag_offset)), as all_gather_object returns them; own: this rank's
    (full_ptr, flag_ptr); opener(handle, offset) -> mapped pointer. Returns
    (full_ptrs, flag_ptrs, opened) -- opened lists what must be unmapped."""
    fulls, flags, opened = [], [], []
    for i, (hf, hg) in enumerate(handles):
        if i == rank:
            fulls.append(own[0])
            flags.append(own[1])
            continue
        pf, pg = opener(*hf), opener(*hg)
        opened += [pf, pg]
        fulls.append(pf)
        flags.append(pg)
    return fulls, flags, opened


class PeerGatherHeff:
    """One rank of the sharded apply with the all-gather done over peer memory
    (tci_heff_apply_gather): the GEMM4 epilogue stores every output element
    into this rank's slab of EVERY rank's `full` buffer (CUDA IPC mappings
    over NVLink), with a flag barrier around the step -- no collective call.

    exchange(obj) -> [obj of rank 0, ..., obj of rank P-1] (e.g. a wrapper of
    torch.distributed.all_gather_object); agree(ok) -> True iff every rank
    passed ok=True (an all-reduce MIN), so a failure on one rank makes every
    rank raise at the same point instead of leaving the others blocked in a
    collective. `peers` = (full_ptrs, flag_ptrs) bypasses IPC (single-process
    emulation of several ranks in tests)."""

    def __init__(self, ctx, L_slice, W1, W2, R, world: int, rank: int, exchange=None, peers=None, full=None,
                 flags=None, agree=None):
        import torch
        import paper_2512_23917_b200 as tci
        self.ctx, self.world, self.rank = ctx, world, rank
        self.L, self.W1, self.W2, self.R = L_slice, W1, W2, R
        chi_lo, d, chi_ro = L_slice.shape[2], W1.shape[2], R.shape[2]
        dev = L_slice.device
        self.full = full if full is not None else torch.empty((chi_lo * world, d, d, chi_ro),
                                                              dtype=L_slice.dtype, device=dev)
        self.flags = flags if flags is not None else torch.zeros(max(world, 1), dtype=torch.int32, device=dev)
        self._opened = []
        if world > 1:
            if peers is None:
                if exchange is None:
                    raise ValueError("PeerGatherHeff needs exchange() (or peers) for world > 1")
                agree = agree or (lambda ok: ok)
                try:
                    mine, err = (tci.tci_ipc_handle(self.full.data_ptr()),
                                 tci.tci_ipc_handle(self.flags.data_ptr())), None
                except Exception as e:   # noqa: BLE001 -- reported after the agreement
                    mine, err = None, e
                if not agree(mine is not None):
                    raise RuntimeError(f"peer gather: IPC export failed on some rank ({err})")
                allh = exchange(mine)
                opened = []

                def opener(h, off):
                    ptr = tci.tci_ipc_open(h, off)
                    opened.append(ptr)
                    return ptr
                try:
                    fulls, flg, _ = peer_pointer_table(rank, allh, (self.full.data_ptr(), self.flags.data_ptr()),
                                                       opener)
                    err = None
                except Exception as e:   # noqa: BLE001
                    err = e
                self._opened = opened
                if not agree(err is None):
                    self.close()
                    raise RuntimeError(f"peer gather: IPC mapping failed on some rank ({err})")
            else:
                fulls, flg = peers
            ctx.gather_register(world, rank, fulls, flg)
        self.out = self.full

    def apply(self, psi):
        self.ctx.heff_apply_gather(self.L, self.W1, self.W2, self.R, psi, self.full)
        return self.full

    def close(self):
        import paper_2512_23917_b200 as tci
        for p in self._opened:
            tci.tci_ipc_close(p)
        self._opened = []
