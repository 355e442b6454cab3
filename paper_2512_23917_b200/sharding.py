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
