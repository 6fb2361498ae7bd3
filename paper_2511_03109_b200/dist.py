"""Multi-GPU plumbing for the row-sharded apply.

Each rank owns a contiguous range of leaf row clusters (tree order, balanced
by near-field entries; host/build.cpp); x is replicated. Two exchanges:

* symmetric near storage (the default in snapshot mode): a rank stores the
  near pairs whose owner leaf it holds, so its transposed products reach
  rows of other ranks. Each rank produces a full-length partial y in tree
  order (`phm_apply_partial_device`) and the partials are summed with one
  all-reduce (`PartialSum`);
* full near storage: each rank computes exactly its rows; the row blocks are
  all-gathered (`RowGather`, a padded all_gather_into_tensor).

NCCL over NVLink on GPUs, gloo in the CPU tests; then the un-permute to the
original point order.
"""
from __future__ import annotations

from typing import List, Sequence


def row_counts(rows: int, group=None) -> List[int]:
    """All ranks' row counts (all_gather of one int64)."""
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([rows], dtype=torch.int64, device=dev)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [int(v.item()) for v in out]


class RowGather:
    """Reusable buffers for the padded all-gather of per-rank row blocks."""

    def __init__(self, counts: Sequence[int], m: int = 1, device="cpu", dtype=None):
        import torch

        self.counts = list(counts)
        self.world = len(self.counts)
        self.maxr = max(self.counts) if self.counts else 0
        self.m = m
        dtype = dtype or torch.float64
        self.send = torch.zeros((m, self.maxr), dtype=dtype, device=device)
        self.recv = torch.empty((self.world, m, self.maxr), dtype=dtype, device=device)
        self.out = torch.empty((m, sum(self.counts)), dtype=dtype, device=device)

    def gather(self, yrows, group=None):
        """yrows: (m, rows_local) tensor (column-major rows x m from the C
        ABI). Returns (m, n) in tree order."""
        import torch.distributed as dist

        r = yrows.shape[-1]
        if yrows.data_ptr() != self.send.data_ptr():
            self.send[:, :r].copy_(yrows)
        dist.all_gather_into_tensor(self.recv.view(-1), self.send.view(-1), group=group)
        off = 0
        for k in range(self.world):
            c = self.counts[k]
            self.out[:, off: off + c].copy_(self.recv[k, :, :c])
            off += c
        return self.out


class PartialSum:
    """Reusable buffer for summing per-rank partial y vectors (tree order)."""

    def __init__(self, n: int, m: int = 1, device="cpu", dtype=None):
        import torch

        self.buf = torch.zeros((m, n), dtype=dtype or torch.float64, device=device)

    def reduce(self, group=None):
        """Sums the ranks' partials in place (all-reduce); returns (m, n)."""
        import torch.distributed as dist

        dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=group)
        return self.buf
