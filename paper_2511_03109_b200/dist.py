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


def nccl_comm(ctx, group=None):
    """The library's own NCCL communicator for this rank (phm_comm_create_nccl):
    rank 0's unique id is broadcast over the torch.distributed group, then
    every rank joins. The sharded step then runs both exchanges inside the
    library (phm_instantiate_apply_sharded), on the library's stream."""
    import torch.distributed as dist

    from . import Comm

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return Comm.nccl(ctx, obj[0], rank, world)


def host_allreduce_comm(group=None):
    """A library communicator whose all-reduce is torch.distributed on host
    copies (gloo): drives the library's sharded step with ranks that share
    one GPU, in tests. Synchronises the device, copies the buffer out,
    all-reduces it, copies it back."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from . import Comm

    rank, world = dist.get_rank(group), dist.get_world_size(group)

    def fn(buf, count, stream):
        torch.cuda.synchronize()
        host = torch.from_numpy(np.empty(count, dtype=np.float64))
        _memcpy(host.data_ptr(), buf, count * 8, 2)  # device -> host
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        _memcpy(buf, host.data_ptr(), count * 8, 1)  # host -> device
        # a pageable H2D cudaMemcpy may return before its DMA lands, and the
        # library's streams are non-blocking (no implicit ordering with the
        # legacy stream): wait for the device before the step continues
        torch.cuda.synchronize()

    return Comm.callback(fn, rank, world)


_CUDART = None


def _memcpy(dst, src, nbytes, kind):
    """Synchronous cudaMemcpy on raw pointers (kind 1: H2D, 2: D2H)."""
    import ctypes

    global _CUDART
    if _CUDART is None:
        _CUDART = ctypes.CDLL("libcudart.so.12")
        _CUDART.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    err = _CUDART.cudaMemcpy(dst, src, nbytes, kind)
    if err != 0:
        raise RuntimeError(f"cudaMemcpy failed ({err})")
