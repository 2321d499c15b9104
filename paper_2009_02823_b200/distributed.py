"""Sharded engines: the state split over 2^g shards by its top g qubits.

* ``virtual_engine(shards)``: every shard on one device -- the distributed
  schedule (qubit swaps, partner fetches, per-shard partials) executed with
  device-local exchanges; used to test the N>1 path on one GPU.
* ``nccl_engine()``: one rank of a one-process-per-GPU job launched with
  torchrun; torch.distributed carries the NCCL unique id, the engine itself
  drives NCCL (pairwise half-shard exchanges over NVLink for qubit swaps,
  partner-shard fetches for observable terms that flip rank bits, one
  all-gather of the (A+1) partial sums per gradient).

Pass the engine to ``reverse_mode_gradient(..., engine=...)``.
"""
from __future__ import annotations

from . import _native


def virtual_engine(shards: int, device: int = 0) -> _native.Engine:
    return _native.Engine(device, shards=shards)


def nccl_engine(device: int | None = None) -> _native.Engine:
    """Collective: every rank of the initialised torch.distributed group must call it."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    if device is None:
        device = torch.cuda.current_device()
    uid = [_native.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    return _native.Engine(device, shards=world, rank=rank, nccl_id=uid[0])
