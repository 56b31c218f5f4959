"""Multi-GPU plumbing for the shearlet hot path (torch.distributed).

* 3D (and large 2D) systems shard the filter bank by shearlet index: rank r
  owns the contiguous band range shard_range(R, r, world) (balanced by count:
  every band costs the same FFT work). The input volume is broadcast from the
  root, each rank decomposes / thresholds / reconstructs its own bands, and
  the reconstruction partial sums -- linear in the coefficients -- are
  combined with a sum-reduce (NCCL over NVLink on the GPU box).
* Batched 2D frames shard by image (frame_range): no collective.
The reference has no distributed code; its
parallel_for over the filter index (parallel.hpp:20-46) is the axis sharded
here.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def shard_range(R: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous balanced band range [lo, hi) of rank `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world size")
    return R * rank // world, R * (rank + 1) // world


def frame_range(nframes: int, rank: int, world: int) -> Tuple[int, int]:
    """Frames of a batch handled by `rank` (shard by image)."""
    return shard_range(nframes, rank, world)


def sharded_denoise(x, local_partial: Callable, group=None, root: int = 0):
    """Broadcast x from `root`, run local_partial(x) -> partial reconstruction
    (this rank's bands only), and sum-reduce the partials onto `root`.
    Returns the full reconstruction on `root` (the partial elsewhere)."""
    import torch.distributed as dist
    dist.broadcast(x, src=root, group=group)
    part = local_partial(x)
    dist.reduce(part, dst=root, op=dist.ReduceOp.SUM, group=group)
    return part


def sharded_denoise_accumulator(x, local_accumulator: Callable, finish: Callable, group=None, root: int = 0,
                                slabs: int = 4):
    """The library's 3D schedule (csrc/comm.cuh denoise_dist), with
    torch.distributed collectives: broadcast x from `root`; every rank forms the
    half-spectrum accumulator sum_b FFT(thr c_b) psi_b of its bands; the
    accumulators are sum-reduced onto the root in `slabs` contiguous slabs along
    the first axis (the order the library overlaps with its last band group);
    only the root runs finish(acc) (divide by W, inverse FFT). Returns finish's
    result on the root, None elsewhere."""
    import torch
    import torch.distributed as dist
    dist.broadcast(x, src=root, group=group)
    acc = local_accumulator(x)
    n0 = acc.shape[0]
    for j in range(slabs):
        lo, hi = n0 * j // slabs, n0 * (j + 1) // slabs
        if hi > lo:
            part = acc[lo:hi].contiguous()
            if torch.is_complex(part):  # gloo reduces real tensors: view complex as (re, im) pairs
                pr = torch.view_as_real(part).contiguous()
                dist.reduce(pr, dst=root, op=dist.ReduceOp.SUM, group=group)
                part = torch.view_as_complex(pr)
            else:
                dist.reduce(part, dst=root, op=dist.ReduceOp.SUM, group=group)
            acc[lo:hi] = part
    return finish(acc) if dist.get_rank(group) == root else None


def sharded_forward_thresholded(x, sys, schedule, group=None, root: int = 0):
    """Device path: broadcast then this rank's thresholded bands."""
    import torch.distributed as dist
    from . import forward_thresholded
    dist.broadcast(x, src=root, group=group)
    return forward_thresholded(x, sys, schedule)


def sharded_inverse(coeffs, sys, group=None, root: int = 0):
    """Partial reconstruction of this rank's bands, sum-reduced to `root`."""
    import torch.distributed as dist
    from . import inverse
    part = inverse(coeffs, sys)
    dist.reduce(part, dst=root, op=dist.ReduceOp.SUM, group=group)
    return part


def library_comm(device: int, group=None):
    """The library's own NCCL communicator over the ranks of a torch.distributed
    group: rank 0 creates the NCCL unique id, torch.distributed broadcasts it
    (any backend, gloo included), every rank joins (sl_comm_create)."""
    import torch.distributed as dist
    from . import Comm
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return Comm(box[0], world, rank, device)


def attach(sys, comm, shard_bands: Optional[bool] = None):
    """Attach `comm` to a system: 3D shards the bank by shearlet index, 2D keeps
    the whole bank (frames shard by image)."""
    sys.set_comm(comm, sys.ndim == 3 if shard_bands is None else shard_bands)
    return sys
