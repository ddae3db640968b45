"""Multi-GPU data parallelism over camera views.

One process per GPU, each holding a full replica of the scene.  Views are dealt
round-robin (rank r owns views r, r+N, ...); each rank renders and backprops its
own views into one contiguous f32[9N] gradient buffer (the five parameter
gradients as views of it, Renderer.grad_views), then ONE all-reduce (SUM) over
the process group -- NCCL over NVLink/NVSwitch on a B200 box.  The forward needs
no collective.  This is the only exchange step on the path.
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def shard_views(views: Sequence, world_size: int, rank: int) -> list:
    """Round-robin deal of views to ranks: rank r gets views r, r+N, ..."""
    if world_size < 1 or not (0 <= rank < world_size):
        raise ValueError("bad world_size / rank")
    return list(views[rank::world_size])


def allreduce_grads(flat: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the flat per-cell gradient buffer over all ranks (in place)."""
    ws, _ = world()
    if ws > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


def sharded_backward(local_views: Sequence, backward_fn: Callable, flat: torch.Tensor,
                     group=None) -> torch.Tensor:
    """Zero `flat`, accumulate backward_fn(view, flat) over this rank's views,
    then all-reduce.  backward_fn is the per-view (or per-batch) gradient
    producer; on a B200 it is Renderer.backward."""
    flat.zero_()
    for v in local_views:
        backward_fn(v, flat)
    return allreduce_grads(flat, group)


def train_step(renderer, cams_local: Sequence, grad_out_local: torch.Tensor, flat: torch.Tensor,
               out: torch.Tensor | None = None, group=None,
               before_backward: Callable | None = None):
    """One data-parallel step on this rank: forward of the local views (one
    batched call), backward into `flat` (f32[grad_size]), all-reduce of `flat`.
    before_backward() runs after the forward is enqueued (e.g. make the stream
    wait for an asynchronous host->device copy of grad_out, which the forward
    does not read).  Returns (images, flat)."""
    img = renderer.forward(list(cams_local), out=out)
    flat.zero_()
    if before_backward is not None:
        before_backward()
    renderer.backward(list(cams_local), grad_out_local, flat)
    allreduce_grads(flat, group)
    return img, flat
