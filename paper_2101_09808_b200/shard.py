"""Multi-GPU partitioning of Eq. 1.

Eq. 1 is parallelised over non-reduction dimensions only (PAPER.md:375,
Sec. 7): each rank computes an independent slab of Out, so no reduction
collective is ever needed.

* batch (n) sharding: rank p owns images [p*N/P, (p+1)*N/P).  In and Out
  slabs are contiguous in NCHW; Ker is replicated.
* output-channel (k) sharding, for N < P: rank p owns channels
  [p*K/P, (p+1)*K/P); In is replicated, the Ker slab is contiguous.  Only
  N == 1 is supported so that the gathered buffer is NCHW without a permute.

``gather`` assembles the full Out with one ``all_gather_into_tensor`` (NCCL
over NVLink on the GPU box; gloo in the CPU tests): n (or k at N == 1) is the
outermost dimension of each slab, so the gathered buffer IS the NCHW Out.
This module only slices, plans and moves buffers -- the convolution itself
runs in libconv.so.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

from .inputs import Shape


@dataclass(frozen=True)
class ShardSpec:
    dim: str          # "n" or "k"
    world: int
    rank: int
    start: int
    stop: int
    local: Shape      # the per-rank problem a plan is created for

    @property
    def size(self) -> int:
        return self.stop - self.start


def shard(shape: Shape, world: int, rank: int, dim: str = "auto") -> ShardSpec:
    """Contiguous, equal split of n (default) or k across ``world`` ranks."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    if dim == "auto":
        dim = "n" if shape.N >= world else "k"
    if dim == "n":
        if shape.N % world:
            raise ValueError(f"N={shape.N} is not divisible by world={world}")
        step = shape.N // world
        local = replace(shape, N=step)          # keeps the stride and input extents
    elif dim == "k":
        if shape.N != 1:
            raise ValueError("k-sharding is supported for N == 1 only (gathered buffer stays NCHW)")
        if shape.K % world:
            raise ValueError(f"K={shape.K} is not divisible by world={world}")
        step = shape.K // world
        local = replace(shape, K=step)
    else:
        raise ValueError(f"unknown shard dim {dim!r}")
    return ShardSpec(dim, world, rank, rank * step, (rank + 1) * step, local)


def local_inputs(spec: ShardSpec, inp, ker):
    """This rank's (In, Ker) views (contiguous) for the full tensors."""
    if spec.dim == "n":
        return inp[spec.start:spec.stop].contiguous(), ker
    return inp, ker[spec.start:spec.stop].contiguous()


def gather(out_local, spec: ShardSpec, group=None):
    """All-gather the per-rank Out slabs into the full NCHW Out."""
    import torch
    import torch.distributed as dist

    full_shape = list(out_local.shape)
    axis = 0 if spec.dim == "n" else 1
    full_shape[axis] *= spec.world
    # gather flat: rank slabs land back to back, which is the NCHW order
    flat = torch.empty(spec.world * out_local.numel(), dtype=out_local.dtype, device=out_local.device)
    dist.all_gather_into_tensor(flat, out_local.contiguous().reshape(-1), group=group)
    return flat.view(full_shape)
