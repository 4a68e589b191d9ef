"""Element sharding and the deterministic global residual norm (config 5).

The volume term has no cross-element coupling (kernel.py / burgers.py:117-131
touch one element at a time), so elements are split into contiguous shards
[e0, e0 + E_local) per rank with no data-path collective.  The only exchange
is the residual norm ||Rhat||_2 over all elements:

  1. the kernel writes sum_v sum_k Rhat[e,v,k]^2 per element (fixed order);
  2. fixed-size blocks of `block` elements are summed with a perfect binary
     tree (sfb_block_sums on the device; numpy-identical order);
  3. the per-block partials are all-gathered (NCCL on GPUs, gloo on CPU) and
     summed in global block order with the same fixed tree, then sqrt.
Steps 2-3 make the norm bitwise identical for any number of ranks that
divides the block count.  ``allreduce=True`` instead sums one scalar per rank
with all_reduce (the plain NCCL reduction; not G-invariant in the last bits).
"""

import torch

from . import _lib


def shard_range(total, rank, world):
    """Contiguous shard [e0, e0 + count) of `total` elements for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(total, world)
    e0 = rank * base + min(rank, extra)
    return e0, base + (1 if rank < extra else 0)


def tree_sum(x):
    """Perfect-binary-tree sum of a power-of-two-length float64 vector (numpy/torch)."""
    n = x.shape[-1]
    if n & (n - 1):
        raise ValueError("tree_sum needs a power-of-two length")
    while x.shape[-1] > 1:
        x = x[..., 0::2] + x[..., 1::2]
    return x[..., 0]


def block_partials(sumsq, block):
    """Per-block tree sums of per-element values (device kernel on CUDA tensors)."""
    count = sumsq.numel()
    if count % block:
        raise ValueError(f"{count} elements are not a multiple of the block {block}")
    if sumsq.is_cuda:
        out = torch.empty(count // block, dtype=torch.float64, device=sumsq.device)
        _lib.call("sfb_block_sums", _lib.ptr(sumsq), count, block, _lib.ptr(out),
                  _lib.stream_ptr())
        return out
    return tree_sum(sumsq.reshape(-1, block))


def global_norm(sumsq, block=4096, group=None, allreduce=False):
    """sqrt(sum over all ranks' elements of sumsq), deterministic across world sizes."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if allreduce:
        total = sumsq.sum().reshape(1)
        if world > 1:
            dist.all_reduce(total, group=group)
        return float(total.sqrt().item())
    part = block_partials(sumsq, block)
    if world > 1:
        gathered = [torch.empty_like(part) for _ in range(world)]
        dist.all_gather(gathered, part, group=group)
        part = torch.cat(gathered)
    nb = part.numel()
    pad = 1 << max(0, (nb - 1).bit_length())
    if pad != nb:
        part = torch.cat([part, torch.zeros(pad - nb, dtype=part.dtype, device=part.device)])
    return float(tree_sum(part).sqrt().item())
