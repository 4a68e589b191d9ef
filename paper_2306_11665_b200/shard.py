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
Steps 2-3 make the norm bitwise identical for any number of ranks when the
shards are whole blocks (block_shard; unequal block counts per rank are
gathered padded and compacted back into global block order).  ``allreduce=True`` instead sums one scalar per rank
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


def job_block(total, max_block=4096):
    """The norm's block size for a whole job: the largest power of two <= max_block
    dividing `total` (chosen once, from the global count, identically on every rank)."""
    if total < 1:
        raise ValueError("total must be positive")
    b = 1
    while b * 2 <= max_block and total % (b * 2) == 0:
        b *= 2
    return b


def block_shard(total, rank, world, block):
    """Contiguous shard of whole blocks: [e0, e0 + count) with e0, count multiples
    of `block` (shard_range over total // block blocks)."""
    if total % block:
        raise ValueError(f"{total} elements are not a multiple of the block {block}")
    b0, nb = shard_range(total // block, rank, world)
    return b0 * block, nb * block


def _gather_partials(part, group, counts):
    """All-gather per-rank block partials (possibly unequal counts) into global order."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if counts is None:
        n = torch.tensor([part.numel()], dtype=torch.int64, device=part.device)
        ns = [torch.empty_like(n) for _ in range(world)]
        dist.all_gather(ns, n, group=group)
        counts = [int(x.item()) for x in ns]
    width = max(counts)
    if part.numel() < width:  # equal-size buffers for the collective
        part = torch.cat([part, part.new_zeros(width - part.numel())])
    gathered = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(gathered, part, group=group)
    return torch.cat([g[:c] for g, c in zip(gathered, counts)])


def global_norm_tensor(sumsq, block=4096, group=None, total=None):
    """Device scalar sqrt(sum over all ranks' elements of sumsq), no host sync.

    Bitwise identical for every world size when the shards are whole blocks
    in rank order (block_shard): per-block tree partials, all-gathered into
    global block order, one fixed tree over them.  ``total`` (elements over all
    ranks) lets every rank derive the per-rank block counts locally; without
    it they are exchanged first.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    part = block_partials(sumsq, block)
    if world > 1:
        counts = None
        if total is not None:
            counts = [block_shard(total, r, world, block)[1] // block for r in range(world)]
            rank = dist.get_rank(group)
            if counts[rank] != part.numel():
                raise ValueError(f"rank {rank} holds {part.numel()} blocks, block_shard("
                                 f"{total}) assigns {counts[rank]}")
        part = _gather_partials(part, group, counts)
    nb = part.numel()
    pad = 1 << max(0, (nb - 1).bit_length())
    if pad != nb:
        part = torch.cat([part, part.new_zeros(pad - nb)])
    return tree_sum(part).sqrt()


def global_norm(sumsq, block=4096, group=None, allreduce=False, total=None):
    """sqrt(sum over all ranks' elements of sumsq) as a float (one host sync)."""
    import torch.distributed as dist

    if allreduce:
        world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        t = sumsq.sum().reshape(1)
        if world > 1:
            dist.all_reduce(t, group=group)
        return float(t.sqrt().item())
    return float(global_norm_tensor(sumsq, block, group, total).item())
