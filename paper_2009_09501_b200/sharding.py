"""Frame sharding for multi-GPU runs.

Frames are independent (reference proj/src/sequence.cpp:59-77 carries no state between
frames), so N GPUs split a frame sequence with no data-path collective: frame i goes to
rank i mod N, every rank converts its own frames on its own device, and the host restores
order by frame index (the reference's FrameSink::write(index, ...) contract,
proj/include/pseudo3d/sequence.hpp:26-30). torch.distributed is plumbing only: start/stop
barriers and the max-over-ranks of a device time.
"""
from __future__ import annotations


def shard_frames(n_frames: int, rank: int, world: int) -> list[int]:
    """Global frame indices owned by `rank` (round-robin, i mod world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    return list(range(rank, n_frames, world))


def frame_seed(index: int) -> int:
    """Seed of synthetic video frame `index` (seed = 1 + frame index)."""
    return 1 + index


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity without a group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def barrier() -> None:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
