"""Frame sharding for multi-GPU runs.

Frames are independent (reference proj/src/sequence.cpp:59-77 carries no state between
frames), so N GPUs split a frame sequence with no data-path collective: frame i goes to
rank i mod N, every rank converts its own frames on its own device, and the host restores
order by frame index (the reference's FrameSink::write(index, ...) contract,
proj/include/pseudo3d/sequence.hpp:26-30). torch.distributed is plumbing only: start/stop
barriers and the max-over-ranks of a device time.
"""
from __future__ import annotations

import os
import socket
import sys


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


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun_argv(nproc: int, script: str, args: list[str], port: int | None = None) -> list[str]:
    """The one-process-per-GPU launch of `script` (what the driver runs for N > 1):
    torch.distributed.run on this node, rendezvous on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr=127.0.0.1", f"--master-port={port or free_port()}", script, *args]


def node_cpus(node: int) -> set[int]:
    """CPUs of a NUMA node from sysfs (empty when unknown)."""
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            text = f.read().strip()
    except OSError:
        return set()
    cpus: set[int] = set()
    for part in filter(None, text.split(",")):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return cpus


def bind_to_node(node: int) -> bool:
    """Restricts this process to a NUMA node's CPUs (so its pinned host buffers, allocated
    afterwards, are node-local); False when the node or its CPUs are unknown."""
    cpus = node_cpus(node) & os.sched_getaffinity(0) if node >= 0 else set()
    if not cpus:
        return False
    os.sched_setaffinity(0, cpus)
    return True
