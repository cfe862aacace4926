"""CPU, world_size 2 over gloo: the frame-sharding host logic of the multi-GPU path
(paper_2009_09501_b200/sharding.py, used by bench.py under torchrun). Frames split with no
data-path collective; the union of the ranks' outputs equals a single-rank run (the
GPU-count analogue of the reference's AC-1 worker-count invariance),
checked here with the CPU oracle as the per-frame converter."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_09501_b200.sharding import frame_seed, max_over_ranks, shard_frames

W, H, NFRAMES = 40, 24, 7


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _convert_frames(indices):
    import oracle
    port = oracle.load("port")
    out = {}
    for i in indices:
        img = port.synthetic_frame(W, H, frame_seed(i))
        out[i] = _digest(port.convert(img, oracle.Cfg(base=6))["anaglyph"])
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard_frames(NFRAMES, rank, world)
        digests = _convert_frames(mine)
        gathered = [None] * world
        dist.all_gather_object(gathered, digests)
        t = max_over_ranks([float(rank + 1), -float(rank)])
        if rank == 0:
            q.put((gathered, t))
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for n in (0, 1, 7, 64):
        for world in (1, 2, 4, 8):
            parts = [shard_frames(n, r, world) for r in range(world)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        shard_frames(4, 2, 2)


def test_two_rank_gloo_matches_single_rank():
    import oracle
    if not oracle.available("port"):
        oracle.build("port")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    merged = {}
    for d in gathered:
        assert not set(d) & set(merged)  # no frame converted twice
        merged.update(d)
    assert merged == _convert_frames(range(NFRAMES))
    assert t == [2.0, 0.0]
