"""Multi-GPU sharding of the shot range (one process per GPU).

Every draw is keyed by (seed, stream, global shot index) (rng.hpp:31-41,
sampler.cpp:82, 91, 268-284), so sharding the global shot range across ranks
reproduces the single-process (and the CPU reference's) bits exactly, with no
data-path communication. The only collective is the final all-reduce of the
per-output flip counts (detector and logical-observable error counts) — one
[num_outputs] int64 vector, over NCCL on GPUs (gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(total_shots: int, rank: int, world: int, align: int = 64) -> tuple[int, int]:
    """[first, first+count) of `rank`: contiguous, disjoint, covering
    [0, total_shots), boundaries on multiples of `align` shots (whole output
    words), balanced to within `align` shots."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    words = (total_shots + align - 1) // align
    lo = words * rank // world
    hi = words * (rank + 1) // world
    first = lo * align
    last = min(total_shots, hi * align)
    return first, max(0, last - first)


def allreduce_counts(counts, group=None):
    """Sums a per-output counts tensor over all ranks (in place)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def count_outputs_sharded(total_shots: int, seed: int, num_outputs: int,
                          counter: Callable[[int, int, int], "object"], group=None, device=None) -> np.ndarray:
    """Per-output flip counts over [0, total_shots) split across the ranks of
    `group`. `counter(seed, first_shot, shots)` returns this rank's counts as a
    torch int64 tensor on `device` (the sampler's zxs_count_device on a GPU)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    first, count = shard_range(total_shots, rank, world)
    counts = counter(seed, first, count) if count else torch.zeros(num_outputs, dtype=torch.int64, device=device)
    allreduce_counts(counts, group)
    return counts.cpu().numpy().astype(np.uint64)


def gpu_counter(cs, stream=None, device=None):
    """counter() for count_outputs_sharded backed by the device sampler
    (zxs_count_device into a device tensor; `device` defaults to the sampler's
    GPU -- the CPU tests pass a host device and a stand-in sampler)."""
    import torch

    def run(seed: int, first: int, shots: int):
        dev = device if device is not None else torch.device("cuda", cs.device)
        counts = torch.zeros(cs.num_outputs, dtype=torch.int64, device=dev)
        st = stream if stream is not None else torch.cuda.current_stream(cs.device).cuda_stream
        cs.count_device(seed, first, shots, counts.data_ptr(), st)
        cs.check_errors(st)
        return counts
    return run
