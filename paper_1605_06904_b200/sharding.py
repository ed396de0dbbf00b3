"""Multi-GPU plumbing for the trial loop: contiguous trial shards, one tiny exchange.

Projection trials are independent given (master seed, trial index) (driver.hpp:164), so rank r of
N runs trials shard_range(m, r, N) on its own GPU against a full replica of the packed sequences
and only the fixed-size per-rank result record is exchanged (all_gather over NCCL on GPUs, gloo in
the CPU tests).  The merge itself is pm_merge_results in libpm_b200.so (ascending-trial scan,
driver.hpp:195-208)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import RunResult, merge_results


def shard_range(m: int, rank: int, world: int):
    """1-based inclusive [begin, end] of the contiguous trial shard of `rank`; empty shards have end < begin."""
    base, extra = divmod(m, world)
    begin = rank * base + min(rank, extra) + 1
    end = begin + base + (1 if rank < extra else 0) - 1
    return begin, end


def result_to_tensor(result: RunResult, positions, t: int):
    import torch
    raw = np.frombuffer(bytes(result), dtype=np.uint8)
    pos = np.zeros(t, dtype=np.int32) if positions is None else np.asarray(positions, dtype=np.int32)
    return torch.from_numpy(np.concatenate([raw, pos.view(np.uint8)]).copy())


def tensor_to_result(tensor, t: int):
    raw = tensor.cpu().numpy().tobytes()
    n = C.sizeof(RunResult)
    res = RunResult.from_buffer_copy(raw[:n])
    pos = np.frombuffer(raw[n:n + 4 * t], dtype=np.int32).copy()
    return res, pos


def all_gather_merge(result: RunResult, positions, t: int, l: int, early_stop: bool, device=None):
    """Every rank contributes its shard result; every rank returns the merged (RunResult, positions)."""
    import torch
    import torch.distributed as dist
    mine = result_to_tensor(result, positions, t)
    if device is not None:
        mine = mine.to(device)
    world = dist.get_world_size()
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    parts, poss = [], []
    for g in gathered:
        r, p = tensor_to_result(g, t)
        parts.append(r)
        poss.append(p)
    return merge_results(parts, poss, t, l, early_stop)
