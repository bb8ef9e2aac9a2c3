"""Multi-GPU plumbing for the hot path: one process per GPU,
torch.distributed for the collectives.

* Queries shard by contiguous id range; each rank routes its shard with
  index_base = its first id, so every heavy-queue id it writes is global.
* The only data-path collective is an all-gather of the per-rank routed
  counts ([T] int64 per rank); an exclusive scan over ranks gives each rank's
  offset inside every global heavy queue, and concatenating the per-rank
  lists in rank order reproduces the single-GPU (= reference) id order.
* Planner problems shard by index; plans are independent (no collective on
  the data path; gather only to report).
* Or one batch of problems shards by THRESHOLD RANGE: each rank searches its
  contiguous slice of the grid (ds_plan_keys), a MIN all-reduce of the packed
  selection keys picks the reference's winner (the key order is its choice
  order), and ds_plan_from_keys decodes (SURVEY.md 8(e) "by t-range").
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of a contiguous, balanced split of n items over world ranks."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return n * rank // world, n * (rank + 1) // world


def exclusive_offsets(gathered_counts: np.ndarray) -> np.ndarray:
    """[world, T] routed counts -> [world, T] start offset of each rank's
    block inside every global heavy queue (exclusive scan over ranks)."""
    c = np.asarray(gathered_counts, np.int64)
    out = np.zeros_like(c)
    out[1:] = np.cumsum(c[:-1], axis=0)
    return out


def gather_counts(counts, group=None):
    """All-gather of a rank's [T] int64 routed counts (torch tensor on the
    rank's device for NCCL, CPU for gloo) -> [world, T] tensor."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "gloo" and counts.is_cuda:
        # gloo test path: gather through host memory
        parts = [torch.empty_like(counts, device="cpu") for _ in range(world)]
        dist.all_gather(parts, counts.cpu(), group=group)
        return torch.stack(parts).to(counts.device)
    out = torch.empty(world * counts.numel(), dtype=counts.dtype, device=counts.device)
    dist.all_gather_into_tensor(out, counts.contiguous(), group=group)
    return out.view(world, counts.numel())


def global_offsets_device(counts, group=None):
    """Device-side version: gathered counts -> this rank's offsets [T]."""
    import torch.distributed as dist
    g = gather_counts(counts, group)
    rank = dist.get_rank(group)
    return g[:rank].sum(0) if rank > 0 else g[0] * 0


KEY_NONE = np.uint64(0xFFFFFFFFFFFFFFFF)
_I64_MAX = np.int64(0x7FFFFFFFFFFFFFFF)


def keys_to_i64(keys: np.ndarray) -> np.ndarray:
    """uint64 selection keys -> int64 with the same order for the reduction
    (real keys are < 2^63: the threshold field is at most 2^23 wide; "none" =
    2^64-1 maps to INT64_MAX)."""
    k = np.asarray(keys, np.uint64)
    out = k.astype(np.int64)
    out[k == KEY_NONE] = _I64_MAX
    return out


def keys_from_i64(keys: np.ndarray) -> np.ndarray:
    k = np.asarray(keys, np.int64)
    out = k.astype(np.uint64)
    out[k == _I64_MAX] = KEY_NONE
    return out


def plan_t_sharded(keys_fn, decode_fn, grid_len: int, group=None, device=None):
    """Threshold-range sharded planning over the ranks of `group`.

    keys_fn(t_lo, t_hi) -> uint64 keys of this rank's grid slice;
    decode_fn(keys) -> plans. The slices are contiguous and balanced, the
    reduction is an all-reduce MIN of the keys (NCCL: on `device`; gloo: CPU).
    """
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    lo, hi = shard_range(grid_len, world, rank)
    mine = torch.from_numpy(keys_to_i64(keys_fn(lo, hi)))
    if device is not None and dist.get_backend(group) != "gloo":
        mine = mine.to(device)
    dist.all_reduce(mine, op=dist.ReduceOp.MIN, group=group)
    return decode_fn(keys_from_i64(mine.cpu().numpy()))
