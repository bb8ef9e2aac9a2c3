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
_SIGN = np.uint64(0x8000000000000000)


def keys_to_i64(keys: np.ndarray) -> np.ndarray:
    """uint64 selection keys -> int64 with the same order for a signed MIN
    reduction: flipping bit 63 maps unsigned order onto signed order for
    every key (including keys >= 2^63 on grids longer than 2^23 points);
    "none" = 2^64-1 lands on INT64_MAX."""
    k = np.asarray(keys, np.uint64)
    return (k ^ _SIGN).view(np.int64)


def keys_from_i64(keys: np.ndarray) -> np.ndarray:
    k = np.ascontiguousarray(keys, np.int64)
    return k.view(np.uint64) ^ _SIGN


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


class TorchHostOps:
    """ds_comm_ops over a torch.distributed process group (host tensors; gloo).

    The host transport of native.Comm.host: the library stages device data
    through pinned host memory and calls these. Used where NCCL cannot run --
    several ranks sharing one GPU in the tests (NCCL refuses duplicate
    devices), or hosts without NCCL."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allgather(self, send: np.ndarray) -> np.ndarray:
        import torch
        import torch.distributed as dist
        t = torch.from_numpy(np.ascontiguousarray(send, np.uint8))
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t, group=self.group)
        return torch.cat(parts).numpy()

    def allreduce_min_u64(self, buf: np.ndarray) -> np.ndarray:
        import torch
        import torch.distributed as dist
        t = torch.from_numpy(keys_to_i64(buf).copy())
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return keys_from_i64(t.numpy())

    def gatherv(self, send: np.ndarray, sizes, root: int):
        import torch
        import torch.distributed as dist
        m = max(max(sizes), 1)
        t = torch.zeros(m, dtype=torch.uint8)
        if len(send):
            t[:len(send)] = torch.from_numpy(np.ascontiguousarray(send, np.uint8))
        if self.rank == root:
            parts = [torch.empty(m, dtype=torch.uint8) for _ in range(self.world)]
            dist.gather(t, parts, dst=root, group=self.group)
            return np.concatenate([p.numpy()[:sizes[r]] for r, p in enumerate(parts)])
        dist.gather(t, None, dst=root, group=self.group)
        return None


def nccl_comm(ctx, group=None):
    """A native.Comm over NCCL for this process's rank of `group`: rank 0 makes
    the unique id, torch.distributed broadcasts it, every rank initialises
    (ncclCommInitRank on its context's device)."""
    import torch.distributed as dist
    from . import native
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    box = [native.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return native.Comm.nccl(ctx, world, rank, box[0])
