"""Batch-sharded multi-GPU inference: one process per GPU, weights replicated,
images split evenly across ranks, NO collective on the data path -- only the
final logits are gathered to rank 0.

Why this is exact: every row (image) of the reference's computation is
independent of every other (R:include/ternkit/linalg.hpp:278-291 partitions
rows across threads; R:tests/test_linalg.cpp:289-304 asserts batch
independence), so concatenating the per-shard outputs in rank order equals
the single-device output bit for bit.

The gather uses `all_gather` of equal-sized (padded) shards, which both the
NCCL backend (GPU boxes) and gloo (the CPU tests) implement.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch


@dataclass(frozen=True)
class Shard:
    start: int
    count: int


def shard_range(batch: int, rank: int, world: int) -> Shard:
    """Even split of `batch` images; the first batch % world ranks take one extra."""
    if world <= 0 or not 0 <= rank < world or batch < 0:
        raise ValueError(f"bad shard request batch={batch} rank={rank} world={world}")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return Shard(start, base + (1 if rank < extra else 0))


def max_shard(batch: int, world: int) -> int:
    return -(-batch // world)


class ShardedForward:
    """Run `forward(x_shard) -> [count, out_dim]` on this rank's slice of a
    global batch and gather the rows to rank 0 in global order.

    forward: the per-device network (e.g. TernaryResNet.forward); it sees only
    its shard, so no data-path collective exists.  Returns the full
    [batch, out_dim] tensor on rank 0 and None elsewhere."""

    def __init__(self, forward: Callable[[torch.Tensor], torch.Tensor], batch: int, out_dim: int,
                 rank: int, world: int, group=None):
        self.forward, self.batch, self.out_dim = forward, batch, out_dim
        self.rank, self.world, self.group = rank, world, group
        self.shard = shard_range(batch, rank, world)
        self.pad = max_shard(batch, world)

    def local_slice(self, x: torch.Tensor) -> torch.Tensor:
        s = self.shard
        return x[s.start:s.start + s.count]

    def gather(self, y: torch.Tensor) -> torch.Tensor | None:
        if y.shape != (self.shard.count, self.out_dim):
            raise ValueError(f"shard output {tuple(y.shape)} != ({self.shard.count}, {self.out_dim})")
        if self.world == 1:
            return y
        import torch.distributed as dist
        buf = torch.zeros((self.pad, self.out_dim), dtype=y.dtype, device=y.device)
        buf[: y.shape[0]] = y
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(parts, buf, group=self.group)
        if self.rank != 0:
            return None
        rows = [parts[r][: shard_range(self.batch, r, self.world).count] for r in range(self.world)]
        return torch.cat(rows, 0)

    def __call__(self, x_shard: torch.Tensor) -> torch.Tensor | None:
        return self.gather(self.forward(x_shard))
