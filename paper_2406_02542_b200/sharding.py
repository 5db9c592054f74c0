"""Multi-GPU layout of the Loki decode path.

Every (batch, KV head) unit is independent: approximate scores, top-k, the
gather and the softmax never cross heads (reference: per-head by construction,
attention.py:18-19).  So the path shards with NO collective inside the
attention: KV heads are split contiguously across ranks, each rank holds its
slice of the caches, its projections and its query heads, and one NCCL
all-gather per layer reassembles the [B, Hq, D] outputs the next layer needs
(the only exchange step).  One process per GPU, torch.distributed for the
plumbing.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import ShapeError


@dataclass(frozen=True)
class HeadShard:
    """Contiguous KV heads [kv0, kv1) of this rank and the query heads they serve."""

    rank: int
    world: int
    kv0: int
    kv1: int
    q0: int
    q1: int

    @property
    def kv_heads(self) -> int:
        return self.kv1 - self.kv0

    @property
    def q_heads(self) -> int:
        return self.q1 - self.q0


def head_shard(Hq: int, Hkv: int, world: int, rank: int) -> HeadShard:
    """KV heads split contiguously and evenly (query head h -> KV head h // (Hq / Hkv)).

    Raises ShapeError when the KV heads do not divide evenly: an uneven split
    would make the all-gather ragged (batch sharding is the alternative then).
    """
    if world < 1 or not 0 <= rank < world:
        raise ShapeError(f"rank {rank} outside world of {world}")
    if Hkv < 1 or Hq % Hkv:
        raise ShapeError(f"query heads {Hq} are not a multiple of kv heads {Hkv}")
    if Hkv % world:
        raise ShapeError(f"{Hkv} KV heads cannot be split evenly over {world} ranks")
    per = Hkv // world
    G = Hq // Hkv
    kv0 = rank * per
    return HeadShard(rank, world, kv0, kv0 + per, kv0 * G, (kv0 + per) * G)


def shard_heads(x: torch.Tensor, shard: HeadShard, kv: bool) -> torch.Tensor:
    """This rank's slice of a [B, H, ...] tensor (KV heads if kv else query heads), as a view."""
    lo, hi = (shard.kv0, shard.kv1) if kv else (shard.q0, shard.q1)
    return x[:, lo:hi]


def gather_heads(local: torch.Tensor, world: int, group=None, out: torch.Tensor | None = None,
                 staging: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather per-rank outputs [B, Hq/world, D] into [B, Hq, D] (rank-major heads).

    `staging` ([world * B, Hq/world, D], optional) avoids an allocation per call;
    the result is written into `out` when given.
    """
    import torch.distributed as dist

    if local.dim() != 3:
        raise ShapeError(f"expected local outputs [B, Hq/world, D], got {tuple(local.shape)}")
    B, hq, D = local.shape
    if staging is None:
        staging = torch.empty((world * B, hq, D), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(staging, local.contiguous(), group=group)  # rank-major along dim 0
    full = staging.view(world, B, hq, D).permute(1, 0, 2, 3).reshape(B, world * hq, D)
    if out is not None:
        out.copy_(full)
        return out
    return full
