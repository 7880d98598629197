"""Host-side multi-GPU plumbing of the pull path (SURVEY.md §8 row e).

One process per GPU.  Ranks [0, N/2) hold prefill caches, ranks [N/2, N)
decode caches; decode rank N/2 + k pulls from prefill rank k -- the paper's
rail rule "GPU i of a decode worker can only connect with GPU i of a
prefill worker".  NVSwitch makes every pair equivalent, so the
rule is a convention here, not a topology constraint.

The only cross-process exchange is the one-time Connect() metadata:
each rank contributes its export blob (or None) to one all_gather_object on
a gloo group.  The data path has no collective: pairs are independent.
With N = 1 there is no pair; the caller runs the loopback (both caches on
the same GPU).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Any, List, Optional, Sequence


@dataclass(frozen=True)
class Role:
    rank: int
    world: int
    role: str            # "prefill", "decode" or "both" (N = 1 loopback)
    peer: Optional[int]  # the rank on the other end of this rank's pair
    pairs: int


def role_of(rank: int, world: int) -> Role:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of world {world}")
    if world == 1:
        return Role(0, 1, "both", 0, 1)
    if world % 2:
        raise ValueError("N > 1 must be even: prefill/decode pairs")
    half = world // 2
    if rank < half:
        return Role(rank, world, "prefill", rank + half, half)
    return Role(rank, world, "decode", rank - half, half)


def ring_role_of(rank: int, world: int) -> Role:
    """A stress of the switch, not the paper's deployment: every rank holds
    both caches and pulls from its ring successor's prefill cache (rank
    k <- rank k + 1 mod N), so N pulls run at once and every GPU's NVLink
    ingress and egress carry one each (full duplex).  With N = 4 that is as
    many concurrent pulls through NVSwitch as the 4P:4D rail pairing at
    N = 8.  N = 1 is the loopback."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of world {world}")
    if world == 1:
        return Role(0, 1, "both", 0, 1)
    return Role(rank, world, "both", (rank + 1) % world, world)


def exchange_blobs(blob: Optional[bytes], group=None) -> List[Optional[bytes]]:
    """All ranks contribute their export blob (prefill) or None (decode)."""
    import torch.distributed as dist
    out: List[Any] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


def peer_blob(role: Role, blobs: Sequence[Optional[bytes]]) -> Optional[bytes]:
    """The blob a pulling rank opens: its partner's (rail partner, or ring
    successor)."""
    if role.role == "prefill":
        return None
    b = blobs[role.peer]
    if b is None:
        raise RuntimeError(f"rank {role.rank}: prefill rank {role.peer} exported nothing")
    return b


def gather_stats(stats: dict, group=None) -> List[dict]:
    import torch.distributed as dist
    out: List[Any] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, stats, group=group)
    return out


def aggregate(all_stats: Sequence[dict]) -> dict:
    """Whole-job numbers from per-rank stats: time = MAX over the ranks that
    moved bytes (the contract's max-over-ranks), bytes = SUM."""
    movers = [s for s in all_stats if s.get("bytes")]
    if not movers:
        return {"bytes": 0, "dev_s": 0.0, "wall_s": 0.0, "ranks": 0}
    return {"bytes": sum(s["bytes"] for s in movers),
            "dev_s": max(s["dev_s"] for s in movers),
            "wall_s": max(s["wall_s"] for s in movers),
            "ranks": len(movers)}
