"""Multi-GPU partitioning: independent sessions sharded over ranks, no data-path collective.

SURVEY.md §8(e): within a session the path is sequential (replicas only); across sessions
it shards trivially. Sessions are assigned contiguously (rank g gets [g*S/G, (g+1)*S/G)),
each rank drives its own device maps, and the only cross-rank traffic is timing: the
per-step device time is reduced with MAX so a step counts as long as its slowest rank.
"""

from __future__ import annotations


def shard_range(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) share of n_items for `rank` of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return (n_items * rank) // world, (n_items * (rank + 1)) // world


def session_seeds(base_seed: int, n_sessions: int, world: int, rank: int) -> list[int]:
    """Seeds of the sessions this rank owns (C5: base 5000, 64 sessions)."""
    lo, hi = shard_range(n_sessions, world, rank)
    return [base_seed + s for s in range(lo, hi)]


def max_over_ranks(value: float, device=None) -> float:
    """MAX-reduce a per-rank scalar (no-op outside torch.distributed)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
