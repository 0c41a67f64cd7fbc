"""Multi-GPU execution = independent DAG replicas.

A benchmark DAG is a single-GPU unit (the paper is
single-GPU; multi-GPU placement is its future work), so under torchrun every
rank runs its own DAG instances on its own GPU with its own dagrt context.
No step of the data path needs a collective; torch.distributed is used only
for the barrier around the timed region and for the max of the per-rank
timings (the job finishes when its slowest rank does).

These helpers are backend-agnostic (NCCL on the GPU box, gloo in the CPU
tests) and hold no benchmark arithmetic.
"""
from __future__ import annotations


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(ms: float, dist, device=None) -> float:
    """Max of a per-rank duration over all ranks (identity without dist)."""
    if dist is None:
        return float(ms)
    import torch
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_ms_per_dag(max_ms: float, steps: int, world: int) -> float:
    """Whole-job time per DAG: every rank ran `steps` DAGs in `max_ms`, so the
    job processed steps*world DAGs in that time (weak scaling)."""
    return max_ms / (steps * world)


def instance_ids(rank: int, world: int, steps: int):
    """The DAG instances rank `rank` runs: instance k of the job goes to rank
    k % world (round robin), `steps` per rank.  Each instance draws its own
    seeded inputs, so no two ranks share or exchange data."""
    return [rank + world * s for s in range(steps)]
