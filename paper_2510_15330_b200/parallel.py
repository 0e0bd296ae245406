"""Scenario sharding and the single exchange step.

Scenarios are independent units: rank r of W simulates ids r, r+W, r+2W, ...
(interleaving puts every (rate, controller) cell on every rank, which balances
per-tick cost).  The only collective is at the end of a step: all_gather of
the 272-byte summary records (NCCL over NVLink on GPUs, gloo in CPU tests)
and an all_reduce(SUM) of the integer segment histograms.  Integer sums are
order-independent, so results are bit-identical for any world size.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

REC = 272  # bytes per bellman_scenario_stats


def shard_count(n: int, rank: int, world: int) -> int:
    return len(range(rank, n, world))


def shard_rows(full_rows: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """This rank's records (ids rank, rank+world, ...) as a contiguous block."""
    return full_rows[rank::world].contiguous()


def gather_summaries(local: torch.Tensor, n: int, rank: int, world: int, out: torch.Tensor | None = None):
    """All-gather every rank's (count_r, REC) uint8 record block and return the
    (n, REC) records in scenario-id order (on every rank)."""
    if world == 1:
        return local[:n]
    m = (n + world - 1) // world
    buf = torch.zeros((m, REC), dtype=torch.uint8, device=local.device)
    buf[: local.shape[0]] = local
    gathered = torch.empty((world * m, REC), dtype=torch.uint8, device=local.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(gathered, buf)
    else:
        parts = list(gathered.chunk(world))
        dist.all_gather(parts, buf)
        gathered = torch.cat(parts)
    full = gathered.view(world, m, REC).transpose(0, 1).reshape(world * m, REC)[:n]
    if out is not None:
        out.copy_(full)
        return out
    return full


def reduce_segments(seg: torch.Tensor) -> torch.Tensor:
    """Sum the int64 segment histograms over ranks (in place)."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(seg, op=dist.ReduceOp.SUM)
    return seg
