"""Request sharding across the GPUs of one box.

The compression path shards naturally: each request's compression touches
only its own KV and blocks (reference engine.py:502-505 transitions one
handle at a time; there is no cross-request reduction). So:

* synthetic batches (configs 2-4) are split across ranks up front --
  ``lpt_shard`` balances raw tokens with longest-processing-time-first;
* a serving trace (config 5) assigns every arrival to one rank with a
  *replicated* decision: once per scheduler tick all ranks all-gather a tiny
  occupancy vector (``OccupancyExchange``, int64[4] per rank: free pool
  bytes, queued raw bytes, in-flight requests, compress backlog tokens) and
  then run the same deterministic rule (``assign_arrivals``), so no
  broadcast of decisions is needed.

NCCL carries only that all-gather (4 x int64 per rank per tick, latency
bound); the compression kernels themselves never communicate.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

FREE, QUEUED, INFLIGHT, BACKLOG = range(4)


def lpt_shard(token_counts: Sequence[int], world: int) -> list[list[int]]:
    """Indices per rank; longest first to the least-loaded rank (ties: lowest rank).

    Deterministic, so every rank computes the same partition without talking.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(token_counts)), key=lambda i: (-int(token_counts[i]), i))
    load = [0] * world
    parts: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        parts[r].append(i)
        load[r] += int(token_counts[i])
    return [sorted(p) for p in parts]


def assign_arrivals(occupancy: Sequence[Sequence[int]], raw_bytes: Sequence[int]) -> list[int]:
    """Rank for each arrival of this tick, in arrival order.

    Rule: the rank with the largest ``free_bytes - queued_raw_bytes``
    (ties to the lowest rank); the chosen rank's copy of the occupancy is
    updated before the next arrival, so one tick's arrivals spread out.
    """
    occ = [list(map(int, row)) for row in occupancy]
    out = []
    for b in raw_bytes:
        r = max(range(len(occ)), key=lambda k: (occ[k][FREE] - occ[k][QUEUED], -k))
        out.append(r)
        occ[r][QUEUED] += int(b)
        occ[r][INFLIGHT] += 1
    return out


@dataclass
class OccupancyExchange:
    """All-gather of int64[4] occupancy per rank over torch.distributed (NCCL on GPUs)."""

    group: object = None
    device: object = None

    def gather(self, free_bytes: int, queued_raw: int, inflight: int, backlog_tokens: int):
        import torch
        import torch.distributed as dist

        if not dist.is_available() or not dist.is_initialized():
            return [[free_bytes, queued_raw, inflight, backlog_tokens]]
        # NCCL moves device tensors; gloo (CPU tests) moves host tensors
        dev = self.device if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        mine = torch.tensor([free_bytes, queued_raw, inflight, backlog_tokens], dtype=torch.int64,
                            device=dev)
        world = dist.get_world_size(self.group)
        out = torch.empty(world * 4, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(out, mine, group=self.group)
        return out.view(world, 4).tolist()
