"""Data-parallel sharding of independent codewords (north-star item 5).

Codewords share no state (``SPEC.md:343``), so a batch is split into contiguous
frame ranges, one per GPU/rank, exactly like the reference's ``np.array_split``
over worker threads (``bench.py:143``, ``decoder.py:467``).  Outputs are
concatenated in rank order.  There is no collective on the data path; in a
multi-process run the only communication is a barrier and a MAX reduction of
timings (bench.py) or an ``all_gather`` of results when a caller wants them on
one rank (``gather_outcomes``).
"""

from __future__ import annotations

import numpy as np

__all__ = ["shard_range", "shard_sizes", "gather_outcomes"]


def shard_sizes(total, world):
    """Per-rank frame counts of ``np.array_split(range(total), world)``."""
    if world < 1:
        raise ValueError("world size must be at least 1")
    base, extra = divmod(int(total), int(world))
    return [base + (1 if r < extra else 0) for r in range(world)]


def shard_range(total, world, rank):
    """Contiguous [start, stop) frame range of ``rank`` (array_split semantics)."""
    sizes = shard_sizes(total, world)
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    start = int(np.sum(sizes[:rank]))
    return start, start + sizes[rank]


def gather_outcomes(words, converged, iterations, group=None):
    """All-gather per-rank (words, converged, iterations) into global arrays on every rank.

    ``torch.distributed`` must be initialised (any backend: gloo exchanges host tensors,
    nccl device tensors on the rank's current GPU).  Words are bit-packed for the exchange
    (n/8 bytes per codeword); this is the only collective of the data-parallel path, and
    only for callers that want every frame's outcome on one rank.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    # NCCL exchanges device tensors (over NVLink on one node); gloo host tensors
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    n = words.shape[1]
    packed = np.packbits(words.astype(np.uint8), axis=1)
    local = torch.from_numpy(
        np.concatenate([packed, converged.astype(np.uint8)[:, None],
                        iterations.astype(np.int64).view(np.uint8).reshape(-1, 8)], axis=1)
    ).to(dev)
    counts = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts, group=group)
    width = local.shape[1]
    cap = int(max(c.item() for c in all_counts))
    padded = torch.zeros((cap, width), dtype=torch.uint8, device=dev)
    padded[: local.shape[0]] = local
    bufs = [torch.zeros_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded, group=group)
    rows = np.concatenate([b[: int(c.item())].cpu().numpy() for b, c in zip(bufs, all_counts)])
    nb = packed.shape[1]
    w = np.unpackbits(rows[:, :nb], axis=1)[:, :n]
    conv = rows[:, nb].astype(bool)
    iters = np.ascontiguousarray(rows[:, nb + 1: nb + 9]).view(np.int64).reshape(-1)
    return w, conv, iters
