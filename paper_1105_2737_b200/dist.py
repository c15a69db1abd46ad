"""Multi-GPU plumbing over torch.distributed (one process per GPU), for the
two paths that shard:

* batches of independent fields: rank r owns the contiguous field range
  ``field_range(r, world, per_rank)`` — no collective on the data path;
* the covariance estimator (grf::estimate_covariance, src/stats.cpp:39-97):
  ranks own contiguous ranges of 1024-sample chunks, compute their chunk
  partials on their device (grfc_covariance_partials), the partials are
  gathered, and every rank merges them in chunk order (Kahan,
  grfc_covariance_merge) — bit-identical to the single-device estimate for
  any world size, as the reference's worker count is (test_stats.cpp:43-56).

The data-path compute is the C-ABI's; this module only partitions work and
moves partial sums. `partials_fn` / `merge_fn` are injectable so the
partition and the ordered merge are testable on CPU (gloo) with the oracle.
"""
from typing import Callable, Optional, Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import grfc


def field_range(rank: int, world: int, per_rank: int) -> Tuple[int, int]:
    """First field and count of `rank` when each of `world` ranks generates per_rank fields."""
    return rank * per_rank, per_rank


def chunk_range(rank: int, world: int, samples: int, chunk: int = grfc.COV_CHUNK) -> Tuple[int, int]:
    """Contiguous chunk range (first, count) of `rank` for a `samples`-sample estimate."""
    total = (samples + chunk - 1) // chunk
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def kahan_merge_numpy(partials: np.ndarray, samples: int) -> np.ndarray:
    """Chunk-ordered Kahan merge x (1/M) (stats.cpp:84-96) — the same IEEE steps as
    grfc_covariance_merge."""
    est = np.zeros_like(partials[0])
    comp = np.zeros_like(partials[0])
    for acc in partials:
        y = acc - comp
        t = est + y
        comp = (t - est) - y
        est = t
    return est * (1.0 / samples)


def estimate_covariance_distributed(plan: Optional["grfc.Plan"], seed: int, samples: int, reference,
                                    group=None,
                                    partials_fn: Optional[Callable[[int, int], torch.Tensor]] = None,
                                    merge_fn: Optional[Callable[[torch.Tensor, int], torch.Tensor]] = None,
                                    points: Optional[int] = None) -> torch.Tensor:
    """Estimate over all ranks of `group`; every rank returns the full estimate.

    Default (GPU): partials via plan.covariance_partials_tensor on this rank's
    device, merge via plan.covariance_merge_tensor. Collectives: one
    all_gather of the (padded) partial stacks.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    first, count = chunk_range(rank, world, samples)
    if partials_fn is None:
        def partials_fn(c0, n):  # noqa: E306
            return plan.covariance_partials_tensor(seed, samples, c0, n, reference).reshape(n, -1)
    if merge_fn is None:
        def merge_fn(parts, m):  # noqa: E306
            return plan.covariance_merge_tensor(parts.reshape((parts.shape[0],) + plan.counts), m).reshape(-1)
    P = points if points is not None else plan.points
    mine = partials_fn(first, count) if count else None
    if world == 1:
        return merge_fn(mine, samples)
    # pad every rank's stack to the largest count, gather, drop the padding in rank order
    maxc = chunk_range(0, world, samples)[1]
    # a rank that owns no chunks still joins the all_gather with a buffer on the
    # backend's device (NCCL: this rank's GPU; mixing CPU and CUDA buffers hangs)
    if mine is not None:
        dev = mine.device
    elif dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    else:
        dev = torch.device("cpu")
    buf = torch.zeros((maxc, P), dtype=torch.float64, device=dev)
    if count:
        buf[:count] = mine
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf, group=group)
    parts = torch.cat([g[:chunk_range(r, world, samples)[1]] for r, g in enumerate(gathered)])
    return merge_fn(parts, samples)
