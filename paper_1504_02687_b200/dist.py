"""Multi-GPU plumbing: edge sharding and the per-iteration histogram sum.

The reference parallelises over contiguous edge ranges on threads and merges
private histograms in worker order (``_parallel.py:20-43``,
``raster.py:85-94``). Here each rank (one process per GPU,
``torch.distributed`` over NCCL) owns a contiguous edge range balanced by
initial point count, splats it into a local int32 group histogram, and one
all-reduce per iteration sums the histograms; integer sums are associative,
so every rank then holds the bit-exact global histogram and smooths it
redundantly. Metrics are summed at the end; polylines are
gathered to every rank only when the caller materialises them.

Everything here also runs on CPU tensors with the gloo backend (tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["rank_world", "shard_edges", "all_reduce_sum", "sum_host_arrays",
           "gather_polylines"]


def rank_world(group=None) -> tuple[int, int]:
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def shard_edges(point_counts: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous [lo, hi) edge ranges, one per rank, splitting the total
    initial point count as evenly as edge boundaries allow. A pure function
    of (counts, world): every rank computes the same table."""
    n = int(point_counts.shape[0])
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(world - 1, 0)
    cum = np.concatenate([[0], np.cumsum(point_counts, dtype=np.int64)])
    total = int(cum[-1])
    cuts = [0]
    for r in range(1, world):
        target = total * r // world
        k = int(np.searchsorted(cum, target, side="left"))
        cuts.append(min(max(k, cuts[-1]), n))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def all_reduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum over ranks (NCCL int32 all-reduce on GPUs; device tensors
    are staged through the host for a gloo group)."""
    if t.is_cuda and dist.get_backend(group) != "nccl":
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
        return t
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def _backend_device(group=None) -> torch.device:
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def sum_host_arrays(arrays: list[np.ndarray], group=None) -> list[np.ndarray]:
    """Element-wise sum of small host arrays over ranks (one collective)."""
    _, world = rank_world(group)
    if world == 1:
        return arrays
    dev = _backend_device(group)
    out = []
    for a in arrays:
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        out.append(t.cpu().numpy())
    return out


def gather_polylines(points: torch.Tensor, starts: torch.Tensor, group=None):
    """All ranks' packed polylines concatenated in rank order (= edge order).

    Returns host numpy ``(world_points (N,2) f64, starts (E+1) i64)``."""
    _, world = rank_world(group)
    if world == 1:
        return points.cpu().numpy(), starts.cpu().numpy()
    dev = _backend_device(group)
    pts = points.to(dev)
    st = starts.to(dev)
    sizes = torch.tensor([pts.shape[0], st.shape[0] - 1], dtype=torch.int64, device=dev)
    all_sizes = [torch.empty_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [tuple(int(v) for v in s.cpu()) for s in all_sizes]
    max_n = max(s[0] for s in all_sizes)
    max_e = max(s[1] for s in all_sizes)
    pad_p = torch.zeros((max_n, 2), dtype=pts.dtype, device=dev)
    pad_p[: pts.shape[0]] = pts
    pad_s = torch.zeros(max_e + 1, dtype=st.dtype, device=dev)
    pad_s[: st.shape[0]] = st
    gp = [torch.empty_like(pad_p) for _ in range(world)]
    gs = [torch.empty_like(pad_s) for _ in range(world)]
    dist.all_gather(gp, pad_p, group=group)
    dist.all_gather(gs, pad_s, group=group)
    pieces, st_pieces, base = [], [np.zeros(1, dtype=np.int64)], 0
    for (n, e), p, s in zip(all_sizes, gp, gs):
        pieces.append(p[:n].cpu().numpy())
        st_pieces.append(s[1: e + 1].cpu().numpy() + base)
        base += n
    return np.concatenate(pieces), np.concatenate(st_pieces)
