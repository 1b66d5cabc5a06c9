"""Multi-GPU plumbing: edge sharding and the per-iteration histogram sum.

The reference parallelises over contiguous edge ranges on threads and merges
private histograms in worker order (``_parallel.py:20-43``,
``raster.py:85-94``). Here each rank (one process per GPU,
``torch.distributed`` over NCCL) owns a contiguous edge range balanced by
initial point count, splats it into a local int32 group histogram, and one
all-reduce per iteration sums the histograms; integer sums are associative,
so every rank then holds the bit-exact global histogram and smooths it
redundantly. Metrics are summed at the end; polylines are
gathered to rank 0 only when the caller materialises them.

Everything here also runs on CPU tensors with the gloo backend (tests).
"""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["rank_world", "distributed", "shard_edges", "all_reduce_sum", "all_reduce_max",
           "all_to_all_var", "all_gather_columns", "sum_host_arrays", "gather_polylines"]


def rank_world(group=None) -> tuple[int, int]:
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def distributed(group=None) -> bool:
    """Whether the collective path runs: more than one rank, or a 1-rank
    process group with HB_FORCE_DIST=1 (so the NCCL branch is exercised on a
    single GPU: an all-reduce over one rank is the identity)."""
    if not (dist.is_available() and dist.is_initialized()):
        return False
    return dist.get_world_size(group) > 1 or os.environ.get("HB_FORCE_DIST") == "1"


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


def all_reduce_max(t: torch.Tensor, group=None) -> torch.Tensor:
    """Element-wise maximum of a small host tensor over ranks (status words,
    bounds spans): every rank gets the same value and takes the same branch."""
    dev = _backend_device(group)
    d = t.to(dev)
    dist.all_reduce(d, op=dist.ReduceOp.MAX, group=group)
    return d.cpu()


def all_to_all_var(t: torch.Tensor, send_counts: list[int], group=None) -> torch.Tensor:
    """Variable-size all-to-all of the rows of ``t`` (rank r gets the
    ``send_counts[r]`` rows starting at ``sum(send_counts[:r])``).  The
    received blocks are concatenated in sender-rank order."""
    dev = _backend_device(group)
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(v) for v in rc.cpu()]
    src = t.to(dev)
    out = torch.empty((sum(recv_counts),) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
    dist.all_to_all_single(out, src, recv_counts, list(send_counts), group=group)
    return out.to(t.device)


def all_gather_columns(t: torch.Tensor, sizes: list[int], group=None) -> torch.Tensor:
    """Concatenate every rank's (B, sizes[r]) block along dim 1, in rank order."""
    dev = _backend_device(group)
    width = max(sizes)
    pad = torch.zeros((t.shape[0], width), dtype=t.dtype, device=dev)
    pad[:, : t.shape[1]] = t.to(dev)
    parts = [torch.empty_like(pad) for _ in sizes]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:, :n] for p, n in zip(parts, sizes)], dim=1).to(t.device)


def _backend_device(group=None) -> torch.device:
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def sum_host_arrays(arrays: list[np.ndarray], group=None) -> list[np.ndarray]:
    """Element-wise sum of small host arrays over ranks (one collective)."""
    if not distributed(group):
        return arrays
    dev = _backend_device(group)
    out = []
    for a in arrays:
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        out.append(t.cpu().numpy())
    return out


def _count_d2h(*arrays) -> None:
    """Host-bound bytes of the public API (bench.py's e2e accounting)."""
    from .engine import IO_BYTES
    IO_BYTES["d2h"] += sum(int(a.nbytes) for a in arrays)


def gather_polylines(points: torch.Tensor, starts: torch.Tensor, group=None, root: int = 0):
    """Every rank's packed polylines concatenated in rank order (= edge
    order) on ``root`` only: the point counts are all-gathered
    (one tiny collective), then each rank sends its exact-size arrays to the
    root point to point.  Returns host numpy ``(world_points (N,2) f64,
    starts (E+1) i64)`` on the root and ``None`` elsewhere."""
    rank, world = rank_world(group)
    if not distributed(group):
        return points.cpu().numpy(), starts.cpu().numpy()
    dev = _backend_device(group)
    sizes = torch.tensor([points.shape[0], starts.shape[0] - 1], dtype=torch.int64, device=dev)
    all_sizes = [torch.empty_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [tuple(int(v) for v in s.cpu()) for s in all_sizes]
    groot = root if group is None else dist.get_global_rank(group, root)
    if rank != root:
        if all_sizes[rank][0]:
            dist.send(points.contiguous().to(dev), dst=groot, group=group)
        dist.send(starts.contiguous().to(dev), dst=groot, group=group)
        return None
    pieces, st_pieces, base = [], [np.zeros(1, dtype=np.int64)], 0
    for r, (n, e) in enumerate(all_sizes):
        if r == root:
            p, s = points.to(dev), starts.to(dev)
        else:
            src = r if group is None else dist.get_global_rank(group, r)
            p = torch.empty((n, 2), dtype=points.dtype, device=dev)
            if n:
                dist.recv(p, src=src, group=group)
            s = torch.empty(e + 1, dtype=starts.dtype, device=dev)
            dist.recv(s, src=src, group=group)
        pieces.append(p[:n].cpu().numpy())
        st_pieces.append(s[1: e + 1].cpu().numpy() + base)
        _count_d2h(pieces[-1], st_pieces[-1])
        base += n
    return np.concatenate(pieces), np.concatenate(st_pieces)
