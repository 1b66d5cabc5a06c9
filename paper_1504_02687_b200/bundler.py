"""Drop-in for ``histobundle.bundler`` (``/root/reference/pkg/src/histobundle/
bundler.py``): the ``bundle()`` entry point with the reference's signature,
parameters and output layout, running every iteration on the B200 kernels.

Host work is limited to what the reference also does once, outside its
timed loop: validation (``bundler.py:325-336``), the grid transform
(``model.py:233-272``), initial point counts (``bundler.py:82-85``) and the
per-edge offset vectors (``bundler.py:92-106``). Everything inside the loop
(``bundler.py:351-376``) and the final grid->world conversion with endpoint
pinning (``bundler.py:152-163``) runs as sm_100a kernels. There is no CPU
path.
"""

from __future__ import annotations

import math
import os
import time
from collections.abc import Sequence
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _native as N
from . import dist as D
from .engine import (MIN_STEP, BundleEngine, download, download_pinned, ordered_plan, ptr,
                     sample_counts, stream_ptr, upload, weight_plan)
from .model import (BundleConfig, DensityField, Graph, GridTransform, SampledEdge,
                    interaction_matrix, make_transform)

__all__ = [
    "MIN_STEP", "IterationMetrics", "BundleResult", "PackedPolylines", "bundle",
    "bundle_packed", "initial_sample", "density_at", "gradient_at", "advect_point",
    "laplacian_smooth", "resample", "used_cell_mask", "used_cell_count",
]


@dataclass
class IterationMetrics:
    """Per-iteration record (bundler.py:51-60)."""

    iteration: int
    bandwidth: float
    moved_points: int
    mean_displacement: float
    used_cells: int
    seconds: float


class PackedPolylines(Sequence):
    """``list[SampledEdge]``-compatible view of the packed result.

    The reference returns one ``SampledEdge`` per edge whose ``points`` are
    views into one packed (N,2) array (bundler.py:152-163). This sequence
    holds that packed array and builds the views on access, so 20M-edge
    results do not create 20M Python objects up front.
    """

    def __init__(self, world: np.ndarray, starts: np.ndarray, edge_base: int = 0):
        self.world = world
        self.starts = starts
        self.edge_base = int(edge_base)  # global index of the first edge held

    def __len__(self) -> int:
        return self.starts.shape[0] - 1

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError(i)
        return SampledEdge(self.edge_base + i, self.world[self.starts[i]:self.starts[i + 1]])


@dataclass
class BundleResult:
    """Output of a full bundling run (bundler.py:63-71)."""

    graph: Graph
    sampled_edges: PackedPolylines
    density: DensityField
    metrics: list[IterationMetrics]
    bundling_seconds: float


def _resolve(graph, config, bins, matrix):
    """bundler.py:325-336."""
    cfg = config if config is not None else BundleConfig()
    bins_arr = graph.bins if bins is None else np.ascontiguousarray(bins, dtype=np.int64)
    if bins_arr.shape[0] != graph.n_edges:
        raise ValueError("bins length does not match edge count")
    # (the reference's numpy indexing would wrap a negative bin; the device
    # layer offsets must not, so the Graph rule, model.py:138, applies here)
    if graph.n_edges and int(bins_arr.min()) < 0:
        raise ValueError("edge bins must be nonnegative")
    nbins = int(bins_arr.max()) + 1 if graph.n_edges else 1
    if matrix is None:
        matrix = interaction_matrix(nbins, cfg.alpha)
    matrix = np.asarray(matrix, dtype=np.float32)
    if matrix.shape[0] < nbins:
        raise ValueError(f"interaction matrix smaller than bin count {nbins}")
    if matrix.ndim != 2 or matrix.shape[0] != matrix.shape[1]:
        raise ValueError("interaction matrix must be square")
    return cfg, bins_arr, matrix


def _offset_vectors(src, dst, amount_cells):
    """Per-edge normal * amount of _offset_packed (bundler.py:92-106): the
    first/last sampled points are exactly the grid endpoints."""
    d = dst - src
    length = np.linalg.norm(d, axis=1)
    normal = np.zeros_like(d)
    ok = length > 0
    normal[ok, 0] = -d[ok, 1] / length[ok]
    normal[ok, 1] = d[ok, 0] / length[ok]
    return normal * amount_cells


@dataclass
class _Run:
    engine: BundleEngine
    transform: GridTransform
    edge_lo: int
    edge_hi: int
    records: list
    wall_seconds: float


def prepare_engine(graph: Graph, config: BundleConfig | None = None, *, bins=None,
                   matrix=None, _fixed_step: bool = False, group=None,
                   capacity_factor: float = 2.0, workers: int = 1, ordered: bool = False,
                   sync_free: bool = True):
    """Validate, transform, shard and sample (everything the reference does
    before its timed loop, bundler.py:325-346) and return
    ``(engine, transform, edge_lo, edge_hi)`` ready for ``engine.run()``.
    ``ordered`` forces the reference-order histogram path; ``sync_free=False``
    reads each iteration's point total on the host (no capacity retries, so
    the engine can be stepped and inspected iteration by iteration)."""
    cfg, bins_arr, matrix = _resolve(graph, config, bins, matrix)
    return _setup(graph, cfg, bins_arr, matrix, _fixed_step, group, capacity_factor,
                  workers=workers, force_ordered=ordered, sync_free=sync_free)


def _plan(graph, cfg, matrix, transform, force_ordered=False):
    """The histogram path for the WHOLE graph (every rank decides alike)."""
    w = np.asarray(graph.weights)
    if force_ordered:
        return ordered_plan(w)
    n0 = 0
    if graph.n_edges and not np.all(w == 1.0):
        pos = graph.positions
        n0 = int(sample_counts(transform.world_to_grid(pos[graph.sources]),
                               transform.world_to_grid(pos[graph.targets]), cfg.delta).sum())
    return weight_plan(w, matrix, n0)


def _setup(graph, cfg, bins_arr, matrix, fixed_step, group, capacity_factor, *,
           workers=1, force_ordered=False, sync_free=True):
    transform = make_transform(graph.positions, cfg.grid_size, cfg.padding_cells)
    rank, world = D.rank_world(group)
    multi = D.distributed(group)
    reduce_hist = (lambda h: D.all_reduce_sum(h, group)) if multi else None
    reduce_flags = (lambda t: D.all_reduce_max(t, group)) if multi else None
    plan = _plan(graph, cfg, matrix, transform, force_ordered)
    common = dict(fixed_step=fixed_step, reduce_hist=reduce_hist,
                  capacity_factor=capacity_factor, workers=workers,
                  reduce_flags=reduce_flags, sync_free=sync_free)
    if not multi and cfg.directed_offset_fraction == 0:
        # per-edge preparation on the device: the host uploads node positions
        # and endpoint indices once, the kernel computes the grid endpoints and
        # the reference's point counts, CUB scans them into `starts`
        dev = torch.device("cuda")
        node_pos = upload(graph.positions, dev)
        srcs = upload(graph.sources, dev)
        tgts = upload(graph.targets, dev)
        E = graph.n_edges
        src = torch.empty((E, 2), dtype=torch.float64, device=dev)
        dst = torch.empty((E, 2), dtype=torch.float64, device=dev)
        counts = torch.empty(max(E, 1), dtype=torch.int64, device=dev)
        starts = torch.empty(E + 1, dtype=torch.int64, device=dev)
        ws = torch.empty(int(N.lib().hb_scan_workspace_bytes(max(E, 1))), dtype=torch.uint8,
                         device=dev)
        s = stream_ptr()
        N.call("hb_edge_prepare", ptr(node_pos), ptr(srcs), ptr(tgts), E,
               float(transform.origin[0]), float(transform.origin[1]),
               float(transform.cell_size), float(cfg.delta), ptr(src), ptr(dst), ptr(counts), s)
        N.call("hb_scan_counts", ptr(counts), E, ptr(starts), ptr(ws), ws.numel(), s)
        eng = BundleEngine(src, dst, bins_arr, plan, matrix,
                           transform.shape, cfg, starts=starts, **common)
        eng.node_arrays = (node_pos, srcs, tgts)
        return eng, transform, 0, E
    pos = graph.positions
    src_all = transform.world_to_grid(pos[graph.sources])
    dst_all = transform.world_to_grid(pos[graph.targets])
    lo, hi = 0, graph.n_edges
    if world > 1:
        counts = sample_counts(src_all, dst_all, cfg.delta)
        lo, hi = D.shard_edges(counts, world)[rank]
    src = np.ascontiguousarray(src_all[lo:hi])
    dst = np.ascontiguousarray(dst_all[lo:hi])
    od = None
    if cfg.directed_offset_fraction > 0:
        od = _offset_vectors(src, dst, cfg.directed_offset_fraction
                             * max(transform.width, transform.height))
    shard = None
    if multi:
        shard = dict(rank=rank, world=world, group=group, edge_base=lo,
                     edges_total=graph.n_edges, weights=graph.weights, bins=bins_arr)
    eng = BundleEngine(src, dst, bins_arr[lo:hi], plan.slice(lo, hi),
                       matrix, transform.shape, cfg, offset_disp=od, shard=shard, **common)
    eng.node_arrays = None
    return eng, transform, lo, hi


def _run_engine(graph, cfg, bins_arr, matrix, fixed_step, on_iteration, group=None,
                capacity_factor=2.0, workers=1):
    t0 = time.perf_counter()
    # a per-iteration callback reads the metrics every iteration anyway, so
    # the run is synchronous (no capacity retry can replay callbacks)
    eng, transform, lo, hi = _setup(graph, cfg, bins_arr, matrix, fixed_step, group,
                                    capacity_factor, workers=workers,
                                    sync_free=on_iteration is None)
    if on_iteration is None:
        eng.run()
    else:
        def cb(e):
            recs = e.finish_metrics()
            on_iteration(_metrics(recs[-1:], group)[0])
        eng.run(on_iteration=cb)
    recs = eng.finish_metrics()
    return _Run(eng, transform, lo, hi, recs, time.perf_counter() - t0)


def _metrics(records, group=None) -> list[IterationMetrics]:
    """IterationMetrics (bundler.py:367-374); shard sums across ranks."""
    moved = np.array([r.moved_points for r in records], dtype=np.int64)
    interior = np.array([r.n_points - 2 * r.n_edges for r in records], dtype=np.int64)
    disp = np.array([r.disp for r in records], dtype=np.float64)
    moved, interior, disp = D.sum_host_arrays([moved, interior, disp], group)
    out = []
    for k, r in enumerate(records):
        out.append(IterationMetrics(
            iteration=r.iteration, bandwidth=r.bandwidth,
            moved_points=int(moved[k]),
            mean_displacement=float(disp[k] / interior[k]) if interior[k] else 0.0,
            used_cells=r.used_cells, seconds=r.seconds))
    return out


def bundle(graph: Graph, config: BundleConfig | None = None, *,
           bins: np.ndarray | None = None, matrix: np.ndarray | None = None,
           workers: int = 1,
           on_iteration: Callable[[IterationMetrics], None] | None = None,
           _fixed_step: bool = False, group=None) -> BundleResult:
    """Run the full bundling pipeline on the GPU (reference ``bundler.py:311-380``).

    Same signature and result as the reference. Parallelism is the device's;
    ``workers`` keeps its reference meaning only where it changes results:
    the number of edge partitions whose float32 histograms the reference
    sums in order (``raster.py:85-94``), which matters for inexact layer
    weights (repulsive matrices, fractional weights) and is reproduced
    exactly. With ``torch.distributed`` initialised, edges are sharded
    across ranks; rank 0 returns the full result and every other rank its
    own edge shard (``sampled_edges.edge_base`` = its first edge).
    ``graph`` may be a reference ``histobundle.model.Graph``.
    """
    cfg, bins_arr, matrix = _resolve(graph, config, bins, matrix)
    if (on_iteration is None and not D.distributed(group)
            and os.environ.get("HB_STREAM_OUT", "1") != "0"):
        # one GPU: the last iteration streams its polylines to the host while
        # the remaining edge chunks are still being advected
        t0 = time.perf_counter()
        eng, tr, _, _ = _setup(graph, cfg, bins_arr, matrix, _fixed_step, group, 2.0,
                               workers=workers)
        if eng.node_arrays is not None:
            world, recs = eng.run_streamed(tr.origin, tr.cell_size, *eng.node_arrays)
            starts = download(eng.starts)
            field = DensityField(tr, download(eng.field))
            metrics = _metrics(recs, group)
            return BundleResult(graph, PackedPolylines(world, starts), field, metrics,
                                sum(m.seconds for m in metrics))
        recs = eng.run()
        run = _Run(eng, tr, 0, graph.n_edges, recs, time.perf_counter() - t0)
    else:
        run = _run_engine(graph, cfg, bins_arr, matrix, _fixed_step, on_iteration, group,
                          workers=workers)
    eng, tr = run.engine, run.transform
    if eng.node_arrays is not None:
        world_dev = eng.world_points_nodes(tr.origin, tr.cell_size, *eng.node_arrays)
    else:
        pos = graph.positions
        src_w = pos[graph.sources[run.edge_lo:run.edge_hi]]
        dst_w = pos[graph.targets[run.edge_lo:run.edge_hi]]
        world_dev = eng.world_points(tr.origin, tr.cell_size, src_w, dst_w)
    edge_base = 0
    if not D.distributed(group):
        world, starts = download_pinned(world_dev), download(eng.starts)
    else:
        got = D.gather_polylines(world_dev, eng.starts, group)
        if got is None:  # not rank 0: this rank's own shard
            world, starts = download_pinned(world_dev), download(eng.starts)
            edge_base = run.edge_lo
        else:
            world, starts = got
    field = DensityField(tr, download(eng.field))
    metrics = _metrics(run.records, group)
    return BundleResult(graph, PackedPolylines(world, starts, edge_base), field, metrics,
                        sum(m.seconds for m in metrics))


def bundle_packed(graph: Graph, config: BundleConfig | None = None, *, bins=None,
                  matrix=None, _fixed_step: bool = False, group=None,
                  capacity_factor: float = 2.0, workers: int = 1):
    """Like :func:`bundle` but keeps the result on the device: returns
    ``(engine, transform, metrics)`` with the shard's packed grid-space
    points in ``engine.packed_points()`` (no host copies, no gathers)."""
    cfg, bins_arr, matrix = _resolve(graph, config, bins, matrix)
    run = _run_engine(graph, cfg, bins_arr, matrix, _fixed_step, None, group,
                      capacity_factor, workers=workers)
    return run.engine, run.transform, _metrics(run.records, group)


# ---------------------------------------------------------------------------
# per-operation surface (bundler.py:169-305), each backed by the kernels


def _dev():
    N.lib()
    if not torch.cuda.is_available():
        raise N.NativeError("a CUDA device is required")
    return torch.device("cuda")


def _polyline_device(points: np.ndarray):
    pts = torch.from_numpy(np.ascontiguousarray(points, dtype=np.float64)).to(_dev())
    starts = torch.tensor([0, pts.shape[0]], dtype=torch.int64, device=pts.device)
    return pts, starts


def initial_sample(graph: Graph, transform: GridTransform,
                   delta: float) -> list[SampledEdge]:
    """bundler.py:169-179 on the device."""
    if delta <= 0:
        raise ValueError("delta must be positive")
    from .engine import sample_counts
    src = transform.world_to_grid(graph.positions[graph.sources])
    dst = transform.world_to_grid(graph.positions[graph.targets])
    counts = sample_counts(src, dst, delta)
    starts = np.zeros(graph.n_edges + 1, dtype=np.int64)
    np.cumsum(counts, out=starts[1:])
    dev = _dev()
    st = torch.from_numpy(starts).to(dev)
    pts = torch.empty((int(starts[-1]), 2), dtype=torch.float64, device=dev)
    s = stream_ptr()
    src_d = torch.from_numpy(np.ascontiguousarray(src)).to(dev)
    dst_d = torch.from_numpy(np.ascontiguousarray(dst)).to(dev)
    N.call("hb_sample_fill", ptr(src_d), ptr(dst_d), ptr(st), graph.n_edges, ptr(pts), s)
    out = torch.empty_like(pts)
    sw = torch.from_numpy(np.ascontiguousarray(graph.positions[graph.sources])).to(dev)
    dw = torch.from_numpy(np.ascontiguousarray(graph.positions[graph.targets])).to(dev)
    N.call("hb_to_world", ptr(pts), ptr(st), graph.n_edges, transform.origin[0],
           transform.origin[1], transform.cell_size, ptr(sw), ptr(dw), ptr(out), s)
    return list(PackedPolylines(out.cpu().numpy(), starts))


def _probe(field: DensityField, layer: int, p, want_grad: bool):
    rho = torch.from_numpy(np.ascontiguousarray(field.values[layer], dtype=np.float32)).to(_dev())
    xy = torch.tensor([[float(p[0]), float(p[1])]], dtype=torch.float64, device=rho.device)
    val = torch.empty(1, dtype=torch.float64, device=rho.device)
    grad = torch.empty((1, 2), dtype=torch.float64, device=rho.device)
    nv, nu = rho.shape
    N.call("hb_probe", ptr(rho), nv, nu, ptr(xy), 1, ptr(val), ptr(grad) if want_grad else None,
           stream_ptr())
    return val.cpu().numpy()[0], grad.cpu().numpy()[0]


def density_at(field: DensityField, layer: int, p) -> float:
    """Bilinear density at a grid point (bundler.py:203-206)."""
    return float(_probe(field, layer, p, False)[0])


def gradient_at(field: DensityField, layer: int, p) -> np.ndarray:
    """Interpolated central-difference gradient (bundler.py:209-217)."""
    return np.array(_probe(field, layer, p, True)[1])


def advect_point(p, field: DensityField, layer: int, h: float, epsilon: float = 1e-8,
                 min_step: float = MIN_STEP, fixed_step: bool = False) -> np.ndarray:
    """One point up the density gradient (bundler.py:220-254): run the
    advection kernel on a 3-point polyline whose middle point is ``p``."""
    rho = torch.from_numpy(np.ascontiguousarray(field.values[layer], dtype=np.float32)).to(_dev())
    nv, nu = rho.shape
    x, y = float(p[0]), float(p[1])
    pts, starts = _polyline_device(np.array([[x, y]] * 3))
    out = torch.empty_like(pts)
    layer0 = torch.zeros(1, dtype=torch.int32, device=pts.device)
    moved = torch.zeros(1, dtype=torch.int64, device=pts.device)
    part = torch.zeros(int(N.lib().hb_advect_partials()), dtype=torch.float64, device=pts.device)
    N.call("hb_advect_laplacian", ptr(pts), ptr(out), ptr(starts), 1, 3, ptr(layer0), ptr(rho), None,
           1, nv, nu, float(h), float(epsilon), float(min_step), int(bool(fixed_step)), 0.5, 0,
           1.0, None, None, ptr(moved), ptr(part), stream_ptr())
    return out.cpu().numpy()[1].copy()


def laplacian_smooth(polyline: SampledEdge, factor: float = 0.5, passes: int = 1) -> None:
    """Jacobi Laplacian smoothing in place, endpoints fixed (bundler.py:257-269)."""
    if not (0.0 < factor <= 1.0):
        raise ValueError("factor must be in (0, 1]")
    pts, starts = _polyline_device(polyline.points)
    n = pts.shape[0]
    moved = torch.zeros(1, dtype=torch.int64, device=pts.device)
    part = torch.zeros(int(N.lib().hb_advect_partials()), dtype=torch.float64, device=pts.device)
    if passes > 0:  # in place; h < 0: Laplacian sweeps only
        N.call("hb_advect_laplacian", ptr(pts), ptr(pts), ptr(starts), 1, n, None, None, None, 1, 3, 3,
               -1.0, 1e-8, MIN_STEP, 0, float(factor), int(passes), 1.0, None, None, ptr(moved),
               ptr(part), stream_ptr())
    polyline.points[...] = pts.cpu().numpy()


def resample(polyline: SampledEdge, delta: float) -> None:
    """Re-space one polyline (bundler.py:272-289) with the resample kernels."""
    if delta <= 0:
        raise ValueError("delta must be positive")
    pts, starts = _polyline_device(polyline.points)
    n = pts.shape[0]
    counts = torch.empty(1, dtype=torch.int64, device=pts.device)
    pos = torch.empty(n, dtype=torch.int32, device=pts.device)
    s = stream_ptr()
    N.call("hb_resample_count", ptr(pts), ptr(starts), 1, float(delta), ptr(counts), ptr(pos), s)
    new_starts = torch.empty(2, dtype=torch.int64, device=pts.device)
    ws = torch.empty(int(N.lib().hb_scan_workspace_bytes(1)), dtype=torch.uint8, device=pts.device)
    N.call("hb_scan_counts", ptr(counts), 1, ptr(new_starts), ptr(ws), ws.numel(), s)
    m = int(new_starts[1].item())
    out = torch.empty((m, 2), dtype=torch.float64, device=pts.device)
    N.call("hb_resample_emit", ptr(pts), ptr(starts), 1, n, ptr(pos), ptr(new_starts), ptr(out),
           None, None, None, 1, 1, None, None, s)
    polyline.points = out.cpu().numpy()


def used_cell_mask(field: DensityField, layer: int, rel_threshold: float = 0.01) -> np.ndarray:
    """bundler.py:292-299 (host comparison on the returned field)."""
    rho = field.values[layer]
    peak = float(rho.max(initial=0.0))
    if peak <= 0:
        return np.zeros_like(rho, dtype=bool)
    return rho > np.float32(rel_threshold * peak)


def used_cell_count(field: DensityField, rel_threshold: float = 0.01) -> int:
    """bundler.py:302-305 on the device (layer peaks + threshold count)."""
    vals = torch.from_numpy(np.ascontiguousarray(field.values, dtype=np.float32)).to(_dev())
    nb, nv, nu = vals.shape
    peak = vals.reshape(nb, -1).amax(dim=1).clamp_min(0.0).contiguous()
    cnt = torch.zeros(1, dtype=torch.int64, device=vals.device)
    N.call("hb_used_cells", ptr(vals), ptr(peak), nb, nv, nu, float(rel_threshold), ptr(cnt),
           stream_ptr())
    return int(cnt.item())
