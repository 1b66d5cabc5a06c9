"""CPU ORACLE driver -- TEST INFRASTRUCTURE, never the product path.

Runs the reference bundling loop (``/root/reference/pkg/src/histobundle/
bundler.py:311-380``) on top of ``hb_oracle.c``, a plain-C restatement of the
reference's numba kernels. Worker threads mirror ``_parallel.py:20-43``
(contiguous edge ranges, results merged in ascending worker order; ctypes
releases the GIL for the C calls), so the oracle is bit-identical to the
reference for the same ``workers`` value.

Who may import this module: ``tests/``, ``__graft_entry__.smoke()`` (as the
checker) and ``bench.py`` (``cpu_baseline`` leg and ``--impl reference``).

Parity of the oracle itself is pinned against the reference by
``tests/test_oracle.py`` using ``tests/golden`` (made by running the
reference, see ``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libhb_oracle.so")
_lib = None

MIN_STEP = 0.25  # bundler.py:48


def build() -> str:
    """Compile hb_oracle.c (gcc, -ffp-contract=off) into oracle/_build."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        sigs = {
            "orc_fill_samples": [P, P, P, I64, P],
            "orc_accumulate": [P, P, P, I, I, I, P, I64, I64],
            "orc_accumulate_counts": [P, P, P, P, I, I, P, I64, I64],
            "orc_box_filter": [P, P, I, I, I, P],
            "orc_smooth_layers": [P, P, I, I, P, I, I, I, P, P],
            "orc_bilinear": [P, I, I, D, D],
            "orc_gradient": [P, I, I, D, D, P],
            "orc_advect": [P, P, P, P, I, I, I, D, D, D, I, I64, I64, P, P],
            "orc_resample_count": [P, P, D, P, I64, I64],
            "orc_resample_emit": [P, P, D, P, P, I64, I64],
            "orc_laplacian": [P, P, D, I, P, I64, I64],
            "orc_used_cells": [P, I, I, I, D],
            "orc_offset": [P, P, P, I64],
        }
        for name, argt in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = argt
            fn.restype = None
        L.orc_bilinear.restype = D
        L.orc_used_cells.restype = I64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# _parallel.py:20-43


def partition_ranges(n: int, workers: int) -> list[tuple[int, int]]:
    if n <= 0:
        return [(0, 0)]
    w = max(1, min(int(workers), n))
    return [(i * n // w, (i + 1) * n // w) for i in range(w)]


_POOLS: dict[int, ThreadPoolExecutor] = {}


def map_partitions(fn, n: int, workers: int):
    parts = partition_ranges(n, workers)
    if len(parts) == 1:
        return [fn(*parts[0])]
    pool = _POOLS.get(len(parts))
    if pool is None:
        pool = _POOLS[len(parts)] = ThreadPoolExecutor(max_workers=len(parts))
    futs = [pool.submit(fn, lo, hi) for lo, hi in parts]
    return [f.result() for f in futs]


# ---------------------------------------------------------------------------
# host restatements (model.py / raster.py)


def box_widths(sigma: float, passes: int) -> list[int]:
    """raster.py:172-193."""
    n = passes
    w_ideal = math.sqrt(12.0 * sigma * sigma / n + 1.0)
    w_lo = int(math.floor(w_ideal))
    if w_lo % 2 == 0:
        w_lo -= 1
    w_lo = max(w_lo, 1)
    m_ideal = (12.0 * sigma * sigma - n * w_lo * w_lo - 4.0 * n * w_lo
               - 3.0 * n) / (-4.0 * w_lo - 4.0)
    m = min(max(int(round(m_ideal)), 0), n)
    return [w_lo] * m + [w_lo + 2] * (n - m)


def transform(positions: np.ndarray, grid_size: int, pad: float):
    """model.py:233-272 -> (origin_x, origin_y, cell, width, height)."""
    lo = positions.min(axis=0)
    hi = positions.max(axis=0)
    ex = float(hi[0] - lo[0])
    ey = float(hi[1] - lo[1])
    if ex == 0.0 and ey == 0.0:
        cell = 1.0
        width = height = int(math.floor(2.0 * pad)) + 1
    else:
        span = grid_size - 2.0 * pad - 1.0
        if ex >= ey:
            width = int(grid_size)
            cell = ex / span
            height = int(math.floor(ey / cell + 2.0 * pad)) + 1
        else:
            height = int(grid_size)
            cell = ey / span
            width = int(math.floor(ex / cell + 2.0 * pad)) + 1
    return (float(lo[0]) - pad * cell, float(lo[1]) - pad * cell, cell,
            width, height)


# ---------------------------------------------------------------------------
# stage wrappers


def sample(positions, sources, targets, origin, cell, delta):
    """bundler.py:77-89 (host numpy part) + fill_samples."""
    org = np.asarray(origin)
    src = np.ascontiguousarray((positions[sources] - org) / cell)
    dst = np.ascontiguousarray((positions[targets] - org) / cell)
    seg = np.linalg.norm(dst - src, axis=1)
    counts = np.maximum(np.ceil(seg / delta).astype(np.int64), 1) + 1
    starts = np.zeros(sources.shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=starts[1:])
    pts = np.empty((int(starts[-1]), 2), dtype=np.float64)
    if sources.shape[0]:
        lib().orc_fill_samples(_p(src), _p(dst), _p(starts), sources.shape[0],
                               _p(pts))
    return pts, starts, src, dst


def offset_disp(pts, starts, amount_cells):
    """bundler.py:92-106 per-edge displacement vectors."""
    firsts = pts[starts[:-1]]
    lasts = pts[starts[1:] - 1]
    d = lasts - firsts
    length = np.linalg.norm(d, axis=1)
    normal = np.zeros_like(d)
    ok = length > 0
    normal[ok, 0] = -d[ok, 1] / length[ok]
    normal[ok, 1] = d[ok, 0] / length[ok]
    return np.ascontiguousarray(normal * amount_cells)


def accumulate(pts, starts, layer_w, shape, workers=1):
    """raster.py:70-94 (bounds check + private float32 buffers, ordered sum)."""
    nv, nu = shape
    nb = layer_w.shape[1]
    n_edges = starts.size - 1
    if pts.size:
        xmin, xmax = pts[:, 0].min(), pts[:, 0].max()
        ymin, ymax = pts[:, 1].min(), pts[:, 1].max()
        if xmin <= -0.5 or ymin <= -0.5 or xmax >= nu - 0.5 or ymax >= nv - 0.5:
            raise ValueError("sample out of bounds")
    lw = np.ascontiguousarray(layer_w, dtype=np.float32)

    def run(lo, hi):
        buf = np.zeros((nb, nv, nu), dtype=np.float32)
        lib().orc_accumulate(_p(pts), _p(starts), _p(lw), nb, nv, nu, _p(buf),
                             lo, hi)
        return buf

    bufs = map_partitions(run, n_edges, workers)
    out = bufs[0]
    for b in bufs[1:]:
        out += b
    return out


def accumulate_counts(pts, starts, group, shape, nbins, weight=None):
    nv, nu = shape
    out = np.zeros((nbins, nv, nu), dtype=np.int32)
    g = np.ascontiguousarray(group, dtype=np.int64)
    w = None if weight is None else np.ascontiguousarray(weight, dtype=np.int32)
    lib().orc_accumulate_counts(_p(pts), _p(starts), _p(g),
                                None if w is None else _p(w), nv, nu, _p(out),
                                0, starts.size - 1)
    return out


def box_filter(layer: np.ndarray, radius: int) -> np.ndarray:
    layer = np.ascontiguousarray(layer, dtype=np.float32)
    nv, nu = layer.shape
    out = np.empty_like(layer)
    table = np.empty((nv, nu), dtype=np.float64)
    lib().orc_box_filter(_p(layer), _p(out), nv, nu, int(radius), _p(table))
    return out


def smooth(values: np.ndarray, sigma: float, passes: int = 3, workers: int = 1):
    """raster.py:203-219 (one worker per layer when B > 1)."""
    widths = np.asarray(box_widths(sigma, passes), dtype=np.int32)
    vals = np.ascontiguousarray(values, dtype=np.float32)
    nb, nv, nu = vals.shape
    out = np.empty_like(vals)

    def run(lo, hi):
        scratch = np.empty((nv, nu), dtype=np.float32)
        table = np.empty((nv, nu), dtype=np.float64)
        lib().orc_smooth_layers(_p(vals), _p(out), nv, nu, _p(widths),
                                len(widths), lo, hi, _p(scratch), _p(table))

    map_partitions(run, nb, workers if nb > 1 else 1)
    return out


def advect(pts, starts, edge_layer, rho, h, eps, fixed_step, workers=1):
    """bundler.py:127-138."""
    nb, nv, nu = rho.shape
    el = np.ascontiguousarray(edge_layer, dtype=np.int64)
    r = np.ascontiguousarray(rho, dtype=np.float32)

    def run(lo, hi):
        ri = np.zeros(2, dtype=np.int64)
        rd = np.zeros(1, dtype=np.float64)
        lib().orc_advect(_p(pts), _p(starts), _p(el), _p(r), nb, nv, nu,
                         float(h), float(eps), MIN_STEP, int(bool(fixed_step)),
                         lo, hi, _p(ri), _p(rd))
        return int(ri[0]), int(ri[1]), float(rd[0])

    res = map_partitions(run, starts.size - 1, workers)
    return (sum(r[0] for r in res), sum(r[1] for r in res),
            sum(r[2] for r in res))


def laplacian(pts, starts, factor, passes, workers=1):
    """bundler.py:141-149."""
    if passes < 1:
        return
    scratch = np.empty_like(pts)
    map_partitions(lambda lo, hi: lib().orc_laplacian(
        _p(pts), _p(starts), float(factor), int(passes), _p(scratch), lo, hi),
        starts.size - 1, workers)


def resample(pts, starts, delta, workers=1):
    """bundler.py:109-124."""
    n_edges = starts.size - 1
    counts = np.empty(n_edges, dtype=np.int64)
    map_partitions(lambda lo, hi: lib().orc_resample_count(
        _p(pts), _p(starts), float(delta), _p(counts), lo, hi), n_edges, workers)
    new_starts = np.zeros(n_edges + 1, dtype=np.int64)
    np.cumsum(counts, out=new_starts[1:])
    out = np.empty((int(new_starts[-1]), 2), dtype=np.float64)
    map_partitions(lambda lo, hi: lib().orc_resample_emit(
        _p(pts), _p(starts), float(delta), _p(new_starts), _p(out), lo, hi),
        n_edges, workers)
    return out, new_starts


def used_cells(rho, rel=0.01) -> int:
    r = np.ascontiguousarray(rho, dtype=np.float32)
    nb, nv, nu = r.shape
    return int(lib().orc_used_cells(_p(r), nb, nv, nu, float(rel)))


# ---------------------------------------------------------------------------
# full loop (bundler.py:311-380, packed form)


@dataclass
class OracleMetrics:
    iteration: int
    bandwidth: float
    moved_points: int
    mean_displacement: float
    used_cells: int
    seconds: float
    n_points: int = 0          # points entering splat/advect this iteration


@dataclass
class OracleRun:
    pts: np.ndarray            # final packed grid-space points (N, 2)
    starts: np.ndarray         # (E+1,) int64
    field: np.ndarray          # last smoothed (B, V, U) float32
    metrics: list = field(default_factory=list)
    transform: tuple = ()
    bundling_seconds: float = 0.0


def bundle_packed(positions, sources, targets, weights, bins, cfg, matrix=None,
                  workers=1, fixed_step=False,
                  on_stage: Callable[[int, str, object], None] | None = None,
                  max_iterations: int | None = None) -> OracleRun:
    """The reference loop on the C oracle. ``cfg`` is any object with the
    BundleConfig fields. ``on_stage(i, name, value)`` observes stage outputs
    (raw histogram, smoothed field, points) for golden capture."""
    bins = np.ascontiguousarray(bins, dtype=np.int64)
    n_edges = sources.shape[0]
    nbins = int(bins.max()) + 1 if n_edges else 1
    if matrix is None:
        m = np.eye(nbins, dtype=np.float32)
        if nbins > 1:
            m = (m + (1.0 - np.eye(nbins)) * (-cfg.alpha / (nbins - 1))).astype(np.float32)
        matrix = m
    matrix = np.asarray(matrix, dtype=np.float32)
    nbins = matrix.shape[0]
    pad = float(int(math.ceil(cfg.h_max)) + 1)
    ox, oy, cell, width, height = transform(positions, cfg.grid_size, pad)
    pts, starts, _, _ = sample(positions, sources, targets, (ox, oy), cell,
                               cfg.delta)
    if cfg.directed_offset_fraction > 0:
        disp = offset_disp(pts, starts, cfg.directed_offset_fraction
                           * max(width, height))
        lib().orc_offset(_p(pts), _p(starts), _p(disp), n_edges)
    layer_w = np.ascontiguousarray(
        weights.astype(np.float32)[:, None] * matrix.T[bins])
    shape = (height, width)
    rho = np.zeros((nbins,) + shape, np.float32)
    metrics = []
    iters = cfg.iterations if max_iterations is None else min(cfg.iterations, max_iterations)
    for i in range(iters):
        t0 = time.perf_counter()
        if i > 0:
            pts, starts = resample(pts, starts, cfg.delta, workers)
        n_i = pts.shape[0]
        raw = accumulate(pts, starts, layer_w, shape, workers)
        if on_stage:
            on_stage(i, "raw", raw)
        rho = smooth(raw, cfg.sigma, cfg.smoothing_passes, workers)
        if on_stage:
            on_stage(i, "field", rho)
        h_i = cfg.lambda_ ** i * cfg.h_max
        interior, moved, disp = advect(pts, starts, bins, rho, h_i,
                                       cfg.epsilon, fixed_step, workers)
        laplacian(pts, starts, cfg.laplacian_factor, cfg.laplacian_passes,
                  workers)
        if on_stage:
            on_stage(i, "pts", pts)
        used = used_cells(rho)
        metrics.append(OracleMetrics(i, h_i, moved,
                                     disp / interior if interior else 0.0,
                                     used, time.perf_counter() - t0, n_i))
    return OracleRun(pts, starts, rho, metrics, (ox, oy, cell, width, height),
                     sum(m.seconds for m in metrics))


def materialize(run: OracleRun, positions, sources, targets):
    """bundler.py:152-163 in packed form: world = pts*cell + origin, then
    endpoints pinned to the node positions."""
    ox, oy, cell = run.transform[:3]
    world = run.pts * cell + np.asarray((ox, oy))
    world[run.starts[:-1]] = positions[sources]
    world[run.starts[1:] - 1] = positions[targets]
    return world
