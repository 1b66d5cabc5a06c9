"""Drop-in for the raster operators of ``histobundle.raster``
(``/root/reference/pkg/src/histobundle/raster.py``), backed by the kernels:
histogram accumulation (hb_splat / hb_mix_layers), integral images
(hb_integral_image) and the box-filter Gaussian approximation (hb_smooth).
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .engine import box_widths, ptr, stream_ptr, weight_plan
from .model import DensityField, Graph, GridTransform, SampledEdge

__all__ = ["rasterize_segment", "accumulate_edges", "integral_image", "box_sum",
           "box_filter", "box_widths", "smooth_gaussian_approx"]


def _dev():
    N.lib()
    if not torch.cuda.is_available():
        raise N.NativeError("a CUDA device is required")
    return torch.device("cuda")


def rasterize_segment(p0, p1) -> np.ndarray:
    """Cell chain of one segment (raster.py:33-54), computed by splatting the
    segment into a scratch grid on the device and reading the hit cells back
    in DDA order."""
    p = np.array([p0, p1], dtype=np.float64)
    c = np.floor(p + 0.5).astype(np.int64)
    lo = c.min(axis=0) - 1
    local = p - lo
    nu, nv = int(c[:, 0].max() - lo[0] + 2), int(c[:, 1].max() - lo[1] + 2)
    dev = _dev()
    pts = torch.from_numpy(np.ascontiguousarray(local)).to(dev)
    starts = torch.tensor([0, 2], dtype=torch.int64, device=dev)
    grp = torch.zeros(1, dtype=torch.int32, device=dev)
    hist = torch.zeros((1, nv, nu), dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    N.call("hb_splat", ptr(pts), ptr(starts), 1, 2, ptr(grp), None, ptr(hist), 1, nv, nu,
           ptr(status), None, stream_ptr())
    v, u = np.nonzero(hist[0].cpu().numpy())
    cells = np.stack([u + lo[0], v + lo[1]], axis=1).astype(np.int64)
    d = c[1] - c[0]
    key = cells[:, 0] * np.sign(d[0]) if abs(d[0]) >= abs(d[1]) else cells[:, 1] * np.sign(d[1])
    return cells[np.argsort(key, kind="stable")]


def _pack_world(sampled: Sequence[SampledEdge], transform: GridTransform):
    counts = np.fromiter((len(se) for se in sampled), dtype=np.int64, count=len(sampled))
    starts = np.zeros(len(sampled) + 1, dtype=np.int64)
    np.cumsum(counts, out=starts[1:])
    pts = np.empty((int(starts[-1]), 2), dtype=np.float64)
    for i, se in enumerate(sampled):
        pts[starts[i]:starts[i + 1]] = se.points
    return transform.world_to_grid(pts), starts


def _accumulate_ordered(dpts, dst, E, n, grp, w32, mat, nb, nv, nu, workers, status):
    """The reference's float32 fold order (raster.py:85-94) on the device."""
    dev = dpts.device
    s = stream_ptr()
    hoff = torch.empty(n + 1, dtype=torch.int64, device=dev)
    hws = torch.empty(int(N.lib().hb_hits_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    N.call("hb_hits_count", ptr(dpts), ptr(dst), E, n, ptr(hoff), ptr(hws), hws.numel(), s)
    n_hits = int(hoff[n].item())
    parts = max(1, min(int(workers), E)) if E else 1
    ows = torch.empty(int(N.lib().hb_ordered_workspace_bytes(n_hits, nv, nu, parts)),
                      dtype=torch.uint8, device=dev)
    out = torch.empty((nb, nv, nu), dtype=torch.float32, device=dev)
    N.call("hb_accumulate_ordered", ptr(dpts), ptr(dst), E, ptr(hoff), n, n_hits, parts, 0, E,
           ptr(w32), ptr(grp) if nb > 1 else None, ptr(mat), nb, nv, nu, ptr(out), ptr(status),
           ptr(ows), ows.numel(), s)
    return out


def accumulate_edges(sampled: Sequence[SampledEdge], graph: Graph, matrix: np.ndarray,
                     transform: GridTransform, workers: int = 1) -> DensityField:
    """Raw multi-layer histogram H (raster.py:108-130) on the device.

    Exact layer weights: per-group int32 counts by DDA splat, then
    H[l] = sum_b M[l,b] C[b] in one rounding (guarded by hb_exact_check).
    Otherwise, or when the guard trips: the reference's own float32
    summation order over ``workers`` edge partitions (hb_accumulate_ordered),
    so H equals the reference bit for bit for the same ``workers``."""
    matrix = np.asarray(matrix, dtype=np.float32)
    nb = matrix.shape[0]
    if matrix.shape != (nb, nb):
        raise ValueError("interaction matrix must be square")
    if graph.n_edges and graph.bins.max() >= nb:
        raise ValueError("edge bin exceeds interaction matrix size")
    pts, starts = _pack_world(sampled, transform)
    edge_idx = np.fromiter((se.edge_index for se in sampled), dtype=np.int64,
                           count=len(sampled))
    nv, nu = transform.shape
    if pts.size:
        xmin, xmax = pts[:, 0].min(), pts[:, 0].max()
        ymin, ymax = pts[:, 1].min(), pts[:, 1].max()
        if xmin <= -0.5 or ymin <= -0.5 or xmax >= nu - 0.5 or ymax >= nv - 0.5:
            raise ValueError(
                f"sample out of bounds: points span ({xmin:.3f}, {ymin:.3f}) to "
                f"({xmax:.3f}, {ymax:.3f}) on a {nu}x{nv} grid")
    dev = _dev()
    E, n = len(sampled), pts.shape[0]
    weights = graph.weights[edge_idx]
    plan = weight_plan(weights, matrix, n)
    grp = torch.from_numpy(graph.bins[edge_idx].astype(np.int32)).to(dev)
    dpts = torch.from_numpy(np.ascontiguousarray(pts)).to(dev)
    dst = torch.from_numpy(starts).to(dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    identity = np.array_equal(matrix, np.eye(nb, dtype=np.float32))
    mat = None if identity else torch.from_numpy(matrix.copy()).to(dev)
    s = stream_ptr()
    if plan.kind != "ordered":
        hist = torch.zeros((nb, nv, nu), dtype=torch.int32, device=dev)
        w = None if plan.kind == "unit" else torch.from_numpy(plan.int_w).to(dev)
        N.call("hb_splat", ptr(dpts), ptr(dst), E, n, ptr(grp), ptr(w), ptr(hist), nb, nv, nu,
               ptr(status), None, s)
        absm = (None if plan.abs_matrix is None
                else torch.from_numpy(np.ascontiguousarray(plan.abs_matrix)).to(dev))
        N.call("hb_exact_check", ptr(hist), ptr(absm), nb, nv, nu, float(plan.limit),
               ptr(status), s)
        if not int(status.item()) & 8:
            out = torch.empty((nb, nv, nu), dtype=torch.float32, device=dev)
            N.call("hb_mix_layers", ptr(hist), None, ptr(mat), nb, nv, nu, ptr(out), s)
            return DensityField(transform, out.cpu().numpy())
    w32 = weights.astype(np.float32)
    wd = None if np.all(w32 == 1.0) else torch.from_numpy(w32).to(dev)
    out = _accumulate_ordered(dpts, dst, E, n, grp, wd, mat, nb, nv, nu, workers, status)
    return DensityField(transform, out.cpu().numpy())


def integral_image(layer: np.ndarray) -> np.ndarray:
    """(V+1, U+1) float64 table (raster.py:133-139)."""
    lay = np.ascontiguousarray(layer, dtype=np.float32)
    nv, nu = lay.shape
    dev = _dev()
    src = torch.from_numpy(lay).to(dev)
    tab = torch.empty((nv, nu), dtype=torch.float64, device=dev)
    N.call("hb_integral_image", ptr(src), 1, nv, nu, ptr(tab), stream_ptr())
    out = np.zeros((nv + 1, nu + 1), dtype=np.float64)
    out[1:, 1:] = tab.cpu().numpy()
    return out


def box_sum(table: np.ndarray, v0: int, v1: int, u0: int, u1: int) -> float:
    """raster.py:142-144."""
    return float(table[v1, u1] - table[v0, u1] - table[v1, u0] + table[v0, u0])


def _smooth(values: np.ndarray, radii: list[int]) -> np.ndarray:
    vals = np.ascontiguousarray(values, dtype=np.float32)
    nb, nv, nu = vals.shape
    dev = _dev()
    src = torch.from_numpy(vals).to(dev)
    out = torch.empty_like(src)
    ws = torch.empty(int(N.lib().hb_smooth_workspace_bytes(nb, nv, nu)), dtype=torch.uint8,
                     device=dev)
    r = torch.tensor(radii, dtype=torch.int32)
    N.call("hb_smooth", None, ptr(src), None, nb, nv, nu, r.data_ptr(), len(radii), ptr(out),
           ptr(ws), ws.numel(), None, stream_ptr())
    return out.cpu().numpy()


def box_filter(layer: np.ndarray, radius: int) -> np.ndarray:
    """Zero-padded mean filter over (2r+1)^2 (raster.py:147-169)."""
    if radius < 0:
        raise ValueError("radius must be >= 0")
    if radius == 0:
        return layer.copy()
    return _smooth(np.asarray(layer)[None], [int(radius)])[0].astype(layer.dtype)


def smooth_gaussian_approx(field: DensityField, sigma: float, passes: int = 3,
                           workers: int = 1) -> DensityField:
    """n-pass box-filter Gaussian approximation of every layer (raster.py:203-219)."""
    del workers
    widths = box_widths(sigma, passes)
    return DensityField(field.transform, _smooth(field.values, [(w - 1) // 2 for w in widths]))
