"""SVG and PNG rendering of a bundling result: the API of the reference's ``render.py``.

Mirrors ``/root/reference/pkg/src/histobundle/render.py`` (``ColorScheme``,
``RenderOptions``, ``color_for_bin``, ``width_for_segment``, ``render_svg``,
``render_png``; same arguments and the same SVG text / image bytes, checked byte for byte against
fixtures made by the reference, tests/golden/make_render_golden.py).  The
per-segment stroke widths -- a clamped bilinear density sample at both ends
of every segment -- are computed on the device (``hb_segment_widths``);
colours, alpha and the text are host work, as in the reference.

``render_png`` computes the same device widths and draws every edge with
PIL's rasteriser (the reference's), compositing the per-edge tiles in edge
order: byte-identical images (tests/golden/make_render_golden.py).
"""

from __future__ import annotations

import colorsys
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .engine import ptr, stream_ptr
from .model import DensityField

__all__ = ["ColorScheme", "RenderOptions", "color_for_bin", "width_for_segment", "render_svg",
           "render_png"]

# qualitative palette (render.py:32-36): distinct up to 16 bins
_NOMINAL = ("#4e79a7", "#f28e2b", "#e15759", "#76b7b2", "#59a14f", "#edc948", "#b07aa1",
            "#ff9da7", "#9c755f", "#bab0ac", "#1f77b4", "#8c564b", "#2ca02c", "#d62728",
            "#9467bd", "#17becf")
_FLOW_SOURCE = (0.10, 0.25, 0.90)  # render.py:38-39
_FLOW_TARGET = (0.90, 0.15, 0.10)
_LOG_GAIN = 9.0


@dataclass(frozen=True)
class ColorScheme:
    """Bin -> colour mapping: "sequential", "modal-hue", "nominal" or
    "flow-blue-red" (render.py:43-58)."""

    kind: str = "nominal"
    base_hue: float = 210.0
    lightness_range: tuple[float, float] = (0.85, 0.30)

    KINDS = ("sequential", "modal-hue", "nominal", "flow-blue-red")


@dataclass
class RenderOptions:
    """Stroke styling in grid cells (render.py:95-112)."""

    width_min: float = 0.6
    width_max: float = 4.0
    alpha: float | None = None
    log_widths: bool = False
    background: str | None = "#ffffff"

    def resolve_alpha(self, n_edges: int) -> float:
        if self.alpha is None:
            return 0.15 if n_edges > 1000 else 0.5
        return self.alpha


def _hex_to_unit(color: str) -> tuple[float, float, float]:
    h = color.lstrip("#")
    return tuple(int(h[k:k + 2], 16) / 255.0 for k in range(0, 6, 2))


def _flow_color(t: float) -> tuple[float, float, float]:
    return tuple(s + t * (e - s) for s, e in zip(_FLOW_SOURCE, _FLOW_TARGET))


def color_for_bin(scheme: ColorScheme, bin_: int, bin_count: int
                  ) -> tuple[float, float, float, float]:
    """RGBA in [0, 1] for a bin (render.py:66-87)."""
    if not 0 <= bin_ < bin_count:
        raise ValueError(f"bin {bin_} out of range for {bin_count} bins")
    kind = scheme.kind
    if kind == "modal-hue":
        rgb = colorsys.hsv_to_rgb((bin_ / bin_count) % 1.0, 0.85, 0.85)
    elif kind == "sequential":
        lo, hi = scheme.lightness_range
        t = bin_ / max(bin_count - 1, 1)
        rgb = colorsys.hls_to_rgb(scheme.base_hue / 360.0, lo + t * (hi - lo), 0.65)
    elif kind == "nominal":
        rgb = _hex_to_unit(_NOMINAL[bin_ % len(_NOMINAL)])
    elif kind == "flow-blue-red":
        rgb = _flow_color(0.5)
    else:
        raise ValueError(f"unknown color scheme kind {kind!r}")
    return (*rgb, 1.0)


def _layer_peaks(field: DensityField) -> np.ndarray:
    """Per-layer maximum density inside the padding ring (render.py:115-126)."""
    vals = field.values
    pad = int(math.ceil(field.transform.padding))
    inner = vals[:, pad:vals.shape[1] - pad, pad:vals.shape[2] - pad]
    if inner.shape[1] == 0 or inner.shape[2] == 0:
        inner = vals
    return np.maximum(inner.reshape(field.bin_count, -1).max(axis=1), 0.0)


def _scale_log(ratio: np.ndarray) -> np.ndarray:
    return np.log1p(_LOG_GAIN * ratio) / math.log1p(_LOG_GAIN)


class _DeviceWidths:
    """Segment widths of packed grid-space polylines, computed on the device."""

    def __init__(self, field: DensityField):
        if not torch.cuda.is_available():
            raise N.NativeError("rendering widths need a CUDA device (no CPU fallback)")
        self.field = field
        self.rho = torch.from_numpy(np.ascontiguousarray(field.values, dtype=np.float32)).cuda()
        self.peaks_np = _layer_peaks(field).astype(np.float32)
        self.peaks = torch.from_numpy(self.peaks_np).cuda()

    def ratios(self, grid_pts: np.ndarray, starts: np.ndarray, layers: np.ndarray | None):
        """Clipped density ratio per segment (0 where the layer peak is 0)."""
        n_edges = len(starts) - 1
        n_seg = int(starts[-1]) - n_edges
        out = torch.empty(max(n_seg, 1), dtype=torch.float64, device="cuda")
        p = torch.from_numpy(np.ascontiguousarray(grid_pts, dtype=np.float64)).cuda()
        st = torch.from_numpy(np.ascontiguousarray(starts, dtype=np.int64)).cuda()
        ly = None if layers is None else torch.from_numpy(
            np.ascontiguousarray(layers, dtype=np.int32)).cuda()
        B, V, U = self.field.values.shape
        N.call("hb_segment_widths", ptr(p), ptr(st), n_edges, ptr(ly), ptr(self.rho), B, V, U,
               ptr(self.peaks), 0.0, 1.0, 1, ptr(out), stream_ptr())
        return out[:n_seg].cpu().numpy()

    def widths(self, grid_pts, starts, layers, w_min, w_max, log_scale) -> np.ndarray:
        if w_min > w_max:
            raise ValueError("w_min must be <= w_max")
        r = self.ratios(grid_pts, starts, layers)
        if log_scale:
            r = _scale_log(r)
        w = w_min + (w_max - w_min) * r
        # a layer without density draws every segment at w_min (render.py:162-163)
        n_edges = len(starts) - 1
        lay = np.zeros(n_edges, dtype=np.int64) if layers is None else np.asarray(layers)
        flat = np.repeat(self.peaks_np[lay] <= 0, np.diff(starts) - 1)
        w[flat] = w_min
        return w


def width_for_segment(field: DensityField, layer: int, a, b, w_min: float, w_max: float,
                      log_scale: bool = False, layer_peak: float | None = None) -> float:
    """Stroke width of the world-space segment a-b (render.py:135-155).  Its
    densities are bilinear_value samples (hb_probe), which -- unlike the
    vectorised widths -- do not clip the point into the grid first."""
    from .bundler import density_at  # (the single-point probe)

    if w_min > w_max:
        raise ValueError("w_min must be <= w_max")
    peak = _layer_peaks(field)[layer] if layer_peak is None else layer_peak
    if peak <= 0:
        return w_min
    ga = field.transform.world_to_grid(np.asarray(a, dtype=np.float64))
    gb = field.transform.world_to_grid(np.asarray(b, dtype=np.float64))
    d = 0.5 * (max(density_at(field, layer, ga), 0.0) + max(density_at(field, layer, gb), 0.0))
    r = min(max(d / peak, 0.0), 1.0)
    if log_scale:
        r = math.log1p(_LOG_GAIN * r) / math.log1p(_LOG_GAIN)
    return w_min + (w_max - w_min) * r


def _g(x: float) -> str:
    return f"{x:.6g}"


def _hex(rgb) -> str:
    return "#" + "".join(f"{min(max(int(round(c * 255)), 0), 255):02x}" for c in rgb[:3])


def _arc_fraction(points: np.ndarray) -> np.ndarray:
    seg = np.linalg.norm(np.diff(points, axis=0), axis=1)
    total = seg.sum()
    pos = np.zeros(points.shape[0])
    if total <= 0:
        return pos
    np.cumsum(seg, out=pos[1:])
    return pos / total


def render_svg(result, scheme: ColorScheme | None = None,
               options: RenderOptions | None = None) -> str:
    """SVG document, one group per edge, per-segment widths (render.py:191-250)."""
    scheme = scheme or ColorScheme()
    opts = options or RenderOptions()
    graph, field = result.graph, result.density
    tr = field.transform
    x0, y0, w, h = tr.world_bounds()
    alpha = opts.resolve_alpha(graph.n_edges)
    cell = tr.cell_size
    flow = scheme.kind == "flow-blue-red"
    per_segment = flow or opts.width_min != opts.width_max
    edges = list(result.sampled_edges)
    seg_w = None
    if per_segment and edges:
        # every polyline's widths in one device call
        counts = np.array([len(se) for se in edges], dtype=np.int64)
        starts = np.concatenate([[0], np.cumsum(counts)])
        grid = tr.world_to_grid(np.concatenate([se.points for se in edges]))
        layers = np.array([int(graph.bins[se.edge_index]) for se in edges], dtype=np.int32)
        seg_w = _DeviceWidths(field).widths(grid, starts, layers, opts.width_min,
                                            opts.width_max, opts.log_widths)
        seg_off = starts[:-1] - np.arange(len(edges))
    lines = ['<?xml version="1.0" encoding="UTF-8"?>',
             f'<svg xmlns="http://www.w3.org/2000/svg" viewBox="0 0 {_g(w)} {_g(h)}">']
    if opts.background:
        lines.append(f'<rect x="0" y="0" width="{_g(w)}" height="{_g(h)}" '
                     f'fill="{opts.background}"/>')
    lines.append('<g fill="none" stroke-linecap="round" stroke-linejoin="round">')
    for k, se in enumerate(edges):
        b = int(graph.bins[se.edge_index])
        sx = se.points[:, 0] - x0
        sy = (y0 + h) - se.points[:, 1]
        head = f' stroke-opacity="{_g(alpha)}"'
        if not flow:
            head += f' stroke="{_hex(color_for_bin(scheme, b, field.bin_count)[:3])}"'
        lines.append(f'<g class="edge"{head}>')
        if not per_segment:
            d = "M " + " L ".join(f"{_g(px)} {_g(py)}" for px, py in zip(sx, sy))
            lines.append(f'<path d="{d}" stroke-width="{_g(opts.width_min * cell)}"/>')
        else:
            ws = seg_w[seg_off[k]:seg_off[k] + len(se) - 1]
            arc = _arc_fraction(se.points) if flow else None
            for j in range(len(se) - 1):
                extra = ""
                if flow:
                    extra = f' stroke="{_hex(_flow_color(0.5 * (arc[j] + arc[j + 1])))}"'
                lines.append(f'<path d="M {_g(sx[j])} {_g(sy[j])} L {_g(sx[j + 1])} '
                             f'{_g(sy[j + 1])}" stroke-width="{_g(ws[j] * cell)}"{extra}/>')
        lines.append("</g>")
    lines += ["</g>", "</svg>"]
    return "\n".join(lines) + "\n"


def render_png(result, scheme: ColorScheme | None = None, options: RenderOptions | None = None,
               size: tuple[int, int] | None = None):
    """Raster image with source-over alpha accumulation (render.py:263-335).

    Every polyline's segment widths come from one device call (as in
    :func:`render_svg`); each edge is then drawn on its own transparent tile
    with PIL's line and disc rasteriser -- the reference's, so the pixels are
    the same -- and composited onto the canvas in edge order, so overlapping
    edges darken each other while one edge's own overlaps do not accumulate.
    Returns a PIL RGBA image."""
    from PIL import Image, ImageDraw

    scheme = scheme or ColorScheme()
    opts = options or RenderOptions()
    graph, field = result.graph, result.density
    tr = field.transform
    x0, y0, w, h = tr.world_bounds()
    if size is None:
        size = (tr.width, tr.height)
    width_px, height_px = int(size[0]), int(size[1])
    if width_px <= 0 or height_px <= 0:
        raise ValueError("image dimensions must be positive")
    alpha = opts.resolve_alpha(graph.n_edges)
    px_per_cell = width_px / tr.width
    flow = scheme.kind == "flow-blue-red"
    bg = (0, 0, 0, 0)
    if opts.background:
        r, g, b = _hex_to_unit(opts.background)
        bg = (int(r * 255), int(g * 255), int(b * 255), 255)
    canvas = Image.new("RGBA", (width_px, height_px), bg)
    edges = list(result.sampled_edges)
    if not edges:
        return canvas
    counts = np.array([len(se) for se in edges], dtype=np.int64)
    starts = np.concatenate([[0], np.cumsum(counts)])
    grid = tr.world_to_grid(np.concatenate([se.points for se in edges]))
    layers = np.array([int(graph.bins[se.edge_index]) for se in edges], dtype=np.int32)
    seg_w = _DeviceWidths(field).widths(grid, starts, layers, opts.width_min, opts.width_max,
                                        opts.log_widths)
    seg_off = starts[:-1] - np.arange(len(edges))
    a8 = int(round(alpha * 255))
    for k, se in enumerate(edges):
        b = int(layers[k])
        px = (se.points[:, 0] - x0) / w * width_px
        py = (1.0 - (se.points[:, 1] - y0) / h) * height_px
        widths_px = np.maximum(seg_w[seg_off[k]:seg_off[k] + len(se) - 1] * px_per_cell, 1.0)
        margin = int(math.ceil(widths_px.max() / 2)) + 2
        tx0 = max(int(math.floor(px.min())) - margin, 0)
        ty0 = max(int(math.floor(py.min())) - margin, 0)
        tx1 = min(int(math.ceil(px.max())) + margin, width_px)
        ty1 = min(int(math.ceil(py.max())) + margin, height_px)
        if tx1 <= tx0 or ty1 <= ty0:
            continue
        tile = Image.new("RGBA", (tx1 - tx0, ty1 - ty0), (0, 0, 0, 0))
        draw = ImageDraw.Draw(tile)
        if not flow:
            rgba = color_for_bin(scheme, b, field.bin_count)
            fill = (int(rgba[0] * 255), int(rgba[1] * 255), int(rgba[2] * 255), a8)
        arc = _arc_fraction(se.points) if flow else None
        for j in range(len(se) - 1):
            if flow:
                r, g, bb = _flow_color(0.5 * (arc[j] + arc[j + 1]))
                fill = (int(r * 255), int(g * 255), int(bb * 255), a8)
            lw = int(round(widths_px[j]))
            draw.line([(px[j] - tx0, py[j] - ty0), (px[j + 1] - tx0, py[j + 1] - ty0)],
                      fill=fill, width=max(lw, 1))
            if lw > 2:  # round joins and caps
                rr = lw / 2.0
                for q in (j, j + 1):
                    draw.ellipse([px[q] - tx0 - rr, py[q] - ty0 - rr,
                                  px[q] - tx0 + rr, py[q] - ty0 + rr], fill=fill)
        canvas.alpha_composite(tile, (tx0, ty0))
    return canvas
