"""SVG and PNG rendering fixtures made by running the REFERENCE (render.py) here.

    python tests/golden/make_render_golden.py

PNG cases use the reference's render_png (pillow 12.2, recorded); the raw
RGBA bytes are hashed.  The bundling result comes from the
reference's own bundle() on a 100-edge config-1 graph (seed 0) -- the device
path reproduces it bit for bit, so both renderers see the same input.
Writes tests/golden/render.npz: per option set, the sha256 and length of the
SVG text, the full text of the smallest case, and per-segment widths.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from histobundle import bundler as RB  # noqa: E402
from histobundle import model as RM  # noqa: E402
from histobundle import render as RR  # noqa: E402

from paper_1504_02687_b200.workloads import workload  # noqa: E402

# (name, scheme kind, RenderOptions kwargs, bins per edge)
CASES = [
    ("default", "nominal", {}, 1),
    ("uniform", "nominal", {"width_min": 1.5, "width_max": 1.5}, 1),
    ("modal", "modal-hue", {"alpha": 0.3}, 3),
    ("sequential", "sequential", {"log_widths": False, "background": None}, 3),
    ("flow", "flow-blue-red", {"width_min": 0.5, "width_max": 3.0}, 1),
    ("logw", "nominal", {"log_widths": True}, 1),
]


# render_png cases: (name, scheme kind, RenderOptions kwargs, bins per edge)
PNG_CASES = [
    ("default", "nominal", {}, 1),
    ("modal", "modal-hue", {"alpha": 0.3}, 3),
    ("flow_wide", "flow-blue-red", {"width_min": 0.5, "width_max": 6.0, "background": None}, 1),
    ("sequential_big", "sequential", {"width_min": 1.0, "width_max": 9.0}, 3),
]
PNG_SIZES = {"sequential_big": (600, 420), "flow_wide": (333, 250)}


def graph_for(bins_n):
    w = workload(1, scale=0.05)
    g = w.graph
    bins = (np.arange(g.n_edges) % bins_n).astype(np.int64)
    return RM.Graph.from_arrays(g.positions, g.sources, g.targets, g.weights, bins), w


def main():
    out = {"numpy": np.array(np.__version__)}
    results = {}
    for name, kind, opts, bins_n in CASES:
        if bins_n not in results:
            rg, w = graph_for(bins_n)
            cfg = RM.BundleConfig(**{f: getattr(w.config, f)
                                     for f in w.config.__dataclass_fields__})
            cfg.iterations = 4
            results[bins_n] = RB.bundle(rg, cfg)
        res = results[bins_n]
        svg = RR.render_svg(res, RR.ColorScheme(kind=kind), RR.RenderOptions(**opts))
        out[f"{name}_sha"] = np.array(hashlib.sha256(svg.encode()).hexdigest())
        out[f"{name}_len"] = np.array(len(svg))
        if name == "default":
            out["default_svg"] = np.array(svg)
    import PIL
    out["pillow"] = np.array(PIL.__version__)
    for name, kind, opts, bins_n in PNG_CASES:
        img = RR.render_png(results[bins_n], RR.ColorScheme(kind=kind), RR.RenderOptions(**opts),
                            size=PNG_SIZES.get(name))
        raw = img.tobytes()
        out[f"png_{name}_sha"] = np.array(hashlib.sha256(raw).hexdigest())
        out[f"png_{name}_size"] = np.array(img.size)
        out[f"png_{name}_mode"] = np.array(img.mode)
    res = results[1]
    peaks = RR._layer_peaks(res.density)
    ws = []
    for se in res.sampled_edges:
        grid = res.density.transform.world_to_grid(se.points)
        ws.append(RR._segment_widths(res.density, 0, grid, 0.6, 4.0, False, float(peaks[0])))
    out["widths"] = np.concatenate(ws)
    # single-segment helper: inside, near the edge and outside the grid
    x0, y0, wd, ht = res.density.transform.world_bounds()
    probes = [((0.3, 0.4), (0.35, 0.42)), ((x0 + 0.01 * wd, y0), (x0 + wd, y0 + ht)),
              ((x0 - 0.1, y0 - 0.2), (0.5, 0.5))]
    out["wfs"] = np.array([[RR.width_for_segment(res.density, 0, a, b, 0.6, 4.0, lg)
                            for a, b in probes] for lg in (False, True)])
    out["wfs_probes"] = np.array(probes)
    out["peaks"] = peaks
    np.savez_compressed(os.path.join(HERE, "render.npz"), **out)
    print("wrote render.npz", {k: (v.shape, v.dtype) for k, v in out.items()})


if __name__ == "__main__":
    main()
