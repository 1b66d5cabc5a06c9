"""SVG rendering (render.py:135-250) against fixtures made by the reference
(tests/golden/render.npz, tests/golden/make_render_golden.py): the SVG text
must be byte-identical for every option set, the per-segment widths bit for
bit."""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN

G = np.load(os.path.join(GOLDEN, "render.npz"))

CASES = {  # must match make_render_golden.CASES
    "default": ("nominal", {}, 1),
    "uniform": ("nominal", {"width_min": 1.5, "width_max": 1.5}, 1),
    "modal": ("modal-hue", {"alpha": 0.3}, 3),
    "sequential": ("sequential", {"log_widths": False, "background": None}, 3),
    "flow": ("flow-blue-red", {"width_min": 0.5, "width_max": 3.0}, 1),
    "logw": ("nominal", {"log_widths": True}, 1),
}


def test_color_and_options_host_logic():
    from paper_1504_02687_b200 import render as PR

    assert PR.RenderOptions().resolve_alpha(10) == 0.5
    assert PR.RenderOptions().resolve_alpha(5000) == 0.15
    assert PR.color_for_bin(PR.ColorScheme(), 1, 4)[:3] == PR._hex_to_unit("#f28e2b")
    with pytest.raises(ValueError, match="out of range"):
        PR.color_for_bin(PR.ColorScheme(), 4, 4)
    with pytest.raises(ValueError, match="unknown color scheme"):
        PR.color_for_bin(PR.ColorScheme(kind="plasma"), 0, 4)


def _result(bins_n):
    from paper_1504_02687_b200 import bundler as B
    from paper_1504_02687_b200.model import Graph
    from paper_1504_02687_b200.workloads import workload

    w = workload(1, scale=0.05)
    g = w.graph
    bins = (np.arange(g.n_edges) % bins_n).astype(np.int64)
    g2 = Graph.from_arrays(g.positions, g.sources, g.targets, g.weights, bins)
    cfg = w.config
    cfg.iterations = 4
    return B.bundle(g2, cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_render_svg_matches_reference(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1504_02687_b200 import render as PR

    kind, opts, bins_n = CASES[name]
    svg = PR.render_svg(_result(bins_n), PR.ColorScheme(kind=kind), PR.RenderOptions(**opts))
    if name == "default":
        ref = str(G["default_svg"])
        if svg != ref:  # point at the first difference
            k = next(i for i, (a, b) in enumerate(zip(svg, ref)) if a != b)
            pytest.fail(f"first difference at {k}: {svg[k - 80:k + 40]!r} vs {ref[k - 80:k + 40]!r}")
    assert len(svg) == int(G[f"{name}_len"])
    assert hashlib.sha256(svg.encode()).hexdigest() == str(G[f"{name}_sha"])


@pytest.mark.gpu
def test_segment_widths_match_reference():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1504_02687_b200 import render as PR

    res = _result(1)
    field = res.density
    edges = list(res.sampled_edges)
    starts = np.concatenate([[0], np.cumsum([len(e) for e in edges])])
    grid = field.transform.world_to_grid(np.concatenate([e.points for e in edges]))
    w = PR._DeviceWidths(field).widths(grid, starts, None, 0.6, 4.0, False)
    assert np.array_equal(PR._layer_peaks(field), G["peaks"])
    assert np.array_equal(w, G["widths"])


@pytest.mark.gpu
def test_width_for_segment_matches_reference():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1504_02687_b200 import render as PR

    res = _result(1)
    got = [[PR.width_for_segment(res.density, 0, a, b, 0.6, 4.0, lg) for a, b in G["wfs_probes"]]
           for lg in (False, True)]
    assert np.array_equal(np.array(got), G["wfs"])


PNG_CASES = {  # must match make_render_golden.PNG_CASES / PNG_SIZES
    "default": ("nominal", {}, 1, None),
    "modal": ("modal-hue", {"alpha": 0.3}, 3, None),
    "flow_wide": ("flow-blue-red", {"width_min": 0.5, "width_max": 6.0, "background": None}, 1,
                  (333, 250)),
    "sequential_big": ("sequential", {"width_min": 1.0, "width_max": 9.0}, 3, (600, 420)),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(PNG_CASES))
def test_render_png_matches_reference(name):
    """render_png (render.py:263-335): device stroke widths, per-edge tiles
    drawn with PIL and composited in edge order -- the same RGBA bytes as the
    reference's image."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import PIL

    from paper_1504_02687_b200 import render as PR

    if str(G["pillow"]) != PIL.__version__:
        pytest.skip(f"fixture made with pillow {G['pillow']}, found {PIL.__version__}")
    kind, opts, bins_n, size = PNG_CASES[name]
    img = PR.render_png(_result(bins_n), PR.ColorScheme(kind=kind), PR.RenderOptions(**opts),
                        size=size)
    assert img.mode == str(G[f"png_{name}_mode"])
    assert list(img.size) == list(G[f"png_{name}_size"])
    assert hashlib.sha256(img.tobytes()).hexdigest() == str(G[f"png_{name}_sha"])


def test_render_png_rejects_empty_size():
    from paper_1504_02687_b200 import render as PR

    class R:  # the size check comes before any drawing
        class graph:
            n_edges = 1

        class density:
            class transform:
                width, height = 10, 10

                @staticmethod
                def world_bounds():
                    return (0.0, 0.0, 1.0, 1.0)
        sampled_edges = []

    with pytest.raises(ValueError, match="image dimensions must be positive"):
        PR.render_png(R, size=(0, 5))
