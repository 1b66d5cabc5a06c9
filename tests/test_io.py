"""Polyline export / import (reference io.py:136-171) -- CPU tests.

The golden text was written by the reference's own export_polylines
(tests/golden/make_io_golden.py); randomized cases compare byte-for-byte
with the reference's formatting expression, f"{x:.9g}".
"""

from __future__ import annotations

import io
import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1504_02687_b200 import io as hio
from paper_1504_02687_b200.bundler import PackedPolylines
from paper_1504_02687_b200.model import SampledEdge


def _result(world, starts, weights, bins, packed=True):
    graph = SimpleNamespace(bins=np.asarray(bins), weights=np.asarray(weights))
    if packed:
        se = PackedPolylines(world, starts)
    else:
        se = [SampledEdge(e, world[starts[e]:starts[e + 1]]) for e in range(len(starts) - 1)]
    return SimpleNamespace(graph=graph, sampled_edges=se)


def _reference_text(world, starts, weights, bins) -> str:
    """io.py:136-145 verbatim in expression (one line per edge)."""
    out = ["# histobundle polylines v1\n", f"# edges {len(starts) - 1}\n"]
    for e in range(len(starts) - 1):
        pts = world[starts[e]:starts[e + 1]]
        coords = " ".join(f"{c:.9g}" for p in pts for c in p)
        out.append(f"{e} {bins[e]} {weights[e]:.9g} {len(pts)} {coords}\n")
    return "".join(out)


def _golden():
    z = np.load(os.path.join(GOLDEN, "io_input.npz"))
    with open(os.path.join(GOLDEN, "io_export.txt")) as f:
        return z["world"], z["starts"], z["weights"], z["bins"], f.read()


@pytest.mark.parametrize("packed", [True, False])
def test_export_matches_reference_golden(packed):
    world, starts, weights, bins, text = _golden()
    buf = io.StringIO()
    hio.export_polylines(_result(world, starts, weights, bins, packed), buf)
    assert buf.getvalue() == text


def test_export_to_file_descriptor_matches_golden(tmp_path):
    world, starts, weights, bins, text = _golden()
    path = tmp_path / "out.txt"
    with open(path, "w") as f:
        f.write("")  # the native writer appends at the file offset
        hio.export_polylines(_result(world, starts, weights, bins), f)
    assert path.read_text() == text


def test_export_random_values_match_python_formatting(tmp_path):
    rng = np.random.default_rng(5)
    n_edges = 3000
    lens = rng.integers(2, 200, size=n_edges)
    starts = np.zeros(n_edges + 1, dtype=np.int64)
    np.cumsum(lens, out=starts[1:])
    n = int(starts[-1])
    mags = 10.0 ** rng.integers(-12, 14, size=(n, 2))
    world = rng.uniform(-1, 1, size=(n, 2)) * mags
    world[rng.uniform(size=(n, 2)) < 0.05] = 0.5  # exact values
    world[rng.uniform(size=(n, 2)) < 0.01] *= 1e-300  # subnormal-ish tails
    weights = rng.uniform(0, 10, size=n_edges)
    bins = rng.integers(0, 100, size=n_edges)
    want = _reference_text(world, starts, weights, bins)
    buf = io.StringIO()
    hio.export_polylines(_result(world, starts, weights, bins), buf)
    assert buf.getvalue() == want
    path = tmp_path / "big.txt"
    with open(path, "w") as f:
        hio.export_polylines(_result(world, starts, weights, bins), f)
    assert path.read_text() == want
    # multi-chunk native parse of the same ~9 MB text
    with open(path) as f:
        recs = hio.read_polylines(f)
    assert len(recs) == n_edges
    back = np.concatenate([r.points for r in recs])
    assert np.array_equal(back, np.vectorize(lambda v: float(f"{v:.9g}"))(world))
    assert [r.bin for r in recs] == bins.tolist()


def test_read_error_line_numbers_are_global_in_large_inputs():
    line = "7 0 1 3 " + " ".join(["0.123456789"] * 6)
    lines = [line] * 200_000
    lines[150_001] = "7 0 1 3 0.5 0.5"  # 2 of 6 coordinates
    with pytest.raises(hio.GraphFormatError,
                       match="polyline line 150002: expected 6 coordinates, got 2"):
        hio.read_polylines(lines)


def test_read_round_trip():
    world, starts, weights, bins, text = _golden()
    recs = hio.read_polylines(io.StringIO(text))
    assert len(recs) == len(starts) - 1
    for e, r in enumerate(recs):
        assert (r.edge_index, r.bin) == (e, int(bins[e]))
        assert r.weight == float(f"{weights[e]:.9g}")
        want = np.array([[float(f"{x:.9g}"), float(f"{y:.9g}")]
                         for x, y in world[starts[e]:starts[e + 1]]])
        assert np.array_equal(r.points, want)
    # also from a list of lines
    recs2 = hio.read_polylines(text.splitlines())
    assert all(np.array_equal(a.points, b.points) for a, b in zip(recs, recs2))


def test_read_errors_use_reference_messages():
    with pytest.raises(hio.GraphFormatError, match="polyline line 3: malformed record"):
        hio.read_polylines(["# c", "1 0 1 1 0.5 0.5", "2 0"])
    with pytest.raises(hio.GraphFormatError,
                       match="polyline line 2: expected 4 coordinates, got 3"):
        hio.read_polylines(["", "1 0 1 2 0 0 1"])
    with pytest.raises(hio.GraphFormatError, match="polyline line 1: malformed record"):
        hio.read_polylines(["1 0 1 1 0.5 abc"])


def test_read_python_only_spellings_fall_back():
    # '+1' and '1_0' are valid for Python's int()/float() but not for the
    # native fast path: the reference loop decides
    recs = hio.read_polylines(["+1 1_0 2.5 1 +0.25 1_0.5"])
    assert (recs[0].edge_index, recs[0].bin, recs[0].weight) == (1, 10, 2.5)
    assert np.array_equal(recs[0].points, [[0.25, 10.5]])


def test_io_header_matches_library_exports():
    import re
    import subprocess

    from paper_1504_02687_b200 import _native

    hio._io_lib()  # builds if missing
    with open(os.path.join(os.path.dirname(GOLDEN), "..", "include", "histobundle_io.h")) as f:
        declared = set(re.findall(r"\b(hb_io_\w+)\s*\(", f.read()))
    out = subprocess.run(["nm", "-D", "--defined-only", _native.HOST_IO_LIB],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (hb_io_\w+)", out))
    assert declared == exported == {"hb_io_format", "hb_io_export_fd", "hb_io_parse"}
