"""Host-side logic, no GPU: boundary types, transform, box widths, sharding,
and the C-ABI library's exported symbol table."""

from __future__ import annotations

import json
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from paper_1504_02687_b200 import model as M
from paper_1504_02687_b200.workloads import workload


def test_box_widths_known_values():
    from paper_1504_02687_b200.engine import box_widths
    # sigma -> widths of the reference's rule
    assert box_widths(16, 3) == [31, 31, 33]
    assert box_widths(24, 3) == [47, 47, 49]
    assert box_widths(12.8, 3) == [25, 25, 27]
    assert box_widths(25.6, 3) == [51, 51, 51]
    assert box_widths(51.2, 3) == [101, 103, 103]
    with pytest.raises(ValueError):
        box_widths(0, 3)


@pytest.mark.parametrize("k", [1, 2])
def test_transform_matches_golden(k):
    g = json.load(open(os.path.join(GOLDEN, f"cfg{k}.json")))
    w = workload(k)
    tr = M.make_transform(w.graph.positions, w.config.grid_size, w.config.padding_cells)
    assert [tr.origin[0], tr.origin[1], tr.cell_size, tr.width, tr.height] == g["transform"]
    assert w.graph.n_edges == g["n_edges"]


def test_make_transform_spec_examples():
    tr = M.make_transform(np.array([[0.0, 0.0], [2.0, 1.0]]), 801, 0)
    assert (tr.width, tr.height) == (801, 401)
    tr = M.make_transform(np.array([[1.0, 1.0]]), 100, 2.5)
    assert (tr.width, tr.height, tr.cell_size) == (6, 6, 1.0)
    with pytest.raises(ValueError):
        M.make_transform(np.zeros((0, 2)), 100, 0)


def test_config_validation_messages():
    with pytest.raises(ValueError, match="grid_size"):
        M.BundleConfig(grid_size=4)
    with pytest.raises(ValueError, match="lambda_"):
        M.BundleConfig(lambda_=0.0)
    cfg = M.BundleConfig(grid_size=400)
    assert cfg.sigma == 10.0 and cfg.h_max == 20.0 and cfg.padding_cells == 21


def test_graph_validation():
    pos = np.zeros((3, 2))
    pos[1] = 1
    with pytest.raises(ValueError, match="self-loop at edge 1"):
        M.Graph(pos, [0, 2], [1, 2])
    with pytest.raises(ValueError, match="out of range"):
        M.Graph(pos, [0], [5])
    g = M.Graph(pos, [0], [1], bins=[3])
    assert g.bin_count == 4


def test_interaction_matrix():
    m = M.interaction_matrix(2, 0.25)
    assert m.dtype == np.float32 and m[0, 1] == np.float32(-0.25) and m[1, 1] == 1
    assert np.array_equal(M.interaction_matrix(1), np.eye(1, dtype=np.float32))


def test_workloads_deterministic():
    a, b = workload(1), workload(1)
    assert np.array_equal(a.graph.sources, b.graph.sources)
    w3 = workload(3, scale=0.01)
    assert w3.matrix.shape == (8, 8) and w3.bins.max() < 8


def test_shard_edges_balanced_and_total():
    from paper_1504_02687_b200.dist import shard_edges
    rng = np.random.default_rng(0)
    counts = rng.integers(2, 300, size=10_000)
    for world in (1, 2, 3, 8):
        parts = shard_edges(counts, world)
        assert parts[0][0] == 0 and parts[-1][1] == counts.size
        assert all(parts[r][1] == parts[r + 1][0] for r in range(world - 1))
        sizes = [counts[lo:hi].sum() for lo, hi in parts]
        assert max(sizes) - min(sizes) <= 2 * counts.max()


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "histobundle_b200.h")).read()
    return sorted(set(re.findall(r"HB_API\s+[\w\s\*]*?\b(hb_\w+)\s*\(", text)))


def test_header_and_bindings_agree():
    from paper_1504_02687_b200._native import SIGNATURES
    assert _header_symbols() == sorted(SIGNATURES)


def test_library_loads_and_exports_every_symbol():
    from paper_1504_02687_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        _native.build()
    lib = _native.load_library()
    assert lib.hb_abi_version() == 1
    nm = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r"\bT (hb_\w+)", nm))
    assert set(_header_symbols()) <= exported
    # workspace queries are pure host functions
    assert lib.hb_smooth_workspace_bytes(1, 16, 16) >= 16 * 16 * 12
    assert lib.hb_advect_partials() == 4096


def test_library_rejects_bad_arguments_without_gpu():
    from paper_1504_02687_b200 import _native
    lib = _native.load_library()
    assert lib.hb_splat(None, None, 5, 10, None, None, None, 1, 4, 4, None, None, None) == -1
    assert b"bad arguments" in lib.hb_last_error()
    assert lib.hb_advect_laplacian(None, None, None, 1, 1, None, None, None, 1, 8, 8, 1.0, 1e-8, 0.25,
                                   0, 0.5, 1, 1.0, None, None, None, None, None) == -1
    # flat advection: null buffers, a field too small for the interior margin,
    # a negative step
    assert lib.hb_advect_points(None, None, 1, 1, None, None, None, 1, 8, 8, 1.0, 1e-8, 0.25, 0,
                                None, None, None) == -1
    assert lib.hb_advect_points(None, None, 1, 1, None, None, None, 1, 2, 8, 1.0, 1e-8, 0.25, 0,
                                None, None, None) == -1
    # Laplacian + count: counts without pos, multi-pass without an output
    assert lib.hb_laplacian_count(None, None, None, 1, 1, 0.5, 1, 1.0, None, None, None) == -1
    assert b"hb_laplacian_count" in lib.hb_last_error()
    # capacity-checked emit needs a status word; clamp needs starts
    assert lib.hb_resample_emit_cap(None, None, 1, 1, None, None, None, 10, None, None, None, 1,
                                    1, None, None, None) == -1
    assert lib.hb_clamp_starts(None, 4, 10, None, None) == -1


def test_tiles_geometry():
    import ctypes
    from paper_1504_02687_b200 import _native
    lib = _native.load_library()
    t = _native.HbTiles()
    assert lib.hb_tiles_geometry(1, 1024, 1024, 1.5 * 4.64 + 2, ctypes.byref(t)) == 0
    assert t.tile == 64 and t.halo == 10 and t.ntx == t.nty == 16 and t.ntiles == 256
    # window (tile + 2 halo)^2 int32 must fit the 96 KB shared-memory budget
    assert lib.hb_tiles_geometry(4, 2048, 2048, 1.5 * 33.0 + 2, ctypes.byref(t)) == 0
    assert (t.tile + 2 * t.halo) ** 2 * 4 <= 96 * 1024 and t.ntiles == 4 * t.ntx * t.nty
    assert lib.hb_tiles_geometry(1, 70000, 10, 3.0, ctypes.byref(t)) == -1
    assert lib.hb_tiles_geometry(1, 100, 100, 200.0, ctypes.byref(t)) == -1
