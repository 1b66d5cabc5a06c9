"""GPU parity: every kernel and the full loop against the CPU oracle and the
reference-generated golden fixtures.  Bit-exact is the bar for integer
histograms, points and fields; ``mean_displacement`` (an order-dependent
float64 sum in the reference too) is compared to rel 1e-12."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from golden_check import check_golden
from hb_hash import digest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
from paper_1504_02687_b200 import _native as N  # noqa: E402
from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200 import raster as R  # noqa: E402
from paper_1504_02687_b200.engine import box_widths, ptr, stream_ptr  # noqa: E402
from paper_1504_02687_b200.model import DensityField, SampledEdge  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402

# mean_displacement is a float64 sum over all interior points: its value depends
# on summation order (the reference itself changes with `workers`); the
# reference sums sequentially, we sum per-CTA partials in a fixed tree.
DISP_RTOL = 1e-9


def kat():
    return np.load(os.path.join(GOLDEN, "kat_ops.npz"))


_KEEP: list = []  # uploaded tensors must outlive the (asynchronous) kernels


@pytest.fixture(autouse=True)
def _release_uploads():
    yield
    torch.cuda.synchronize()
    _KEEP.clear()


def dev(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    _KEEP.append(t)
    return t


def sync():
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------
# per-kernel parity on the branch-coverage fixture


def test_native_library_is_the_loaded_path():
    lib = N.lib()
    assert lib.hb_abi_version() == 1
    assert lib.hb_device_sm_count() >= 100  # B200: 148


def test_splat_counts_match_reference_kat():
    k = kat()
    pts, starts, groups = k["pts"], k["starts"], k["groups"]
    nv, nu = int(k["nv"]), int(k["nu"])
    hist = torch.zeros((3, nv, nu), dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("hb_splat", ptr(dev(pts)), ptr(dev(starts)), len(starts) - 1, len(pts),
           ptr(dev(groups.astype(np.int32))), None, ptr(hist), 3, nv, nu, ptr(status), None,
           stream_ptr())
    sync()
    assert np.array_equal(hist.cpu().numpy().astype(np.float32), k["raw"])
    assert int(status.item()) == 0


def test_mix_layers_repulsive_matrix_kat():
    """Repulsive M (-alpha/(B-1)): per-group int counts mixed in f64 equal the
    reference's f32 accumulation on this small case."""
    k = kat()
    pts, starts, groups = k["pts"], k["starts"], k["groups"]
    nv, nu = int(k["nv"]), int(k["nu"])
    hist = torch.zeros((3, nv, nu), dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty((3, nv, nu), dtype=torch.float32, device="cuda")
    s = stream_ptr()
    N.call("hb_splat", ptr(dev(pts)), ptr(dev(starts)), len(starts) - 1, len(pts),
           ptr(dev(groups.astype(np.int32))), None, ptr(hist), 3, nv, nu, ptr(status), None, s)
    N.call("hb_mix_layers", ptr(hist), None, ptr(dev(k["mat"])), 3, nv, nu, ptr(out), s)
    sync()
    np.testing.assert_allclose(out.cpu().numpy(), k["raw_rep"], rtol=0, atol=1e-6)


def test_smooth_matches_reference_kat():
    k = kat()
    sm = R.smooth_gaussian_approx(DensityField(None, k["fld"]), 3.3, 3)
    assert np.array_equal(sm.values, k["sm"])
    assert np.array_equal(R.box_filter(k["fld"][0], 4), k["box"])


@pytest.mark.parametrize("delta,key", [(1.0, "rs1"), (2.5, "rs2")])
def test_resample_matches_reference_kat(delta, key):
    k = kat()
    pts, starts = k["pts"], k["starts"]
    E, n = len(starts) - 1, len(pts)
    dp, ds = dev(pts), dev(starts)
    counts = torch.empty(E, dtype=torch.int64, device="cuda")
    pos = torch.empty(n, dtype=torch.int32, device="cuda")
    ns = torch.empty(E + 1, dtype=torch.int64, device="cuda")
    ws = torch.empty(int(N.lib().hb_scan_workspace_bytes(E)), dtype=torch.uint8, device="cuda")
    s = stream_ptr()
    N.call("hb_resample_count", ptr(dp), ptr(ds), E, delta, ptr(counts), ptr(pos), s)
    N.call("hb_scan_counts", ptr(counts), E, ptr(ns), ptr(ws), ws.numel(), s)
    m = int(ns[-1].item())
    out = torch.empty((m, 2), dtype=torch.float64, device="cuda")
    N.call("hb_resample_emit", ptr(dp), ptr(ds), E, n, ptr(pos), ptr(ns), ptr(out), None, None,
           None, 1, 1, None, None, s)
    sync()
    assert np.array_equal(ns.cpu().numpy(), k[key + "_starts"])
    assert np.array_equal(out.cpu().numpy(), k[key])


@pytest.mark.parametrize("fixed", [False, True])
def test_advect_matches_reference_kat(fixed):
    k = kat()
    pts, starts, groups, rho = k["pts"], k["starts"], k["groups"], k["rho"]
    nb, nv, nu = rho.shape
    E, n = len(starts) - 1, len(pts)
    out = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    moved = torch.zeros(1, dtype=torch.int64, device="cuda")
    part = torch.zeros(int(N.lib().hb_advect_partials()), dtype=torch.float64, device="cuda")
    disp = torch.zeros(1, dtype=torch.float64, device="cuda")
    h = 3.0 if fixed else 6.0
    s = stream_ptr()
    N.call("hb_advect_laplacian", ptr(dev(pts)), ptr(out), ptr(dev(starts)), E, n,
           ptr(dev(groups.astype(np.int32))), ptr(dev(rho)), None, nb, nv, nu, h, 1e-8, 0.25,
           int(fixed), 0.5, 0, 1.0, None, None, ptr(moved), ptr(part), s)
    N.call("hb_reduce_f64", ptr(part), part.numel(), ptr(disp), s)
    sync()
    tag = "advf" if fixed else "adv"
    assert np.array_equal(out.cpu().numpy(), k[tag])
    assert int(moved.item()) == int(k[tag + "_stats"][1])
    np.testing.assert_allclose(disp.item(), k[tag + "_disp"][0], rtol=DISP_RTOL)


@pytest.mark.parametrize("factor,passes,key", [(0.5, 1, "lap"), (0.3, 3, "lap3")])
def test_laplacian_matches_reference_kat(factor, passes, key):
    k = kat()
    pts, starts = k["pts"], k["starts"]
    E, n = len(starts) - 1, len(pts)
    out = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    moved = torch.zeros(1, dtype=torch.int64, device="cuda")
    part = torch.zeros(int(N.lib().hb_advect_partials()), dtype=torch.float64, device="cuda")
    rho = torch.zeros((1, 3, 3), dtype=torch.float32, device="cuda")
    grp = torch.zeros(E, dtype=torch.int32, device="cuda")
    N.call("hb_advect_laplacian", ptr(dev(pts)), ptr(out), ptr(dev(starts)), E, n, ptr(grp),
           ptr(rho), None, 1, 3, 3, -1.0, 1e-8, 0.25, 0, factor, passes, 1.0, None, None, ptr(moved),
           ptr(part), stream_ptr())
    sync()
    assert np.array_equal(out.cpu().numpy(), k[key])


def test_probe_bilinear_and_gradient_kat():
    k = kat()
    rho = k["rho"][1]
    f = DensityField(None, k["rho"])
    for (x, y), b, g in list(zip(k["q"], k["bil"], k["grad"]))[:40]:
        assert B.density_at(f, 1, (x, y)) == b
        assert np.array_equal(B.gradient_at(f, 1, (x, y)), g)
    assert rho.dtype == np.float32


def test_used_cell_count_kat():
    k = kat()
    assert B.used_cell_count(DensityField(None, k["rho"])) == int(k["used"][0])


# ---------------------------------------------------------------------------
# random stress against the oracle (ragged edges, long edges, ties)


def _random_polylines(rng, n_edges, nv, nu, max_pts=400):
    lens = rng.integers(2, max_pts, size=n_edges)
    lens[rng.uniform(size=n_edges) < 0.3] = 2
    starts = np.zeros(n_edges + 1, dtype=np.int64)
    np.cumsum(lens, out=starts[1:])
    steps = rng.normal(0, 1.3, size=(int(starts[-1]), 2))
    steps[rng.uniform(size=steps.shape[0]) < 0.1] *= 0.05  # dense clusters -> merges
    pts = np.empty_like(steps)
    for e in range(n_edges):
        s, t = starts[e], starts[e + 1]
        p = np.cumsum(steps[s:t], axis=0) + rng.uniform([5, 5], [nu - 5, nv - 5])
        pts[s:t] = np.clip(p, 1.0, [nu - 2.0, nv - 2.0])
    return pts, starts


@pytest.mark.parametrize("seed", [0, 1])
def test_resample_emit_splat_random_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    nv, nu = 120, 150
    pts, starts = _random_polylines(rng, 700, nv, nu)
    E, n = len(starts) - 1, len(pts)
    groups = rng.integers(0, 2, size=E)
    delta = 1.7
    ref_pts, ref_starts = O.resample(pts.copy(), starts, delta, workers=1)
    ref_counts = O.accumulate_counts(ref_pts, ref_starts, groups, (nv, nu), 2)
    dp, ds = dev(pts), dev(starts)
    counts = torch.empty(E, dtype=torch.int64, device="cuda")
    pos = torch.empty(n, dtype=torch.int32, device="cuda")
    ns = torch.empty(E + 1, dtype=torch.int64, device="cuda")
    ws = torch.empty(int(N.lib().hb_scan_workspace_bytes(E)), dtype=torch.uint8, device="cuda")
    hist = torch.zeros((2, nv, nu), dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = stream_ptr()
    N.call("hb_resample_count", ptr(dp), ptr(ds), E, delta, ptr(counts), ptr(pos), s)
    N.call("hb_scan_counts", ptr(counts), E, ptr(ns), ptr(ws), ws.numel(), s)
    m = int(ns[-1].item())
    out = torch.empty((m, 2), dtype=torch.float64, device="cuda")
    N.call("hb_resample_emit", ptr(dp), ptr(ds), E, n, ptr(pos), ptr(ns), ptr(out),
           ptr(dev(groups.astype(np.int32))), None, ptr(hist), nv, nu, ptr(status), None, s)
    sync()
    assert np.array_equal(ns.cpu().numpy(), ref_starts)
    assert np.array_equal(out.cpu().numpy(), ref_pts)
    assert np.array_equal(hist.cpu().numpy(), ref_counts)


def test_resample_emit_long_edges_vs_oracle():
    """Edges of tens of thousands of points with long merged runs: warps of
    the flat emit start deep inside an edge (the 32-way cursor search on pos)
    and behind runs of dropped inputs (its linear fall-back)."""
    rng = np.random.default_rng(11)
    nv, nu = 200, 220
    lens = np.array([2, 60000, 3, 25000, 2, 2, 9000, 40000, 5], dtype=np.int64)
    starts = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=starts[1:])
    steps = rng.normal(0, 0.9, size=(int(starts[-1]), 2))
    steps[starts[1] + 100:starts[1] + 9000] *= 1e-3   # a 8900-point cluster: one long merge
    steps[starts[7] + 5000:starts[7] + 30000:2] *= 1e-2  # alternating merges
    pts = np.empty_like(steps)
    for e in range(lens.size):
        s_, t_ = starts[e], starts[e + 1]
        p = np.cumsum(steps[s_:t_], axis=0) * 0.05 + rng.uniform([20, 20], [nu - 20, nv - 20])
        pts[s_:t_] = np.clip(p, 1.0, [nu - 2.0, nv - 2.0])
    E, n = len(starts) - 1, len(pts)
    groups = rng.integers(0, 2, size=E)
    delta = 0.9
    ref_pts, ref_starts = O.resample(pts.copy(), starts, delta, workers=1)
    ref_counts = O.accumulate_counts(ref_pts, ref_starts, groups, (nv, nu), 2)
    dp, ds = dev(pts), dev(starts)
    counts = torch.empty(E, dtype=torch.int64, device="cuda")
    pos = torch.empty(n, dtype=torch.int32, device="cuda")
    ns = torch.empty(E + 1, dtype=torch.int64, device="cuda")
    ws = torch.empty(int(N.lib().hb_scan_workspace_bytes(E)), dtype=torch.uint8, device="cuda")
    hist = torch.zeros((2, nv, nu), dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = stream_ptr()
    N.call("hb_resample_count", ptr(dp), ptr(ds), E, delta, ptr(counts), ptr(pos), s)
    N.call("hb_scan_counts", ptr(counts), E, ptr(ns), ptr(ws), ws.numel(), s)
    m = int(ns[-1].item())
    out = torch.empty((m, 2), dtype=torch.float64, device="cuda")
    N.call("hb_resample_emit", ptr(dp), ptr(ds), E, n, ptr(pos), ptr(ns), ptr(out),
           ptr(dev(groups.astype(np.int32))), None, ptr(hist), nv, nu, ptr(status), None, s)
    sync()
    pos_h = pos.cpu().numpy()
    assert (pos_h < 0).sum() > 9000  # the merged runs are really there
    assert np.array_equal(ns.cpu().numpy(), ref_starts)
    assert np.array_equal(out.cpu().numpy(), ref_pts)
    assert np.array_equal(hist.cpu().numpy(), ref_counts)


def test_advect_laplacian_random_vs_oracle():
    rng = np.random.default_rng(7)
    nv, nu = 96, 128
    pts, starts = _random_polylines(rng, 500, nv, nu, max_pts=700)
    E, n = len(starts) - 1, len(pts)
    groups = rng.integers(0, 2, size=E)
    counts = O.accumulate_counts(pts, starts, groups, (nv, nu), 2)
    rho = O.smooth(counts.astype(np.float32), 4.0, 3)
    ref = pts.copy()
    interior, moved, disp = O.advect(ref, starts, groups, rho, 9.0, 1e-8, False)
    O.laplacian(ref, starts, 0.5, 2)
    out = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    dmoved = torch.zeros(1, dtype=torch.int64, device="cuda")
    part = torch.zeros(int(N.lib().hb_advect_partials()), dtype=torch.float64, device="cuda")
    # fused next-iteration resample count on the final points
    delta = 1.7
    counts = torch.empty(E, dtype=torch.int64, device="cuda")
    pos = torch.empty(n, dtype=torch.int32, device="cuda")
    N.call("hb_advect_laplacian", ptr(dev(pts)), ptr(out), ptr(dev(starts)), E, n,
           ptr(dev(groups.astype(np.int32))), ptr(dev(rho)), None, 2, nv, nu, 9.0, 1e-8, 0.25, 0, 0.5,
           2, delta, ptr(counts), ptr(pos), ptr(dmoved), ptr(part), stream_ptr())
    sync()
    assert np.array_equal(out.cpu().numpy(), ref)
    ref_counts = np.empty(E, dtype=np.int64)
    O.lib().orc_resample_count(O._p(ref), O._p(starts), delta, O._p(ref_counts), 0, E)
    assert np.array_equal(counts.cpu().numpy(), ref_counts)
    assert int(dmoved.item()) == moved
    np.testing.assert_allclose(part.sum().item(), disp, rtol=DISP_RTOL)


def test_smooth_random_multilayer_vs_oracle():
    rng = np.random.default_rng(3)
    vals = (rng.gamma(0.5, 2.0, size=(3, 77, 203)) *
            (rng.uniform(size=(3, 77, 203)) < 0.4)).astype(np.float32)
    for sigma in (1.0, 5.5, 12.0):
        got = R.smooth_gaussian_approx(DensityField(None, vals), sigma, 3).values
        assert np.array_equal(got, O.smooth(vals, sigma, 3)), sigma


@pytest.mark.parametrize("shape", [(1, 1), (5, 3), (77, 203), (300, 1030)])
def test_integral_image_vs_reference_expression(shape):
    """raster.integral_image (hb_integral_image) against the reference's own
    expression (raster.py:133-139): strict float64 cumsums down the columns,
    then along the rows, zero first row and column."""
    rng = np.random.default_rng(shape[0] + shape[1])
    lay = (rng.gamma(0.5, 2.0, size=shape) * (rng.uniform(size=shape) < 0.4)).astype(np.float32)
    ref = np.zeros((shape[0] + 1, shape[1] + 1), dtype=np.float64)
    ref[1:, 1:] = np.cumsum(np.cumsum(lay, axis=0, dtype=np.float64), axis=1)
    assert np.array_equal(R.integral_image(lay), ref)


# fused integral table (fold_kernel): strip widths 64 and 128, partial strips
# and row blocks, a single strip, and the two-kernel fallback (too many strips
# to be co-resident)
@pytest.mark.parametrize("shape", [(1, 37, 45), (2, 100, 200), (3, 257, 130), (1, 70, 64),
                                   (20, 40, 512), (40, 33, 1024)])
def test_smooth_fused_fold_shapes_vs_oracle(shape):
    rng = np.random.default_rng(sum(shape))
    vals = (rng.gamma(0.5, 2.0, size=shape) * (rng.uniform(size=shape) < 0.4)).astype(np.float32)
    for sigma in (2.0, 9.0):
        got = R.smooth_gaussian_approx(DensityField(None, vals), sigma, 3).values
        assert np.array_equal(got, O.smooth(vals, sigma, 3)), (shape, sigma)


# extreme aspect ratios and sizes: single cells, rows and columns, fewer rows
# than a 32-row block, more strips than co-resident CTAs at S = 64 (S = 128)
@pytest.mark.parametrize("shape,sigma", [((1, 1, 1), 2.0), ((1, 3, 700), 5.0),
                                         ((2, 700, 3), 5.0), ((1, 33, 10000), 3.0),
                                         ((3, 31, 129), 40.0), ((1, 64, 64), 0.6)])
def test_smooth_extreme_shapes_vs_oracle(shape, sigma):
    rng = np.random.default_rng(shape[1] * 7 + shape[2])
    vals = (rng.gamma(0.5, 2.0, size=shape) * (rng.uniform(size=shape) < 0.4)).astype(np.float32)
    got = R.smooth_gaussian_approx(DensityField(None, vals), sigma, 3).values
    assert np.array_equal(got, O.smooth(vals, sigma, 3)), (shape, sigma)


@pytest.mark.parametrize("seed", range(6))
def test_smooth_counts_random_shapes_match_float_path(seed):
    """Exact integer first pass (tile or separable + prefix rows) against the
    all-float path on random shapes and radii, bit for bit."""
    rng = np.random.default_rng(100 + seed)
    nb = int(rng.integers(1, 4))
    nv = int(rng.integers(1, 300))
    nu = int(rng.integers(1, 700))
    radii = [int(rng.integers(1, 60)), int(rng.integers(0, 60)), int(rng.integers(0, 60))]
    counts = (rng.poisson(2.0, size=(nb, nv, nu)) * (rng.uniform(size=(nb, nv, nu)) < 0.5)
              ).astype(np.int32)
    r = torch.tensor(radii, dtype=torch.int32)
    ws = torch.empty(int(N.lib().hb_smooth_workspace_bytes(nb, nv, nu)), dtype=torch.uint8,
                     device="cuda")
    c = dev(counts)
    ref = torch.empty((nb, nv, nu), dtype=torch.float32, device="cuda")
    got = torch.empty_like(ref)
    pk_ref = torch.zeros(nb, dtype=torch.float32, device="cuda")
    pk = torch.zeros_like(pk_ref)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("hb_smooth", ptr(c), None, None, nb, nv, nu, r.data_ptr(), 3, ptr(ref), ptr(ws),
           ws.numel(), ptr(pk_ref), stream_ptr())
    N.call("hb_smooth_counts", ptr(c), None, 1.0, 2.0 ** 24, nb, nv, nu, r.data_ptr(), 3,
           ptr(got), ptr(ws), ws.numel(), ptr(pk), ptr(status), stream_ptr())
    sync()
    assert torch.equal(got, ref), (nb, nv, nu, radii)
    assert torch.equal(pk, pk_ref)
    assert int(status.item()) == 0


def test_smooth_fused_fold_equals_two_fold_kernels_config5_map(monkeypatch):
    """The config-5 map (4 x 2047 x 2048, radii 50/51/51): fused fold vs the
    column-fold + row-fold kernels, bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(5)
    vals = (torch.rand((4, 2047, 2048), generator=g, device="cuda") ** 8 * 300).float()
    vals = vals.cpu().numpy()
    got = R.smooth_gaussian_approx(DensityField(None, vals), 51.2, 3).values
    monkeypatch.setenv("HB_FOLD", "0")
    ref = R.smooth_gaussian_approx(DensityField(None, vals), 51.2, 3).values
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------------------
# end to end against the reference goldens


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _check_run(k, scale=1.0, golden=None):
    """Config k against its reference golden: per-iteration raw histogram,
    smoothed field, N_i and metrics; final points / starts; and bundle()'s
    world polylines (golden_check.check_golden)."""
    w = workload(k, scale=scale)
    g = _golden(golden or f"cfg{k}.json")
    check_golden(w, g, workers=g.get("workers", 1), check_graph=False)


def test_bundle_cfg1_mini_world_points_bit_exact():
    w = workload(1, scale=0.25)
    res = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)
    ref = np.load(os.path.join(GOLDEN, "cfg1_mini.npz"))
    assert np.array_equal(res.sampled_edges.world, ref["world"])
    assert np.array_equal(res.density.values, ref["field"])
    e = res.sampled_edges[5]
    assert np.array_equal(e.points[0], w.graph.positions[w.graph.sources[5]])
    assert np.array_equal(e.points[-1], w.graph.positions[w.graph.targets[5]])


def test_bundle_cfg1_bit_exact():
    _check_run(1)


@pytest.mark.parametrize("mode", ["tiles", "direct"])
def test_bundle_cfg1_bit_exact_splat_paths(mode, monkeypatch):
    """The emit's splat through tile records (config 5's path) and through
    direct atomics gives the same bits as the segment-key table."""
    monkeypatch.setenv("HB_SPLAT_MODE", mode)
    _check_run(1)


@pytest.mark.parametrize("k", [1, 2])
def test_bundle_bit_exact_fused_field(k, monkeypatch):
    """hb_advect_laplacian_count (advection inside the Laplacian + count
    pass) gives the same bits as the two kernels."""
    monkeypatch.setenv("HB_FUSED_FIELD", "1")
    _check_run(k)


def test_bundle_cfg2_bit_exact():
    _check_run(2)


@pytest.mark.slow
def test_bundle_cfg3_bit_exact():
    if not os.path.exists(os.path.join(GOLDEN, "cfg3.json")):
        pytest.skip("cfg3 golden not generated")
    _check_run(3)


@pytest.mark.slow
def test_bundle_cfg4_bit_exact():
    if not os.path.exists(os.path.join(GOLDEN, "cfg4.json")):
        pytest.skip("cfg4 golden not generated")
    _check_run(4)


def test_bundle_on_iteration_and_fixed_step():
    w = workload(1, scale=0.1)
    w.config.iterations = 4
    seen = []
    res = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix, on_iteration=seen.append)
    assert [m.iteration for m in seen] == [0, 1, 2, 3]
    assert [m.moved_points for m in seen] == [m.moved_points for m in res.metrics]
    g = w.graph
    ref = O.bundle_packed(g.positions, g.sources, g.targets, g.weights, w.bins, w.config,
                          w.matrix, fixed_step=True)
    res_f = B.bundle(g, w.config, bins=w.bins, matrix=w.matrix, _fixed_step=True)
    assert np.array_equal(res_f.sampled_edges.world,
                          O.materialize(ref, g.positions, g.sources, g.targets))


def test_bundle_weights_offset_and_default_matrix_vs_oracle():
    """Integer weights, B=3 with the default repulsive matrix (-0.125 off the
    diagonal, dyadic, so every float32 layer sum is exact) and a directed
    offset: bit-exact vs the oracle."""
    w = workload(1, scale=0.15)
    g = w.graph
    rng = np.random.default_rng(0)
    weights = rng.integers(1, 4, size=g.n_edges).astype(np.float64)
    bins = (np.arange(g.n_edges) % 3).astype(np.int64)
    from paper_1504_02687_b200.model import Graph
    g2 = Graph(g.positions, g.sources, g.targets, weights, bins)
    cfg = w.config
    cfg.iterations = 4
    cfg.directed_offset_fraction = 0.002
    res = B.bundle(g2, cfg)
    ref = O.bundle_packed(g2.positions, g2.sources, g2.targets, weights, bins, cfg, None)
    world = O.materialize(ref, g2.positions, g2.sources, g2.targets)
    assert np.array_equal(res.sampled_edges.world, world)
    assert np.array_equal(res.density.values, ref.field)


# ---------------------------------------------------------------------------
# per-operator API (SPEC examples)


def test_spec_rasterize_segment():
    assert R.rasterize_segment((0.0, 0.0), (3.0, 0.0)).tolist() == [[0, 0], [1, 0], [2, 0], [3, 0]]
    assert R.rasterize_segment((0.0, 0.0), (0.0, 0.0)).tolist() == [[0, 0]]
    c = R.rasterize_segment((0.0, 0.0), (5.0, 3.0))
    assert c.shape == (6, 2) and (np.diff(c[:, 0]) == 1).all()


def test_spec_box_filter_impulse():
    a = np.zeros((21, 21), np.float32)
    a[10, 10] = 1.0
    out = R.box_filter(a, 2)
    assert np.allclose(out[8:13, 8:13], 1 / 25) and out.sum() == pytest.approx(1.0)
    assert np.array_equal(R.box_filter(a, 0), a)


def test_spec_advect_ramp_and_peak():
    u = np.arange(32, dtype=np.float32)
    ramp = np.tile(u, (32, 1))[None]
    f = DensityField(None, ramp)
    assert np.allclose(B.advect_point((10.0, 10.0), f, 0, 2.0), (12.0, 10.0))
    vv, uu = np.mgrid[0:41, 0:41]
    bump = np.exp(-((uu - 20.0) ** 2 + (vv - 20.0) ** 2) / 8.0).astype(np.float32)[None]
    assert np.array_equal(B.advect_point((20.0, 20.0), DensityField(None, bump), 0, 30.0),
                          (20.0, 20.0))


def test_spec_laplacian_and_resample():
    se = SampledEdge(0, np.array([[0.0, 0.0], [1.0, 2.0], [2.0, 0.0]]))
    B.laplacian_smooth(se, 0.5, 1)
    assert np.allclose(se.points[1], (1.0, 1.0))
    line = SampledEdge(0, np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]]))
    B.laplacian_smooth(line, 0.5, 1)
    assert np.array_equal(line.points[1], (1.0, 0.0))
    gap = SampledEdge(0, np.array([[0.0, 0.0], [4.0, 0.0]]))
    B.resample(gap, 1.0)
    assert gap.points.shape[0] == 5


def test_spec_initial_sample():
    from paper_1504_02687_b200.model import Graph, make_transform
    g = Graph(np.array([[0.0, 0.0], [9.0, 0.0], [0.0, 9.0]]), [0, 0], [1, 2])
    tr = make_transform(g.positions, 10, 0)  # cell = 1 world unit
    se = B.initial_sample(g, tr, 3.0)
    assert len(se[0]) == 4 and se[0].points[:, 0].tolist() == [0.0, 3.0, 6.0, 9.0]
    assert se[1].points[-1].tolist() == [0.0, 9.0]


def test_accumulate_edges_spec_overlap():
    from paper_1504_02687_b200.model import Graph, make_transform
    g = Graph(np.array([[0.0, 0.0], [10.0, 0.0], [0.0, 10.0]]), [0, 0], [1, 1])
    tr = make_transform(g.positions, 16, 2)
    se = B.initial_sample(g, tr, 3.0)
    f = R.accumulate_edges(se, g, np.eye(1, dtype=np.float32), tr)
    assert f.values.max() == 2.0


# ---------------------------------------------------------------------------
# lane-sequential Laplacian + resample count (hb_lapcount.cu)

def _lc_case(shape: str):
    """Polylines stressing the speculative per-lane walk: merge chains longer
    than a 32-point run, pieces > 1, 2-point edges, ranges spanning many
    1024-point groups."""
    rng = np.random.default_rng({"random": 3, "chains": 4, "short": 5, "big": 6}[shape])
    delta = 1.7
    if shape == "random":
        pts, starts = _random_polylines(rng, 400, 96, 128, max_pts=700)
        return pts, starts, delta
    if shape == "short":
        lens = rng.integers(2, 5, size=20000)
    elif shape == "chains":
        lens = rng.integers(2, 900, size=300)
    else:  # big: > 1024 points per warp range on a full B200 grid
        lens = rng.integers(300, 700, size=12000)
    starts = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=starts[1:])
    n = int(starts[-1])
    step = rng.normal(0, 1.0, size=(n, 2)) * delta
    u = rng.uniform(size=n)
    if shape == "chains":
        # runs of tiny steps (merge chains of random length) and big jumps
        tiny = np.zeros(n, dtype=bool)
        i = 0
        while i < n:
            k = int(rng.integers(1, 120))
            if rng.uniform() < 0.5:
                tiny[i:i + k] = True
            i += k
        step[tiny] *= 0.02
        step[u < 0.03] *= 8.0
    else:
        step[u < 0.25] *= 0.05
        step[u > 0.97] *= 6.0
    pts = np.cumsum(step, axis=0) + 500.0
    return pts, starts, delta


@pytest.mark.parametrize("inplace", [False, True])
@pytest.mark.parametrize("shape", ["random", "chains", "short", "big"])
def test_laplacian_count_vs_oracle(shape, inplace):
    pts, starts, delta = _lc_case(shape)
    E, n = len(starts) - 1, len(pts)
    ref = pts.copy()
    O.laplacian(ref, starts, 0.5, 1)
    ref_counts = np.empty(E, dtype=np.int64)
    O.lib().orc_resample_count(O._p(ref), O._p(starts), delta, O._p(ref_counts), 0, E)
    dp, ds = dev(pts), dev(starts)
    out = dp if inplace else torch.empty((n, 2), dtype=torch.float64, device="cuda")
    counts = torch.full((E,), -7, dtype=torch.int64, device="cuda")
    pos = torch.full((n,), -7, dtype=torch.int32, device="cuda")
    N.call("hb_laplacian_count", ptr(dp), ptr(out), ptr(ds), E, n, 0.5, 1, delta, ptr(counts),
           ptr(pos), stream_ptr())
    sync()
    assert np.array_equal(out.cpu().numpy(), ref)
    assert np.array_equal(counts.cpu().numpy(), ref_counts)
    # pos: the per-edge (ballot) implementation on the same final points, and
    # the emitted polylines against the oracle's resample
    pos2 = torch.empty_like(pos)
    counts2 = torch.empty_like(counts)
    moved = torch.zeros(1, dtype=torch.int64, device="cuda")
    part = torch.zeros(int(N.lib().hb_advect_partials()), dtype=torch.float64, device="cuda")
    N.call("hb_advect_laplacian", ptr(dev(ref)), ptr(torch.empty_like(out)), ptr(ds), E, n, None,
           None, None, 1, 3, 3, -1.0, 1e-8, 0.25, 0, 0.5, 0, delta, ptr(counts2), ptr(pos2),
           ptr(moved), ptr(part), stream_ptr())
    sync()
    assert np.array_equal(pos.cpu().numpy(), pos2.cpu().numpy())
    assert np.array_equal(counts2.cpu().numpy(), ref_counts)
    if shape in ("random", "chains"):
        ref_pts, ref_starts = O.resample(ref, starts, delta)
        ns = torch.zeros(E + 1, dtype=torch.int64, device="cuda")
        ns[1:] = torch.cumsum(counts, 0)
        emitted = torch.empty((int(ns[-1].item()), 2), dtype=torch.float64, device="cuda")
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        N.call("hb_resample_emit", ptr(out), ptr(ds), E, n, ptr(pos), ptr(ns), ptr(emitted),
               None, None, None, 1, 1, ptr(status), None, stream_ptr())
        sync()
        assert np.array_equal(ns.cpu().numpy(), ref_starts)
        assert np.array_equal(emitted.cpu().numpy(), ref_pts)


def test_laplacian_count_passes_and_count_only():
    pts, starts, delta = _lc_case("random")
    E, n = len(starts) - 1, len(pts)
    for passes, factor in [(0, 0.5), (3, 0.3)]:
        ref = pts.copy()
        if passes:
            O.laplacian(ref, starts, factor, passes)
        ref_counts = np.empty(E, dtype=np.int64)
        O.lib().orc_resample_count(O._p(ref), O._p(starts), delta, O._p(ref_counts), 0, E)
        out = torch.empty((n, 2), dtype=torch.float64, device="cuda")
        counts = torch.empty(E, dtype=torch.int64, device="cuda")
        pos = torch.empty(n, dtype=torch.int32, device="cuda")
        N.call("hb_laplacian_count", ptr(dev(pts)), ptr(out), ptr(dev(starts)), E, n, factor,
               passes, delta, ptr(counts), ptr(pos), stream_ptr())
        sync()
        assert np.array_equal(out.cpu().numpy(), ref)
        assert np.array_equal(counts.cpu().numpy(), ref_counts)
    # Laplacian only (no counts)
    ref = pts.copy()
    O.laplacian(ref, starts, 0.5, 1)
    out = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    N.call("hb_laplacian_count", ptr(dev(pts)), ptr(out), ptr(dev(starts)), E, n, 0.5, 1, delta,
           None, None, stream_ptr())
    sync()
    assert np.array_equal(out.cpu().numpy(), ref)


# ---------------------------------------------------------------------------
# small and degenerate shapes through the public API, bit-exact vs the oracle

def _graph_from(pos, src, dst, bins=None):
    from paper_1504_02687_b200.model import Graph
    return Graph(np.asarray(pos, dtype=np.float64), np.asarray(src, dtype=np.int64),
                 np.asarray(dst, dtype=np.int64), None, bins)


def _small_case(name):
    from paper_1504_02687_b200.model import BundleConfig
    rng = np.random.default_rng(len(name))
    if name == "one_edge":
        return _graph_from([[0.1, 0.2], [0.9, 0.7]], [0], [1]), BundleConfig(grid_size=32,
                                                                             iterations=3)
    if name == "tiny_grid":
        pos = rng.uniform(0, 1, size=(20, 2))
        src = rng.integers(0, 20, size=60)
        dst = (src + 1 + rng.integers(0, 19, size=60)) % 20
        return _graph_from(pos, src, dst), BundleConfig(grid_size=8, delta=1.0, iterations=4)
    if name == "two_point_edges":  # delta larger than every edge: 2 samples each
        pos = rng.uniform(0, 1, size=(300, 2))
        src = rng.integers(0, 300, size=2000)
        dst = (src + 1 + rng.integers(0, 299, size=2000)) % 300
        return _graph_from(pos, src, dst), BundleConfig(grid_size=64, delta=500.0, iterations=3)
    if name == "dense_short":  # many near-coincident clusters: merges everywhere
        centers = rng.uniform(0.2, 0.8, size=(4, 2))
        pos = centers[rng.integers(0, 4, size=400)] + rng.normal(0, 0.01, size=(400, 2))
        src = rng.integers(0, 400, size=3000)
        dst = (src + 1 + rng.integers(0, 399, size=3000)) % 400
        return _graph_from(pos, src, dst), BundleConfig(grid_size=128, delta=0.7, iterations=5,
                                                        lambda_=1.0)
    if name == "groups_identity":  # 3 groups, identity matrix, 1-pass smoothing
        pos = rng.uniform(0, 1, size=(200, 2))
        src = rng.integers(0, 200, size=1500)
        dst = (src + 1 + rng.integers(0, 199, size=1500)) % 200
        bins = rng.integers(0, 3, size=1500)
        return (_graph_from(pos, src, dst, bins),
                BundleConfig(grid_size=96, iterations=3, smoothing_passes=1, alpha=0.0))
    raise KeyError(name)


@pytest.mark.parametrize("name", ["one_edge", "tiny_grid", "two_point_edges", "dense_short",
                                  "groups_identity"])
def test_bundle_small_shapes_vs_oracle(name):
    g, cfg = _small_case(name)
    res = B.bundle(g, cfg)
    ref = O.bundle_packed(g.positions, g.sources, g.targets, g.weights, g.bins, cfg, None)
    world = O.materialize(ref, g.positions, g.sources, g.targets)
    assert np.array_equal(res.sampled_edges.starts, ref.starts)
    assert np.array_equal(res.sampled_edges.world, world)
    assert np.array_equal(res.density.values, ref.field)
    for m, r in zip(res.metrics, ref.metrics):
        assert (m.moved_points, m.used_cells) == (r.moved_points, r.used_cells)
        assert m.bandwidth == r.bandwidth
        np.testing.assert_allclose(m.mean_displacement, r.mean_displacement, rtol=DISP_RTOL)


def test_sync_free_capacity_overflow_retries_exactly(monkeypatch):
    """The sync-free loop keeps N_i on the device; when a resample outgrows
    the buffers the run is redone with room for it -- same bits either way,
    and a following reset()+run() needs no retry."""
    w = workload(1, scale=0.5)
    cfg = w.config
    monkeypatch.setenv("HB_SYNC_FREE", "0")
    ref, _, ref_m = B.bundle_packed(w.graph, cfg, bins=w.bins, matrix=w.matrix)
    rp, rs = (t.cpu().numpy() for t in ref.packed_points())
    monkeypatch.setenv("HB_SYNC_FREE", "1")
    monkeypatch.setenv("HB_ASYNC_CAP_FACTOR", "0.5")  # below N_0 x growth: overflows
    eng, _, metrics = B.bundle_packed(w.graph, cfg, bins=w.bins, matrix=w.matrix,
                                      capacity_factor=1.0)
    assert getattr(eng, "_cap_retries", 0) >= 1 and eng.async_n
    pts, starts = (t.cpu().numpy() for t in eng.packed_points())
    assert np.array_equal(starts, rs) and np.array_equal(pts, rp)
    assert [m.moved_points for m in metrics] == [m.moved_points for m in ref_m]
    retries = eng._cap_retries
    eng.reset()
    eng.run()
    assert eng._cap_retries == retries
    pts2 = eng.packed_points()[0].cpu().numpy()
    assert np.array_equal(pts2, rp)
    res = B.bundle(w.graph, cfg, bins=w.bins, matrix=w.matrix)
    assert np.array_equal(res.sampled_edges.starts, rs)

@pytest.mark.parametrize("limit", [2.0 ** 24, 2.0 ** 20])
@pytest.mark.parametrize("mixed", [False, True])
def test_smooth_counts_integer_first_pass_matches_float_path(limit, mixed):
    """hb_smooth_counts (exact integer first pass) equals hb_smooth (the
    reference's float64 integral-image folds) bit for bit, and the guard
    flags a cell past the limit."""
    rng = np.random.default_rng(5)
    nb, nv, nu = 3, 131, 517
    counts = (rng.poisson(3.0, size=(nb, nv, nu)) *
              (rng.uniform(size=(nb, nv, nu)) < 0.5)).astype(np.int32)
    counts[1, 60:70, 100:140] += 4000  # a bundle
    mat = (np.eye(nb) + 0.5 * (1 - np.eye(nb))).astype(np.float32) if mixed else None
    mix = (mat * 2).astype(np.int32) if mixed else None
    scale = 0.5 if mixed else 1.0
    for radii in ([15, 15, 16], [1, 0, 2], [40, 41, 41], [51, 51, 51]):
        r = torch.tensor(radii, dtype=torch.int32)
        ws = torch.empty(int(N.lib().hb_smooth_workspace_bytes(nb, nv, nu)), dtype=torch.uint8,
                         device="cuda")
        c = dev(counts)
        ref = torch.empty((nb, nv, nu), dtype=torch.float32, device="cuda")
        got = torch.empty_like(ref)
        pk_ref = torch.zeros(nb, dtype=torch.float32, device="cuda")
        pk = torch.zeros_like(pk_ref)
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        N.call("hb_smooth", ptr(c), None, ptr(dev(mat) if mixed else None), nb, nv, nu,
               r.data_ptr(), 3, ptr(ref), ptr(ws), ws.numel(), ptr(pk_ref), stream_ptr())
        N.call("hb_smooth_counts", ptr(c), ptr(dev(mix) if mixed else None), scale, limit, nb,
               nv, nu, r.data_ptr(), 3, ptr(got), ptr(ws), ws.numel(), ptr(pk), ptr(status),
               stream_ptr())
        sync()
        assert torch.equal(got, ref), radii
        assert torch.equal(pk, pk_ref)
        assert int(status.item()) == 0
    r3 = torch.tensor([3, 3, 3], dtype=torch.int32)
    with pytest.raises(N.NativeError):  # int32 window sums could overflow: refused
        N.call("hb_smooth_counts", ptr(dev(counts)), None, 1.0, 2.0 ** 40, nb, nv, nu,
               r3.data_ptr(), 3, ptr(got), ptr(ws), ws.numel(), None, None, stream_ptr())
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("hb_smooth_counts", ptr(dev(counts)), None, 1.0, 4000.0, nb, nv, nu,
           r3.data_ptr(), 3, ptr(got), ptr(ws), ws.numel(), None, ptr(status), stream_ptr())
    sync()
    assert int(status.item()) & 8  # 4000+ counts reach the limit


@pytest.mark.parametrize("env", [{"HB_QUAD_LIMIT_MB": "0"}, {"HB_FLAT_ADVECT": "0"},
                                 {"HB_SYNC_FREE": "0"}, {"HB_SMOOTH_INT": "0"},
                                 {"HB_STREAM_OUT": "0"}])
def test_bundle_cfg2_bit_exact_alternate_paths(env, monkeypatch):
    """Every switchable path gives the reference's bits: advection gathering
    rho directly (no quad field, as for fields past the memory limit), the
    per-edge fused advect + Laplacian kernel, synchronous point totals, the
    float64-fold first smoothing pass, and the unstreamed result copy."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _check_run(2)
