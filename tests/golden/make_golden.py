"""Generate tests/golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [--big]

It imports the reference package from /root/reference/pkg/src (numba +
numpy), replays ``bundler.bundle``'s loop (bundler.py:351-376) with the
reference's own stage functions so every stage output of every iteration can
be hashed, checks the replay equals ``bundle()`` itself, and writes:

  cfg{k}.json        per-iteration sha256 of raw histogram / smoothed field /
                     points+starts, metrics, final shapes, versions
  cfg1_mini.npz      a 500-edge config-1 run with full arrays (diagnostics)
  kat_ops.npz        per-operator known-answer cases (branch coverage for
                     accumulate / resample / laplacian / advect / smoothing)

The GPU box never reads /root/reference: only these committed files travel.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import numba  # noqa: E402
from histobundle import _kernels as RK  # noqa: E402
from histobundle import bundler as RB  # noqa: E402
from histobundle import model as RM  # noqa: E402
from histobundle import raster as RR  # noqa: E402

from hb_hash import digest  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402

VERSIONS = {"numpy": np.__version__, "numba": numba.__version__,
            "python": sys.version.split()[0]}


def ref_graph(w):
    g = w.graph
    return RM.Graph.from_arrays(g.positions, g.sources, g.targets, g.weights,
                                g.bins)


def ref_config(cfg):
    return RM.BundleConfig(**{f: getattr(cfg, f)
                              for f in cfg.__dataclass_fields__})


def replay(w, workers):
    """bundler.py:325-376 step by step with the reference's own functions."""
    g = ref_graph(w)
    cfg = ref_config(w.config)
    bins = np.ascontiguousarray(w.bins, dtype=np.int64)
    matrix = np.asarray(w.matrix, dtype=np.float32)
    nbins = matrix.shape[0]
    tr = RM.make_transform(g.positions, cfg.grid_size, cfg.padding_cells)
    pts, starts = RB._sample_packed(g, tr, cfg.delta)
    layer_w = np.ascontiguousarray(
        g.weights.astype(np.float32)[:, None] * matrix.T[bins])
    iters = []
    for i in range(cfg.iterations):
        if i > 0:
            pts, starts = RB._resample_packed(pts, starts, cfg.delta, workers)
        n_i = int(pts.shape[0])
        raw = RR._accumulate_packed(pts, starts, layer_w, tr.shape, workers)
        field = RR.smooth_gaussian_approx(RM.DensityField(tr, raw), cfg.sigma,
                                          cfg.smoothing_passes, workers)
        h_i = cfg.lambda_ ** i * cfg.h_max
        interior, moved, disp = RB._advect_packed(pts, starts, bins,
                                                  field.values, h_i,
                                                  cfg.epsilon, False, workers)
        RB._laplacian_packed(pts, starts, cfg.laplacian_factor,
                             cfg.laplacian_passes, workers)
        iters.append({
            "iteration": i, "n_points": n_i, "bandwidth": h_i,
            "moved_points": int(moved), "interior": int(interior),
            "disp": float(disp),
            "mean_displacement": disp / interior if interior else 0.0,
            "used_cells": RB.used_cell_count(field),
            "raw": digest(raw), "field": digest(field.values),
            "pts": digest(pts), "starts": digest(starts),
        })
    return g, cfg, tr, pts, starts, field, iters


def golden_config(k, workers, scale=1.0, save_arrays=None):
    w = workload(k, scale=scale)
    g, cfg, tr, pts, starts, field, iters = replay(w, workers)
    # the replay must equal the public entry point bit for bit
    res = RB.bundle(g, cfg, bins=w.bins, matrix=w.matrix, workers=workers)
    world = np.concatenate([se.points for se in res.sampled_edges])
    assert np.array_equal(res.density.values, field.values)
    for a, b in zip(res.metrics, iters):
        assert a.moved_points == b["moved_points"]
        assert a.used_cells == b["used_cells"]
    out = {
        "config": k, "scale": scale, "workload": w.name, "workers": workers,
        "bundle_config": {f: getattr(w.config, f)
                          for f in w.config.__dataclass_fields__},
        "grid": [int(field.values.shape[0]), tr.height, tr.width],
        "transform": [tr.origin[0], tr.origin[1], tr.cell_size, tr.width,
                      tr.height],
        "n_edges": g.n_edges, "iterations": iters,
        "final_world": digest(world), "final_pts": digest(pts),
        "final_starts": digest(starts), "final_field": digest(field.values),
        "versions": VERSIONS,
    }
    if save_arrays:
        np.savez_compressed(save_arrays, world=world, pts=pts, starts=starts,
                            field=field.values)
    return out


def kat_ops():
    """Small hand-made cases covering the kernels' branches."""
    rng = np.random.default_rng(1234)
    nv, nu = 40, 48
    polys = [
        np.array([[5.0, 5.0], [5.2, 5.3], [12.0, 5.0]]),        # zero-length seg at j==0
        np.array([[20.0, 20.0], [24.0, 22.0], [24.1, 22.2], [30.4, 30.6]]),  # zero-length at j>0
        np.array([[3.0, 30.0], [3.4, 30.1], [3.6, 30.2], [3.9, 30.3],
                  [20.0, 35.0]]),                               # dense cluster (gap merge)
        np.array([[10.0, 10.0], [40.0, 14.0]]),                 # long gap -> power-of-two pieces
        np.array([[44.0, 3.0], [44.0, 3.0]]),                   # coincident endpoints
        np.array([[7.5, 7.5], [8.5, 8.5], [9.5, 7.5], [10.5, 8.49999999]]),  # .5 rounding ties
    ]
    for _ in range(30):
        n = int(rng.integers(2, 12))
        p = np.cumsum(rng.normal(0, 2.0, size=(n, 2)), axis=0) + [24.0, 20.0]
        polys.append(np.clip(p, 1.0, [nu - 2.0, nv - 2.0]))
    counts = np.array([p.shape[0] for p in polys], dtype=np.int64)
    starts = np.zeros(len(polys) + 1, dtype=np.int64)
    np.cumsum(counts, out=starts[1:])
    pts = np.ascontiguousarray(np.concatenate(polys), dtype=np.float64)
    ne = len(polys)
    groups = (np.arange(ne) % 3).astype(np.int64)
    eye_w = np.ascontiguousarray(np.eye(3, dtype=np.float32)[groups])
    raw = np.zeros((3, nv, nu), np.float32)
    RK.accumulate(pts, starts, eye_w, raw, 0, ne)
    mat = RM.interaction_matrix(3, 0.25)
    lw = np.ascontiguousarray(np.float32(1.0) * mat.T[groups])
    raw_rep = np.zeros((3, nv, nu), np.float32)
    RK.accumulate(pts, starts, lw, raw_rep, 0, ne)
    # smoothing of a random non-integer field (passes 2/3 order sensitivity)
    fld = (rng.gamma(0.6, 3.0, size=(2, nv, nu)) * (rng.uniform(size=(2, nv, nu)) < 0.3)).astype(np.float32)
    sm = RR.smooth_gaussian_approx(RM.DensityField(None, fld), 3.3, 3, 1).values
    box = RR.box_filter(fld[0], 4)
    # resample
    for delta in (1.0, 2.5):
        c = np.empty(ne, dtype=np.int64)
        RK.resample_count(pts, starts, delta, c, 0, ne)
        ns = np.zeros(ne + 1, dtype=np.int64)
        np.cumsum(c, out=ns[1:])
        o = np.empty((int(ns[-1]), 2))
        RK.resample_emit(pts, starts, delta, ns, o, 0, ne)
        if delta == 1.0:
            rs1, rs1_starts = o, ns
        else:
            rs2, rs2_starts = o, ns
    lap = pts.copy()
    RK.laplacian(lap, starts, 0.5, 1, np.empty_like(lap), 0, ne)
    lap3 = pts.copy()
    RK.laplacian(lap3, starts, 0.3, 3, np.empty_like(lap3), 0, ne)
    # advect over the smoothed per-group histogram
    rho = RR.smooth_gaussian_approx(RM.DensityField(None, raw), 2.0, 3, 1).values
    adv = pts.copy()
    adv_stats = RK.advect(adv, starts, groups, rho, 6.0, 1e-8, 0.25, False, 0, ne)
    advf = pts.copy()
    advf_stats = RK.advect(advf, starts, groups, rho, 3.0, 1e-8, 0.25, True, 0, ne)
    # sampled points for gradient / bilinear
    q = np.column_stack([rng.uniform(0.0, nu - 1.0, 200), rng.uniform(0.0, nv - 1.0, 200)])
    bil = np.array([RK.bilinear_value(rho[1], x, y) for x, y in q])
    grad = np.array([RK.gradient_xy(rho[1], x, y) for x, y in q])
    used = RB.used_cell_count(RM.DensityField(None, rho))
    return dict(nv=nv, nu=nu, pts=pts, starts=starts, groups=groups, raw=raw,
                mat=mat, raw_rep=raw_rep, fld=fld, sm=sm, box=box,
                rs1=rs1, rs1_starts=rs1_starts, rs2=rs2, rs2_starts=rs2_starts,
                lap=lap, lap3=lap3, rho=rho, adv=adv,
                adv_stats=np.array(adv_stats[:2], dtype=np.int64),
                adv_disp=np.array([adv_stats[2]]), advf=advf,
                advf_stats=np.array(advf_stats[:2], dtype=np.int64),
                advf_disp=np.array([advf_stats[2]]), q=q, bil=bil, grad=grad,
                used=np.array([used]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true",
                    help="also configs 3 and 4 (minutes of CPU)")
    ap.add_argument("--workers", type=int, default=8)
    args = ap.parse_args()
    np.savez_compressed(os.path.join(HERE, "kat_ops.npz"), **kat_ops())
    mini = golden_config(1, 1, scale=0.25,
                         save_arrays=os.path.join(HERE, "cfg1_mini.npz"))
    with open(os.path.join(HERE, "cfg1_mini.json"), "w") as f:
        json.dump(mini, f, indent=1)
    ks = [1, 2] + ([3, 4] if args.big else [])
    for k in ks:
        out = golden_config(k, args.workers)
        with open(os.path.join(HERE, f"cfg{k}.json"), "w") as f:
            json.dump(out, f, indent=1)
        print("wrote", k, out["workload"], out["final_world"]["sha256"][:16])


if __name__ == "__main__":
    main()
