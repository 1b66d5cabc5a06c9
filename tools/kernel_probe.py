"""Decompose the per-iteration kernels on a realistic mid-run state.

    python tools/kernel_probe.py [--config 4] [--iters 6]

Runs the workload for --iters iterations (so the polylines are bundled and
resampled like in the timed loop), then times, with CUDA events on the
current stream, variants of the two dominant kernels:
  emit+splat, emit only, splat only (standalone), advect+lap+count,
  advect+lap, lap only, count only.
Prints one JSON object.  Diagnostic tool; not part of the product path.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1504_02687_b200 import _native as N  # noqa: E402
from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200.engine import MIN_STEP, ptr, stream_ptr  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--sort-edges", default="none", choices=["none", "srcdst", "mid"],
                    help="experiment: reorder the graph's edges spatially first")
    args = ap.parse_args()
    w = workload(args.config)
    if args.sort_edges != "none":
        import numpy as np

        from paper_1504_02687_b200.model import Graph

        g = w.graph
        ps, pt = g.positions[g.sources], g.positions[g.targets]

        def q(v, bits):  # quantise [0,1] -> int
            return np.clip((v * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)

        def interleave(cols, bits):
            key = np.zeros(len(cols[0]), dtype=np.int64)
            for b in range(bits):
                for c, col in enumerate(cols):
                    key |= ((col >> b) & 1) << (b * len(cols) + c)
            return key

        if args.sort_edges == "srcdst":
            key = interleave([q(ps[:, 0], 8), q(ps[:, 1], 8), q(pt[:, 0], 8), q(pt[:, 1], 8)], 8)
        else:
            mid = 0.5 * (ps + pt)
            key = interleave([q(mid[:, 0], 16), q(mid[:, 1], 16)], 16)
        order = np.argsort(key, kind="stable")
        bins = None if w.bins is None else np.asarray(w.bins)[order]
        w = type(w)(**{**w.__dict__, "graph": Graph(g.positions, g.sources[order],
                                                         g.targets[order]), "bins": bins})
    eng, tr, _, _ = B.prepare_engine(w.graph, w.config, bins=w.bins, matrix=w.matrix)
    for _ in range(args.iters):
        eng.step()
    eng.sync_count()
    torch.cuda.synchronize()
    s = stream_ptr()
    E, Bn, nv, nu = eng.n_edges, eng.nbins, eng.nv, eng.nu
    # state: eng.pts holds final points of iteration iters-1, ecounts/pos valid
    # the real count input: final (advected + smoothed) points of iteration iters-1
    cnt_tmp = torch.empty_like(eng.ecounts)
    pos_tmp = torch.empty_like(eng.pos)
    out_count = timed(lambda: N.call(
        "hb_resample_count", ptr(eng.pts), ptr(eng.starts), E, float(w.config.delta),
        ptr(cnt_tmp), ptr(pos_tmp), s))
    # resample shape of the real state: pieces per kept point, chunk classes
    pos_i = pos_tmp[:eng.n_pts].long()
    st = eng.starts[:E + 1].long()
    kept = pos_i >= 0
    kp = torch.nonzero(kept).squeeze(1)
    pv = pos_i[kp]
    edge_of = torch.searchsorted(st, kp, right=True) - 1
    same = edge_of[1:] == edge_of[:-1]
    pieces = (pv[1:] - pv[:-1])[same]
    hist = torch.bincount(pieces.clamp_max(64)).cpu().tolist()
    tot = max(1, int(pieces.numel()))
    local = kp - st[edge_of]
    chunk_id = edge_of * 4096 + local // 32  # (edge, chunk) key, edges < 2^31/4096 chunks ok
    multi = torch.unique(chunk_id[1:][same & ((pv[1:] - pv[:-1]) != 1)])
    allp = torch.arange(eng.n_pts, device=pos_i.device)
    e_all = torch.searchsorted(st, allp, right=True) - 1
    ck_all = e_all * 4096 + (allp - st[e_all]) // 32
    dropped = torch.unique(ck_all[~kept])
    merged_chunks = int(torch.unique(torch.cat([multi, dropped])).numel())
    n_chunks = int(((st[1:] - st[:-1] + 31) // 32).sum().item())
    del allp, e_all, ck_all
    out_stats = {"pieces_hist_frac": {i: round(c / tot, 5) for i, c in enumerate(hist) if c},
                 "kept_frac": float(kept.float().mean().item()),
                 "complex_chunk_frac": merged_chunks / max(1, n_chunks)}
    del cnt_tmp, pos_tmp, pos_i, kp, pv, edge_of, pieces, local, chunk_id
    N.call("hb_scan_counts", ptr(eng.ecounts), E, ptr(eng.starts_alt), ptr(eng.scan_ws),
           eng.scan_ws.numel(), s)
    n_new = int(eng.starts_alt[E].item())
    eng._ensure_capacity(n_new)
    n_old = eng.n_pts
    out = {"config": w.name, "iteration_state": args.iters, "n_old": n_old, "n_new": n_new,
           "edges": E, "count_final_ms": out_count, "resample_shape": out_stats}

    def emit(splat: bool):
        if splat:
            eng.hist.zero_()
        N.call("hb_resample_emit", ptr(eng.pts), ptr(eng.starts), E, n_old, ptr(eng.pos),
               ptr(eng.starts_alt), ptr(eng.alt), ptr(eng.groups), ptr(eng.wint),
               ptr(eng.hist) if splat else None, nv, nu, ptr(eng.status), None, s)

    out["emit_splat_ms"] = timed(lambda: emit(True))
    out["emit_only_ms"] = timed(lambda: emit(False))
    out["hist_zero_ms"] = timed(lambda: eng.hist.zero_())

    def splat():
        eng.hist.zero_()
        N.call("hb_splat", ptr(eng.alt), ptr(eng.starts_alt), E, n_new, ptr(eng.groups),
               ptr(eng.wint), ptr(eng.hist), Bn, nv, nu, ptr(eng.status), None, s)

    out["splat_only_ms"] = timed(splat)
    if eng.tile_mode == 1:
        import ctypes
        tl = ctypes.byref(eng.tiles)

        def expand():
            N.call("hb_segtab_expand", tl, ptr(eng.hist), nv, nu, None, s)

        def emit_segtab():
            eng.hist.zero_()
            N.call("hb_resample_emit", ptr(eng.pts), ptr(eng.starts), E, n_old, ptr(eng.pos),
                   ptr(eng.starts_alt), ptr(eng.alt), ptr(eng.groups), ptr(eng.wint),
                   ptr(eng.hist), nv, nu, ptr(eng.status), tl, s)

        def splat_segtab():  # the emitted points splatted by a separate pass
            eng.hist.zero_()
            N.call("hb_splat", ptr(eng.alt), ptr(eng.starts_alt), E, n_new, ptr(eng.groups),
                   ptr(eng.wint), ptr(eng.hist), Bn, nv, nu, ptr(eng.status), tl, s)

        emit(False)
        out["splat_segtab_only_ms"] = timed(lambda: (splat_segtab(), expand()), reps=1)
        out["segtab"] = {"halo": eng.tiles.halo, "entries": int(eng.t_tab.numel())}
        out["emit_segtab_ms"] = timed(lambda: (emit_segtab(), expand()), reps=1)
        emit_segtab()
        out["segtab"]["nonzero_keys"] = int((eng.t_tab != 0).sum().item())
        out["expand_ms"] = timed(expand, reps=1)
        out["expand_empty_ms"] = timed(expand)
    if eng.tile_mode == 0:
        import ctypes
        tl = ctypes.byref(eng.tiles)
        # demand of the real pass that produced this state's plan
        N.call("hb_tiles_plan", tl, ptr(eng.t_total), s)
        fill_prev = None

        def emit_binned():
            eng.hist.zero_()
            eng.t_fill.zero_()
            N.call("hb_resample_emit", ptr(eng.pts), ptr(eng.starts), E, n_old, ptr(eng.pos),
                   ptr(eng.starts_alt), ptr(eng.alt), ptr(eng.groups), ptr(eng.wint),
                   ptr(eng.hist), nv, nu, ptr(eng.status), tl, s)

        eng._ensure_records(int(eng.t_total.item()))
        tl = ctypes.byref(eng.tiles)
        out["tiles"] = {"tile": eng.tiles.tile, "halo": eng.tiles.halo,
                        "ntiles": eng.tiles.ntiles, "records_capacity": int(eng.t_total.item())}
        out["emit_binned_ms"] = timed(emit_binned)
        fill = eng.t_fill.clone()
        cap = eng.t_cap.clone()
        out["tiles"]["demand"] = int(fill.sum().item())
        out["tiles"]["overflow"] = int((fill - cap).clamp_min(0).sum().item())
        out["tiles"]["max_tile_demand"] = int(fill.max().item())
        out["flush_ms"] = timed(lambda: N.call("hb_tiles_flush", tl, ptr(eng.hist), nv, nu, s))
        # plan sized exactly from this pass's own demand: no overflow
        N.call("hb_tiles_plan", tl, ptr(eng.t_total), s)
        eng._ensure_records(int(eng.t_total.item()))
        tl = ctypes.byref(eng.tiles)
        out["emit_binned_planned_ms"] = timed(emit_binned)
        fill = eng.t_fill.clone()
        out["tiles"]["overflow_planned"] = int((fill - eng.t_cap).clamp_min(0).sum().item())
        out["flush_planned_ms"] = timed(
            lambda: N.call("hb_tiles_flush", tl, ptr(eng.hist), nv, nu, s))
        # record multiplicity: identical (start cell, delta, k0, w) rasterise identically
        off = eng.t_off.cpu().numpy()
        fillc = torch.minimum(eng.t_fill, eng.t_cap).cpu().numpy()
        hot = int(fillc.argmax())
        recs = eng.t_rec[int(off[hot]):int(off[hot]) + int(fillc[hot])]
        out["tiles"]["hot_tile_records"] = int(recs.numel())
        out["tiles"]["hot_tile_unique"] = int(torch.unique(recs).numel())
        chunk = recs[: 16384]
        out["tiles"]["hot_chunk_unique_of_16384"] = int(torch.unique(chunk).numel())
        allr = torch.cat([eng.t_rec[int(off[t]):int(off[t]) + int(fillc[t])]
                          for t in range(len(fillc)) if fillc[t] > 0])
        out["tiles"]["all_unique"] = int(torch.unique(allr).numel())
        # per 16384-record chunk uniqueness over all tiles (what a chunk-local dedupe sees)
        tot_u = 0
        for t in range(len(fillc)):
            r = eng.t_rec[int(off[t]):int(off[t]) + int(fillc[t])]
            for c0 in range(0, r.numel(), 16384):
                tot_u += int(torch.unique(r[c0:c0 + 16384]).numel())
        out["tiles"]["chunk_local_unique"] = tot_u
        del fill_prev
    hist = eng.hist.clone()
    out["hist_max"] = int(hist.max().item())
    out["hist_nonzero_frac"] = float((hist > 0).float().mean().item())
    out["hist_sum"] = int(hist.sum().item())
    # field for advect
    N.call("hb_smooth", ptr(eng.hist), None, ptr(eng.mat_dev), Bn, nv, nu,
           eng.radii.data_ptr(), int(eng.radii.numel()), ptr(eng.field), ptr(eng.smooth_ws),
           eng.smooth_ws.numel(), ptr(eng.peak), s)
    cfg = w.config
    h = cfg.lambda_ ** args.iters * cfg.h_max
    work = torch.empty_like(eng.alt)

    gfield = torch.empty(N.lib().hb_grad_field_bytes(Bn, nv, nu) // 4, dtype=torch.float32,
                         device="cuda")
    N.call("hb_grad_field", ptr(eng.field), Bn, nv, nu, ptr(gfield), s)
    out["grad_field_ms"] = timed(lambda: N.call("hb_grad_field", ptr(eng.field), Bn, nv, nu,
                                                ptr(gfield), s))
    use_gf = [None]

    def adv(h_, lap, count):
        N.call("hb_advect_laplacian", ptr(eng.alt), ptr(work), ptr(eng.starts_alt), E, n_new,
               ptr(eng.groups), ptr(eng.field), use_gf[0], Bn, nv, nu, float(h_), float(cfg.epsilon),
               MIN_STEP, 0, float(cfg.laplacian_factor), lap, float(cfg.delta),
               ptr(eng.ecounts) if count else None, ptr(eng.pos) if count else None,
               eng.m_moved.data_ptr(), ptr(eng._partials), s)

    out["adv_lap_count_ms"] = timed(lambda: adv(h, 1, True))
    out["adv_lap_ms"] = timed(lambda: adv(h, 1, False))
    out["adv_only_ms"] = timed(lambda: adv(h, 0, False))
    out["lap_only_ms"] = timed(lambda: adv(-1.0, 1, False))
    out["count_only_ms"] = timed(lambda: adv(-1.0, 0, True))
    use_gf[0] = ptr(gfield)
    out["gf_adv_lap_count_ms"] = timed(lambda: adv(h, 1, True))
    out["gf_adv_lap_ms"] = timed(lambda: adv(h, 1, False))
    out["gf_adv_only_ms"] = timed(lambda: adv(h, 0, False))
    out["copy_pts_ms"] = timed(lambda: work[:n_new].copy_(eng.alt[:n_new]))
    # flat advection (in place on a copy) and the Laplacian+count pass after it
    work[:n_new].copy_(eng.alt[:n_new])

    def flat():
        N.call("hb_advect_points", ptr(work), ptr(eng.starts_alt), E, n_new, ptr(eng.groups),
               ptr(eng.field), ptr(gfield), Bn, nv, nu, float(h), float(cfg.epsilon), MIN_STEP, 0,
               eng.m_moved.data_ptr(), ptr(eng._partials), s)

    out["gf_flat_adv_ms"] = timed(flat, reps=1)
    cnt2 = torch.empty_like(eng.ecounts)
    pos2 = torch.empty_like(eng.pos)
    out["lap_count_ms"] = timed(lambda: N.call(
        "hb_advect_laplacian", ptr(work), ptr(work), ptr(eng.starts_alt), E, n_new, None, None,
        None, Bn, nv, nu, -1.0, float(cfg.epsilon), MIN_STEP, 0, float(cfg.laplacian_factor), 1,
        float(cfg.delta), ptr(cnt2), ptr(pos2), None, None, s), reps=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
