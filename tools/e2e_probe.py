"""Phase breakdown of the public bundle() call (host in, host out).

    python tools/e2e_probe.py [--config 4] [--reps 3]

Replays bundle()'s steps (bundler.py) with a device sync after each and
prints one JSON object of wall-clock seconds per phase (median of --reps).
Diagnostic tool; not part of the product path.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200 import engine as EN  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402


def one(w) -> dict:
    g, cfg = w.graph, w.config
    out = {}
    t = time.perf_counter()

    def lap(name):
        nonlocal t
        torch.cuda.synchronize()
        now = time.perf_counter()
        out[name] = now - t
        t = now

    c, bins_arr, matrix = B._resolve(g, cfg, w.bins, w.matrix)
    eng, tr, lo, hi = B._setup(g, c, bins_arr, matrix, False, None, 2.0)
    lap("setup (transform, device sampling, uploads, allocations)")
    eng.run()
    lap("iterations")
    recs = eng.finish_metrics()
    lap("metrics")
    wd = eng.world_points_nodes(tr.origin, tr.cell_size, *eng.node_arrays)
    lap("grid->world + endpoint pinning")
    host = EN.download_pinned(wd)
    lap("D2H polylines (pinned)")
    starts = EN.download(eng.starts)
    field = EN.download(eng.field)
    lap("D2H starts + field")
    out["gbytes_d2h"] = wd.numel() * 8 / 1e9
    del host, starts, field, recs
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    w = workload(args.config)
    B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)  # warm
    runs = [one(w) for _ in range(args.reps)]
    res = {k: round(statistics.median(r[k] for r in runs), 4) for k in runs[0]}
    res["d2h_GBps"] = round(res["gbytes_d2h"] / res["D2H polylines (pinned)"], 1)
    t0 = time.perf_counter()
    r = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)
    torch.cuda.synchronize()
    res["bundle_total"] = round(time.perf_counter() - t0, 4)
    del r
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
