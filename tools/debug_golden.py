"""Localise a per-iteration golden mismatch on the GPU box.

    python tools/debug_golden.py table1_b1 [--mode auto|table|tiles|direct] [--sync]

Steps the engine against tests/golden/<name>.json; at the first iteration
whose raw histogram differs it compares the engine's own resampled points
(before the splat) with the C oracle's resample of the previous iteration's
points, and the engine's histogram with the oracle's accumulate of the
engine's points, printing where they first differ.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import torch  # noqa: E402

import oracle as O  # noqa: E402
from golden_check import _raw_h  # noqa: E402
from hb_hash import digest  # noqa: E402
from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200.workloads import table1_workload, workload  # noqa: E402


def load_workload(name, g):
    if name.startswith("table1_b"):
        b = int(name.split("_b")[1].split("_")[0])
        return table1_workload(200_000, b)
    if name == "cfg5_slice":
        return workload(5, scale=g["scale"])
    k = int(name[3])
    return workload(k)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--sync", action="store_true")
    a = ap.parse_args()
    os.environ["HB_SPLAT_MODE"] = a.mode
    if a.sync:
        os.environ["HB_SYNC_FREE"] = "0"
    g = json.load(open(os.path.join(ROOT, "tests", "golden", f"{a.name}.json")))
    w = load_workload(a.name, g)
    eng, tr, _, _ = B.prepare_engine(w.graph, w.config, bins=w.bins, matrix=w.matrix,
                                     workers=g.get("workers", 1))
    print("mode", a.mode, "sync", a.sync, "tile_mode", eng.tile_mode, "async", eng.async_n,
          "wkind", eng.wkind)
    prev = None
    for gi in g["iterations"]:
        i = gi["iteration"]
        if i > 0:
            n = eng.sync_count()
            prev = (eng.pts[:n].cpu().numpy().copy(), eng.starts.cpu().numpy().copy())
        eng.step_splat()
        if eng.reduce_hist is not None:
            eng.reduce_hist(eng.hist)
        n = eng.sync_count()
        pts = eng.pts[:n].cpu().numpy()
        starts = eng.starts.cpu().numpy()
        raw = _raw_h(eng)
        ok_raw = digest(raw)["sha256"] == gi["raw"]["sha256"]
        print(f"iter {i}: n {n} vs {gi['n_points']}, raw {'ok' if ok_raw else 'DIFF'}, "
              f"keyratio {eng.key_ratio[-1:] if eng.key_ratio else None}", flush=True)
        if not ok_raw:
            if prev is not None:
                rp, rs = O.resample(prev[0], prev[1], w.config.delta, 8)
                print("  resample vs oracle:", np.array_equal(rp, pts), np.array_equal(rs, starts))
            ref = O.accumulate_counts(pts, starts, w.bins, tr.shape, int(w.matrix.shape[0]))
            got = eng.hist.cpu().numpy()
            d = np.argwhere(got != ref)
            print("  hist vs oracle accumulate of engine points: cells differing", len(d))
            for c in d[:10]:
                print("   cell", c.tolist(), "got", got[tuple(c)], "ref", ref[tuple(c)])
            return
        eng.step_field()
    print("all iterations ok")


if __name__ == "__main__":
    main()
