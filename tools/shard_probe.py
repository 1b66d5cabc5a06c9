"""Per-rank work of the N-GPU edge sharding, emulated on one GPU.

    python tools/shard_probe.py [--config 4] [--shards 1,2,4,8]

For each N, builds the N shard engines of bench.py's multi-rank path
(dist.shard_edges over the initial point counts), runs the iterations with
the histograms summed between the splat and field halves (what the NCCL
all-reduce does), and times every engine's own kernels with CUDA events.
Engines run one after another, so each kernel has the GPU to itself, as it
would on its own B200.  Reports per N the predicted step time
sum_i max_rank(t_rank,i) (the all-reduce excluded), the implied strong-scaling
efficiency against N = 1, and the per-rank spread.  Diagnostic only: the
driver's SCALE run on 8 GPUs is the measurement.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1504_02687_b200.dist import shard_edges  # noqa: E402
from paper_1504_02687_b200.engine import BundleEngine, sample_counts, weight_plan  # noqa: E402
from paper_1504_02687_b200.model import make_transform  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402


def run(w, shards):
    g, cfg = w.graph, w.config
    tr = make_transform(g.positions, cfg.grid_size, cfg.padding_cells)
    src = tr.world_to_grid(g.positions[g.sources])
    dst = tr.world_to_grid(g.positions[g.targets])
    parts = shard_edges(sample_counts(src, dst, cfg.delta), shards)
    engs = [BundleEngine(np.ascontiguousarray(src[lo:hi]), np.ascontiguousarray(dst[lo:hi]),
                         w.bins[lo:hi], weight_plan(g.weights, w.matrix).slice(lo, hi), w.matrix, tr.shape, cfg)
            for lo, hi in parts]
    for e in engs:
        e.keep_initial_state()
    times = np.zeros((cfg.iterations, shards))
    pts = 0
    for rep in range(2):  # warm, then timed
        for e in engs:
            e.reset()
        engs[0].trace = {} if rep == 1 else None
        for i in range(cfg.iterations):
            ev = []
            for e in engs:
                a = torch.cuda.Event(enable_timing=True)
                a.record()
                e.step_splat()
                b = torch.cuda.Event(enable_timing=True)
                b.record()
                ev.append([a, b])
            total = engs[0].hist.clone()
            for e in engs[1:]:
                total += e.hist
            for k, e in enumerate(engs):
                e.hist.copy_(total)
                a = torch.cuda.Event(enable_timing=True)
                a.record()
                e.step_field()
                b = torch.cuda.Event(enable_timing=True)
                b.record()
                ev[k] += [a, b]
            torch.cuda.synchronize()
            for k, (a, b, c, d) in enumerate(ev):
                times[i, k] = a.elapsed_time(b) + c.elapsed_time(d)
        if rep == 1:
            pts = sum(r.n_points for e in engs for r in e.finish_metrics())
    kern = {}
    for name, evs in (engs[0].trace or {}).items():
        kern[name] = round(sum(a.elapsed_time(b) for a, b, _ in evs) / cfg.iterations, 4)
    engs[0].trace = None
    print(json.dumps({"shards": shards, "rank0_ms_per_iteration": kern}), file=sys.stderr)
    step = float(times.max(axis=1).sum())
    per_rank = times.sum(axis=0)
    del engs
    torch.cuda.empty_cache()
    return step, per_rank, pts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--shards", default="1,2,4,8")
    a = ap.parse_args()
    w = workload(a.config)
    out = {"workload": w.name, "note": __doc__.split("\n\n")[1].replace("\n", " ")}
    base = None
    for n in (int(s) for s in a.shards.split(",")):
        step, per_rank, pts = run(w, n)
        base = base or step
        out[f"n{n}"] = {"pred_ms_per_step": round(step, 2),
                        "pred_points_per_s": pts / (step / 1e3),
                        "pred_efficiency": round(base / (n * step), 3),
                        "rank_ms_min_max": [round(float(per_rank.min()), 2),
                                            round(float(per_rank.max()), 2)]}
        print(json.dumps({n: out[f"n{n}"]}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
