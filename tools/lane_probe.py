"""Would a lane-per-edge advect share gradient-record sectors?  For the
bundled state of a config (after --iters iterations, edges in the given
order), count the distinct 32-byte sectors of the 48-byte quad records that
one warp-wide gather touches, per point, under two lane mappings:
  flat : lane = one of 32 consecutive points of the packed stream (today)
  edge : lane = one of 32 consecutive edges, all at the same point index j
Diagnostic only.

    python tools/lane_probe.py [--config 4] [--iters 6] [--order none|srcdst|mid]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200.model import Graph  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--order", default="none", choices=["none", "srcdst", "mid"])
a = ap.parse_args()
w = workload(a.config)
g = w.graph
if a.order != "none":
    ps, pt = g.positions[g.sources], g.positions[g.targets]

    def q(v, bits):
        return np.clip((v * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)

    def inter(cols, bits):
        key = np.zeros(len(cols[0]), dtype=np.int64)
        for b in range(bits):
            for c, col in enumerate(cols):
                key |= ((col >> b) & 1) << (b * len(cols) + c)
        return key

    if a.order == "srcdst":
        key = inter([q(ps[:, 0], 8), q(ps[:, 1], 8), q(pt[:, 0], 8), q(pt[:, 1], 8)], 8)
    else:
        mid = 0.5 * (ps + pt)
        key = inter([q(mid[:, 0], 16), q(mid[:, 1], 16)], 16)
    order = np.argsort(key, kind="stable")
    w = type(w)(**{**w.__dict__, "graph": Graph(g.positions, g.sources[order], g.targets[order]),
                   "bins": np.asarray(w.bins)[order]})
eng, tr, _, _ = B.prepare_engine(w.graph, w.config, bins=w.bins, matrix=w.matrix)
for _ in range(a.iters):
    eng.step()
n = eng.sync_count()
torch.cuda.synchronize()
E = eng.n_edges
st = eng.starts[:E + 1].long()
pts = eng.pts[:n]
u = torch.clamp(torch.floor(pts[:, 0]).long(), 0, eng.nu - 2)
v = torch.clamp(torch.floor(pts[:, 1]).long(), 0, eng.nv - 2)
rec = v * eng.nu + u
s0 = (rec * 48) // 32  # the record's two sectors: s0, s0 + 1
idx = torch.arange(n, device=pts.device)
edge = torch.searchsorted(st, idx, right=True) - 1
j = idx - st[edge]
lens = st[1:] - st[:-1]
interior = (j > 0) & (j < lens[edge] - 1)
res = {"points": int(interior.sum().item())}

def distinct(group_key):
    # distinct (group, sector) pairs over the interior points, both sectors
    gk = group_key[interior]
    sec = s0[interior]
    keys = torch.cat([gk * (1 << 32) + sec, gk * (1 << 32) + sec + 1])
    return int(torch.unique(keys).numel())

flat_grp = idx // 32
res["flat_sectors_per_point"] = round(distinct(flat_grp) / res["points"], 3)
maxj = int(lens.max().item())
edge_grp = (edge // 32) * maxj + j
res["edge_sectors_per_point"] = round(distinct(edge_grp) / res["points"], 3)
# lane occupancy of the edge mapping: points / (warps * max length per warp)
wl = torch.zeros((E + 31) // 32, dtype=torch.long, device=pts.device)
wl.scatter_reduce_(0, torch.arange(E, device=pts.device) // 32, lens, reduce="amax")
res["edge_lane_occupancy"] = round(n / (32 * int(wl.sum().item())), 3)
res.update({"config": w.name, "order": a.order, "iters": a.iters})
print(json.dumps(res))
