"""How many segment-key atomics would pre-aggregation over windows of
consecutive edges remove, for different edge orders?  Diagnostic only.

    python tools/dedup_probe.py [--config 4] [--iters 6]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402


def morton2(x: torch.Tensor, y: torch.Tensor, bits: int = 16) -> torch.Tensor:
    out = torch.zeros_like(x)
    for b in range(bits):
        out |= ((x >> b) & 1) << (2 * b)
        out |= ((y >> b) & 1) << (2 * b + 1)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--global-only", action="store_true")
    a = ap.parse_args()
    w = workload(a.config)
    eng, tr, _, _ = B.prepare_engine(w.graph, w.config, bins=w.bins, matrix=w.matrix)
    for _ in range(a.iters):
        eng.step()
    eng.sync_count()
    torch.cuda.synchronize()
    E = eng.n_edges
    st = eng.starts[:E + 1].long()
    if a.global_only:  # chunked (config 5 does not leave room for whole-array temporaries)
        uniq, nseg = [], 0
        chunk = 1 << 26
        for i0 in range(0, eng.n_pts - 1, chunk):
            idx = torch.arange(i0, min(i0 + chunk, eng.n_pts - 1), device=st.device)
            edge = torch.searchsorted(st, idx, right=True) - 1
            ok = (idx + 1) < st[edge + 1]
            idx, edge = idx[ok], edge[ok]
            c0 = torch.floor(eng.pts[idx] + 0.5).long()
            d = torch.floor(eng.pts[idx + 1] + 0.5).long() - c0
            nz = (d != 0).any(1)
            edge, c0, d = edge[nz], c0[nz], d[nz]
            key = ((d[:, 1] + 64) * 129 + (d[:, 0] + 64)) * (1 << 22) + c0[:, 1] * 2048 + c0[:, 0]
            if eng.nbins > 1:
                key = key + eng.groups.long()[edge] * (1 << 37)
            nseg += int(key.numel())
            uniq.append(torch.unique(key))
            del idx, edge, c0, d, key, ok, nz
        u = torch.unique(torch.cat(uniq))
        print(json.dumps({"segments": nseg, "unique_keys": int(u.numel()),
                          "ratio": round(nseg / max(1, int(u.numel())), 2)}))
        return
    pts = eng.pts[:eng.n_pts]
    n = st[1:] - st[:-1]
    cell = torch.floor(pts + 0.5).long()
    # segment j -> j+1 inside each edge
    idx = torch.arange(eng.n_pts - 1, device=pts.device)
    edge = torch.searchsorted(st, idx, right=True) - 1
    ok = (idx + 1) < st[edge + 1]
    idx, edge = idx[ok], edge[ok]
    c0, c1 = cell[idx], cell[idx + 1]
    d = c1 - c0
    nz = (d != 0).any(1)
    idx, edge, c0, d = idx[nz], edge[nz], c0[nz], d[nz]
    key = ((d[:, 1] + 64) * 129 + (d[:, 0] + 64)) * (1 << 22) + c0[:, 1] * 2048 + c0[:, 0]
    out = {"segments": int(key.numel()), "unique_keys": int(torch.unique(key).numel())}
    # edge orders
    p0 = cell[st[:-1]]
    p1 = cell[st[1:] - 1]
    ordk = {
        "original": torch.arange(E, device=pts.device),
        "morton_mid": morton2(((p0[:, 0] + p1[:, 0]) // 2).clamp(0, 65535),
                              ((p0[:, 1] + p1[:, 1]) // 2).clamp(0, 65535)),
        "morton_src_dst": morton2(morton2(p0[:, 0].clamp(0, 255), p0[:, 1].clamp(0, 255), 8),
                                  morton2(p1[:, 0].clamp(0, 255), p1[:, 1].clamp(0, 255), 8), 16),
    }
    for name, k in ordk.items():
        rank = torch.empty(E, dtype=torch.long, device=pts.device)
        rank[torch.argsort(k)] = torch.arange(E, device=pts.device)
        r = rank[edge]
        res = {}
        for win in (1, 8, 32, 128):
            wk = (r // win) * (1 << 40) + key  # key < 2^40
            res[win] = round(int(key.numel()) / int(torch.unique(wk).numel()), 2)
        out[name] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()
