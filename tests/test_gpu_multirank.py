"""Multi-rank bundling on one GPU.

* shard emulation: two BundleEngines over the two halves of the edge list
  (dist.shard_edges), histograms summed between the splat and field halves
  of every iteration -- exactly what the NCCL all-reduce does across GPUs.
  Must be bit-identical to one engine (integer sums are associative).
* two real processes (gloo backend, both on cuda:0) through the public
  bundle(): sharding, histogram all-reduce, metric sums, polyline gather.
"""

from __future__ import annotations

import json
import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from hb_hash import digest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200.dist import shard_edges  # noqa: E402
from paper_1504_02687_b200.engine import BundleEngine, sample_counts, weight_plan  # noqa: E402
from paper_1504_02687_b200.model import make_transform  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402


def _emulated(w, shards):
    g, cfg = w.graph, w.config
    tr = make_transform(g.positions, cfg.grid_size, cfg.padding_cells)
    src = tr.world_to_grid(g.positions[g.sources])
    dst = tr.world_to_grid(g.positions[g.targets])
    parts = shard_edges(sample_counts(src, dst, cfg.delta), shards)
    engs = [BundleEngine(np.ascontiguousarray(src[lo:hi]), np.ascontiguousarray(dst[lo:hi]),
                         w.bins[lo:hi], weight_plan(g.weights, w.matrix).slice(lo, hi), w.matrix, tr.shape, cfg)
            for lo, hi in parts]
    for _ in range(cfg.iterations):
        for e in engs:
            e.step_splat()
        total = engs[0].hist.clone()
        for e in engs[1:]:
            total += e.hist
        for e in engs:
            e.hist.copy_(total)
            e.step_field()
    recs = [e.finish_metrics() for e in engs]
    pts = np.concatenate([e.packed_points()[0].cpu().numpy() for e in engs])
    starts, base = [np.zeros(1, dtype=np.int64)], 0
    for e in engs:
        st = e.starts.cpu().numpy()
        starts.append(st[1:] + base)
        base += int(st[-1])
    return engs, recs, pts, np.concatenate(starts)


@pytest.mark.parametrize("k,scale,shards", [(1, 1.0, 2), (3, 0.02, 3)])
def test_shard_emulation_bit_exact(k, scale, shards):
    w = workload(k, scale=scale)
    engs, recs, pts, starts = _emulated(w, shards)
    ref, _, metrics = B.bundle_packed(w.graph, w.config, bins=w.bins, matrix=w.matrix)
    rp, rs = ref.packed_points()
    assert np.array_equal(pts, rp.cpu().numpy())
    assert np.array_equal(starts, rs.cpu().numpy())
    for e in engs:
        assert torch.equal(e.field, ref.field)
    moved = [sum(r[i].moved_points for r in recs) for i in range(w.config.iterations)]
    assert moved == [m.moved_points for m in metrics]
    if k == 1:
        gold = json.load(open(os.path.join(GOLDEN, "cfg1.json")))
        assert digest(pts)["sha256"] == gold["final_pts"]["sha256"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1504_02687_b200 import bundler as Bm
        from paper_1504_02687_b200.workloads import workload as wl
        w = wl(1, scale=0.5)
        res = Bm.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), world=res.sampled_edges.world,
                 starts=res.sampled_edges.starts, field=res.density.values,
                 edge_base=res.sampled_edges.edge_base, n_edges=len(res.sampled_edges),
                 moved=np.array([m.moved_points for m in res.metrics]),
                 used=np.array([m.used_cells for m in res.metrics]),
                 disp=np.array([m.mean_displacement for m in res.metrics]))
    finally:
        dist.destroy_process_group()


def test_two_processes_gloo_bundle_matches_single(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.start_processes(_rank_main, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    w = workload(1, scale=0.5)
    ref = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)
    rs = ref.sampled_edges.starts
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npz")
        if r == 0:  # rank 0 holds the gathered result
            assert int(got["edge_base"]) == 0
            assert np.array_equal(got["world"], ref.sampled_edges.world)
            assert np.array_equal(got["starts"], rs)
        else:       # other ranks: their own edge shard
            lo, n = int(got["edge_base"]), int(got["n_edges"])
            assert lo > 0 and lo + n == w.graph.n_edges
            assert np.array_equal(got["starts"], rs[lo:lo + n + 1] - rs[lo])
            assert np.array_equal(got["world"], ref.sampled_edges.world[rs[lo]:rs[lo + n]])
        assert np.array_equal(got["field"], ref.density.values)
        assert got["moved"].tolist() == [m.moved_points for m in ref.metrics]
        assert got["used"].tolist() == [m.used_cells for m in ref.metrics]
        np.testing.assert_allclose(got["disp"], [m.mean_displacement for m in ref.metrics],
                                   rtol=1e-9)
