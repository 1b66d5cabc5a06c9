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


def _case_workload(case):
    """Workloads of the multi-process tests (built identically in every process)."""
    from paper_1504_02687_b200.model import Graph, interaction_matrix
    from paper_1504_02687_b200.workloads import workload as wl
    if case == "exact":
        return wl(1, scale=0.5), 1
    if case in ("rep_w1", "rep_w3"):  # the golden's repulsive B=4 case
        w = wl(2, scale=0.1)
        bins = np.arange(w.graph.n_edges, dtype=np.int64) % 4
        w.graph = Graph(w.graph.positions, w.graph.sources, w.graph.targets, None, bins)
        w.bins, w.matrix = bins, interaction_matrix(4, 0.25)
        return w, int(case[-1])
    if case == "mixed_weights":
        # integer weights on the first half of the edges (rank 0's shard),
        # fractional on the rest: the plan must be the same on every rank
        w = wl(1, scale=0.5)
        n = w.graph.n_edges
        rng = np.random.default_rng(11)
        wts = rng.integers(1, 4, size=n).astype(np.float64)
        wts[n // 2:] = np.round(rng.uniform(0.3, 2.0, size=n - n // 2), 2)
        w.graph = Graph(w.graph.positions, w.graph.sources, w.graph.targets, wts, w.bins)
        return w, 1
    raise ValueError(case)


def _rank_main(rank, world, port, outdir, case="exact", env=None):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.update(env or {})
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1504_02687_b200 import bundler as Bm
        w, workers = _case_workload(case)
        res = Bm.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix, workers=workers)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), world=res.sampled_edges.world,
                 starts=res.sampled_edges.starts, field=res.density.values,
                 edge_base=res.sampled_edges.edge_base, n_edges=len(res.sampled_edges),
                 moved=np.array([m.moved_points for m in res.metrics]),
                 used=np.array([m.used_cells for m in res.metrics]),
                 disp=np.array([m.mean_displacement for m in res.metrics]))
    finally:
        dist.destroy_process_group()


def _run_ranks(tmp_path, world, case="exact", env=None):
    import torch.multiprocessing as mp
    mp.start_processes(_rank_main, args=(world, _free_port(), str(tmp_path), case, env),
                       nprocs=world, join=True, start_method="spawn")
    return [np.load(tmp_path / f"r{r}.npz") for r in range(world)]


def _compare_ranks(got_all, ref, n_edges):
    rs = ref.sampled_edges.starts
    for r, got in enumerate(got_all):
        if r == 0:  # rank 0 holds the gathered result
            assert int(got["edge_base"]) == 0
            assert np.array_equal(got["world"], ref.sampled_edges.world)
            assert np.array_equal(got["starts"], rs)
        else:       # other ranks: their own edge shard
            lo, n = int(got["edge_base"]), int(got["n_edges"])
            assert lo > 0 and lo + n <= n_edges
            assert np.array_equal(got["starts"], rs[lo:lo + n + 1] - rs[lo])
            assert np.array_equal(got["world"], ref.sampled_edges.world[rs[lo]:rs[lo + n]])
        assert np.array_equal(got["field"], ref.density.values)
        assert got["moved"].tolist() == [m.moved_points for m in ref.metrics]
        assert got["used"].tolist() == [m.used_cells for m in ref.metrics]
        np.testing.assert_allclose(got["disp"], [m.mean_displacement for m in ref.metrics],
                                   rtol=1e-9)


def test_two_processes_gloo_bundle_matches_single(tmp_path):
    got = _run_ranks(tmp_path, 2)
    w, _ = _case_workload("exact")
    ref = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)
    _compare_ranks(got, ref, w.graph.n_edges)


def test_two_processes_capacity_retry_is_collective(tmp_path):
    """No headroom for the sync-free resample: every rank overflows at a
    different iteration, agrees on the retry through the status all-reduce,
    and the result still equals one process."""
    got = _run_ranks(tmp_path, 2, env={"HB_ASYNC_CAP_FACTOR": "0.3"})
    w, _ = _case_workload("exact")
    ref = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)
    _compare_ranks(got, ref, w.graph.n_edges)


@pytest.mark.parametrize("case", ["rep_w1", "rep_w3"])
def test_three_processes_ordered_histogram_matches_reference(tmp_path, case):
    """Repulsive B=4 matrix over 3 edge shards: hit records exchanged by cell
    slab (all-to-all) and folded in the reference's order -- the final world
    points equal the reference golden made at the same `workers`."""
    got = _run_ranks(tmp_path, 3, case)
    gold = json.load(open(os.path.join(GOLDEN, f"{case}.json")))
    assert digest(got[0]["world"])["sha256"] == gold["final_world"]["sha256"]
    for g in got:
        assert digest(g["field"])["sha256"] == gold["final_field"]["sha256"]


def test_two_processes_mixed_weight_kinds(tmp_path):
    """Integer weights on one shard, fractional on the other: the weight plan
    is taken from the whole graph (ordered on both ranks), never per shard."""
    got = _run_ranks(tmp_path, 2, "mixed_weights")
    w, _ = _case_workload("mixed_weights")
    ref = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)
    _compare_ranks(got, ref, w.graph.n_edges)
