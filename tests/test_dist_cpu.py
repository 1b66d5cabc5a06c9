"""Multi-rank plumbing on CPU: world_size 2 over gloo (127.0.0.1).

Covers the pieces the NCCL run uses: edge sharding, the int32 histogram
all-reduce (checked against the oracle's single-process histogram: integer
sums are associative, so the sharded sum is bit-exact), metric sums and the
polyline gather/rebase."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_1504_02687_b200 import dist as D
        from paper_1504_02687_b200.engine import sample_counts
        from paper_1504_02687_b200.model import make_transform
        from paper_1504_02687_b200.workloads import workload

        w = workload(2, scale=0.05)
        g, cfg = w.graph, w.config
        tr = make_transform(g.positions, cfg.grid_size, cfg.padding_cells)
        src = tr.world_to_grid(g.positions[g.sources])
        dst = tr.world_to_grid(g.positions[g.targets])
        counts = sample_counts(src, dst, cfg.delta)
        assert D.rank_world() == (rank, world)
        lo, hi = D.shard_edges(counts, world)[rank]
        pts, starts, _, _ = O.sample(g.positions, g.sources[lo:hi], g.targets[lo:hi],
                                     tr.origin, tr.cell_size, cfg.delta)
        hist = O.accumulate_counts(pts, starts, w.bins[lo:hi], tr.shape, 1)
        t = torch.from_numpy(hist)
        D.all_reduce_sum(t)
        moved, disp = D.sum_host_arrays([np.array([rank + 1], dtype=np.int64),
                                         np.array([0.5 * (rank + 1)])])
        got = D.gather_polylines(torch.from_numpy(pts), torch.from_numpy(starts))
        # the status / span agreement used by the engine: max over ranks
        mx = D.all_reduce_max(torch.tensor([float(rank), -float(rank), 4.0 * (rank == 1)],
                                           dtype=torch.float64))
        wp, ws = got if got is not None else (np.zeros((0, 2)), np.zeros(0, np.int64))
        np.savez(os.path.join(outdir, f"r{rank}.npz"), hist=t.numpy(), moved=moved, disp=disp,
                 wp=wp, ws=ws, lo=lo, hi=hi, gathered=got is not None, mx=mx.numpy())
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_histogram_and_gather(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    import oracle as O
    from paper_1504_02687_b200.model import make_transform
    from paper_1504_02687_b200.workloads import workload
    w = workload(2, scale=0.05)
    g, cfg = w.graph, w.config
    tr = make_transform(g.positions, cfg.grid_size, cfg.padding_cells)
    pts, starts, _, _ = O.sample(g.positions, g.sources, g.targets, tr.origin, tr.cell_size,
                                 cfg.delta)
    full = O.accumulate_counts(pts, starts, w.bins, tr.shape, 1)
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(world)]
    for k in range(world):
        assert np.array_equal(r[k]["hist"], full)          # bit-exact global histogram
        assert int(r[k]["moved"][0]) == 3 and float(r[k]["disp"][0]) == 1.5
        assert list(r[k]["mx"]) == [1.0, 0.0, 4.0]
    # polylines gathered to rank 0 only, in edge order
    assert bool(r[0]["gathered"]) and not bool(r[1]["gathered"])
    assert np.array_equal(r[0]["wp"], pts)
    assert np.array_equal(r[0]["ws"], starts)
    assert r[0]["hi"] == r[1]["lo"] and r[1]["hi"] == g.n_edges


def _exchange_worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1504_02687_b200 import dist as D
        # rank r sends (r, dest) tagged rows: dest d gets d + 1 rows from every rank
        rows = [np.array([[rank, d]] * (d + 1), dtype=np.int32) for d in range(world)]
        send = torch.from_numpy(np.concatenate(rows))
        recv = D.all_to_all_var(send, [d + 1 for d in range(world)])
        # column blocks of unequal width, gathered in rank order
        block = torch.full((2, rank + 1), float(rank))
        cols = D.all_gather_columns(block, [r + 1 for r in range(world)])
        np.savez(os.path.join(outdir, f"x{rank}.npz"), recv=recv.numpy(), cols=cols.numpy())
    finally:
        dist.destroy_process_group()


def test_exchange_helpers_gloo(tmp_path):
    """The ordered path's record exchange (variable all-to-all, sender-rank
    order) and slab all-gather over gloo, world size 3."""
    world = 3
    mp.start_processes(_exchange_worker, args=(world, _free_port(), str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    for r in range(world):
        x = np.load(tmp_path / f"x{r}.npz")
        want = np.concatenate([np.array([[s, r]] * (r + 1), dtype=np.int32)
                               for s in range(world)])
        assert np.array_equal(x["recv"], want)
        cols = x["cols"]
        assert cols.shape == (2, 6)
        assert cols[0].tolist() == [0, 1, 1, 2, 2, 2]
