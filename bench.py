#!/usr/bin/env python
"""Benchmark of the B200 bundling iteration (BASELINE.json metric:
sample-point updates/s = sum_i N_i / T, and ms per bundling iteration).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4]
    python bench.py --impl reference ...        # the CPU reference arm
    python bench.py --dist ...                  # collective path at N=1 (1-rank NCCL)

A *step* bundles the whole synthetic graph from its straight initial
polylines through all ``config.iterations`` iterations (the reference's
timed loop, bundler.py:351-376): the step first restores the sampled points
(device copy), then runs every iteration. Inputs are device-resident when
the timed region starts; the ~2 GB point arrays of config 4 exceed the
126 MB L2, so no L2 flush is needed between steps.

N > 1: one process per GPU over NCCL -- under torchrun, or launched by this
script itself when ``--gpus N`` is given without torchrun.  Edges are
sharded by initial point count, the int32 histogram is all-reduced every
iteration, the same total work is split over N GPUs ("strong" scaling),
time = max over ranks.

``--impl reference`` times the reference's CPU path (the oracle port of the
numba kernels, every host thread) on the same workload and the same
``config`` object, one step = the whole loop; under torchrun only rank 0
runs it.

Extra keys: ``e2e`` (same metric through the public ``bundle()`` with host
numpy inputs and the world-coordinate polylines copied back every step),
``roofline`` (dominant kernel, CUDA events over the timed region),
``cpu_baseline`` (the oracle port on this host's cores, bounded sample),
``clocks`` (nvidia-smi sampled during the timed region), ``gpu_launches``
(kernels our library launched inside the timed region, hb_launch_count),
``run`` (how it ran: backend, histogram path, splat path).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1,
                    help="GPUs (ranks); without torchrun the script launches N ranks itself")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--scale", type=float, default=1.0,
                    help="shrink node/edge counts (debug only; not a bench number)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-iterations", type=int, default=2,
                    help="iterations of the workload timed for our line's cpu_baseline")
    ap.add_argument("--ref-iterations", type=int, default=None,
                    help="--impl reference: iterations per step (default: all of the "
                         "workload's, i.e. the same work as our arm)")
    ap.add_argument("--dist", action="store_true",
                    help="run the collective path even at N=1 (1-rank NCCL group: the "
                         "histogram all-reduce, status agreement and gather execute)")
    return ap.parse_args()


def launch_ranks(n: int) -> int:
    """`--gpus N` without torchrun: run this script under
    torch.distributed.run with N ranks (one per GPU) and return its exit
    code (rank 0 prints the JSON line)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def measured_peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        for line in out.splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# algorithmic bytes, per launch


def algorithmic_bytes(name: str, n_prev: int, n_cur: int, n_edges: int, cells: int,
                      passes: int, nbins: int) -> int:
    if name == "hb_advect_points":      # advect: read + write every point
        return 32 * n_cur + 8 * n_edges + 4 * cells
    if name == "hb_laplacian_count":    # Laplacian + next resample count (pos codes)
        return 32 * n_cur + 4 * n_cur + 16 * n_edges
    if name == "hb_advect_laplacian":   # Laplacian (+ fused next resample count)
        return 32 * n_cur + 16 * n_edges + 4 * cells
    if name in ("hb_resample_emit", "hb_resample_emit_cap"):  # resample emit + fused splat
        return 16 * n_prev + 16 * n_cur + 40 * n_edges + 4 * cells
    if name == "hb_exact_check":
        return 4 * cells
    if name == "hb_accumulate_ordered":  # hits -> sort -> fold (ordered path)
        return 16 * n_cur + 16 * n_edges + 4 * cells
    if name == "hb_resample_count":
        return 16 * n_prev + 8 * n_edges
    if name == "hb_splat":
        return 16 * n_cur + 16 * n_edges + 4 * cells
    if name == "hb_smooth":
        return 4 * cells + 8 * cells * passes + (8 * cells if nbins > 1 else 0)
    if name == "hb_used_cells":
        return 4 * cells
    return 0


def roofline_from_trace(trace, records, eng, peak, peak_src):
    cells = eng.nbins * eng.nv * eng.nu
    passes = int(eng.radii.numel())
    per = {}
    for name, evs in trace.items():
        tot_ms, tot_b = 0.0, 0
        for a, b, it in evs:
            tot_ms += a.elapsed_time(b)
            n_cur = records[it].n_points
            n_prev = records[it - 1].n_points if it > 0 else n_cur
            tot_b += algorithmic_bytes(name, n_prev, n_cur, eng.n_edges, cells, passes,
                                       eng.nbins)
        per[name] = {"launches": len(evs), "ms_total": tot_ms, "bytes_total": tot_b}
    dom = max(per, key=lambda k: per[k]["ms_total"])
    d = per[dom]
    achieved = d["bytes_total"] / (d["ms_total"] / 1e3) / 1e9 if d["ms_total"] else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            t = json.load(f).get(dom)
        if t and "bytes_per_point" in t:
            mean_n = statistics.mean(r.n_points for r in records)
            traffic = float(t["bytes_per_point"]) * mean_n
    total_ms = sum(v["ms_total"] for v in per.values())
    # the measured limit of the dominant kernel when it is not HBM (ncu --set full)
    ceiling = None
    cpath = os.path.join(ROOT, "profiles", "r02_ncu_full_summary.json")
    if os.path.exists(cpath):
        with open(cpath) as f:
            c = json.load(f).get(dom)
        if c and "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed" in c:
            pct = float(c["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]
                        .split()[0])
            sect = float(c["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"].split()[0])
            ceiling = {"bound": "l1tex data pipe (gathers)", "frac_of_ceiling": round(pct / 100, 4),
                       "global_load_sectors_per_point": round(sect / c["points"], 2),
                       "source": "profiles/r02_ncu_full_summary.json (" + c["capture"] + ")"}
    return {
        "kernel": dom, "bound": "hbm", "achieved": round(achieved, 1),
        "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
        "traffic": traffic, "peak_source": peak_src, "ceiling": ceiling,
        "avg_launch_ms": d["ms_total"] / max(d["launches"], 1),
        "share_of_kernel_time": round(d["ms_total"] / total_ms, 4) if total_ms else None,
        "per_kernel": {k: {"launches": v["launches"],
                           "avg_ms": round(v["ms_total"] / max(v["launches"], 1), 4),
                           "share": round(v["ms_total"] / total_ms, 4) if total_ms else None,
                           "GBps": round(v["bytes_total"] / (v["ms_total"] / 1e3) / 1e9, 1)
                           if v["ms_total"] else None}
                       for k, v in sorted(per.items(), key=lambda kv: -kv[1]["ms_total"])},
    }


# ---------------------------------------------------------------------------
# CPU reference (oracle port, all host threads) on a bounded sample


def cpu_reference_sample(w, iterations: int, workers: int):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    g = w.graph
    t0 = time.perf_counter()
    run = O.bundle_packed(g.positions, g.sources, g.targets, g.weights, w.bins, w.config,
                          w.matrix, workers=workers, max_iterations=iterations)
    wall = time.perf_counter() - t0
    pts = sum(m.n_points for m in run.metrics)
    return pts / run.bundling_seconds, run, wall


def workload_config(w, grid, points_per_step: int) -> dict:
    """The ``config`` object both arms print: what the workload IS (graph,
    grid, parameters and the sum of N_i per step -- identical in both arms,
    the results being bit-identical), nothing about how it was run."""
    cfg = w.config
    return {"workload": w.name, "edges": int(w.graph.n_edges), "grid": [int(x) for x in grid],
            "iterations": int(cfg.iterations), "points_per_step": int(points_per_step),
            "delta": cfg.delta, "sigma": cfg.sigma, "lambda": cfg.lambda_,
            "l2": "inputs > L2 (point arrays >> 126 MB), no flush"}


def run_reference_arm(args, rank, world):
    """--impl reference: rank 0 times the reference's CPU path -- the oracle
    port (oracle/hb_oracle.c, the numba kernels restated in C, driven like
    _parallel.py on every host thread) -- on the same workload, metric and
    config as our arm: one step = the whole bundling loop, all iterations
    (sampling excluded, like the reference's own timer).  Warm-up steps run
    one iteration each (the C port has no JIT or cache to warm)."""
    if rank != 0:
        return
    from paper_1504_02687_b200.workloads import workload
    w = workload(args.config, scale=args.scale)
    cores = host_cores()
    iters = args.ref_iterations or w.config.iterations
    for _ in range(args.warmup):
        cpu_reference_sample(w, 1, cores)
    vals, secs = [], []
    for _ in range(args.steps):
        v, run, _ = cpu_reference_sample(w, iters, cores)
        vals.append(v)
        secs.append(run.bundling_seconds)
    n_pts = sum(m.n_points for m in run.metrics)
    value = n_pts * len(secs) / sum(secs)
    sample = (f"{w.name}: iterations 0-{iters - 1} of {w.config.iterations}, all "
              f"{w.graph.n_edges} edges, {n_pts} point updates per step, oracle port "
              f"(oracle/hb_oracle.c) on {cores} threads")
    line = {
        "impl": "reference", "metric": "sample-point updates/sec", "value": value,
        "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(secs), "higher_is_better": True,
        "ms_per_iteration": 1e3 * statistics.mean(secs) / iters,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(w, (int(w.matrix.shape[0]), *map(int, run.field.shape[1:])),
                                  n_pts),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


def main():
    args = parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_1504_02687_b200 import _native as N
    from paper_1504_02687_b200 import bundler as B
    from paper_1504_02687_b200.engine import IO_BYTES
    from paper_1504_02687_b200.workloads import workload

    # HB_BENCH_ONE_DEVICE=1 / HB_DIST_BACKEND=gloo: test-only switches that
    # let the multi-rank code path run with every rank on cuda:0 (NCCL
    # refuses two ranks on one GPU).  Bench numbers always use NCCL.
    device_index = 0 if os.environ.get("HB_BENCH_ONE_DEVICE") == "1" else local
    torch.cuda.set_device(device_index)
    group = None
    if world > 1 or args.dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if world == 1:  # --dist at N=1: a 1-rank group, collective path forced
            os.environ.setdefault("MASTER_PORT", "29531")
            os.environ.setdefault("RANK", "0")
            os.environ["HB_FORCE_DIST"] = "1"
        backend = os.environ.get("HB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device_index),
                                    world_size=world, rank=rank)
        else:
            dist.init_process_group(backend, world_size=world, rank=rank)
    dist_on = dist.is_available() and dist.is_initialized()
    backend_name = dist.get_backend() if dist_on else None

    def barrier():
        if dist_on:
            dist.barrier()

    def coll_device():
        return "cuda" if dist.get_backend() == "nccl" else "cpu"

    def max_over_ranks(x: float) -> float:
        if not dist_on:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_device())
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: int) -> int:
        if not dist_on:
            return x
        t = torch.tensor([x], dtype=torch.int64, device=coll_device())
        dist.all_reduce(t)
        return int(t.item())

    w = workload(args.config, scale=args.scale)
    cfg = w.config
    eng, tr, lo, hi = B.prepare_engine(w.graph, cfg, bins=w.bins, matrix=w.matrix, group=group)
    eng.keep_initial_state()

    def one_step():
        eng.reset()
        return eng.run()

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local) if rank == 0 else None
    eng.trace = {}
    launches0 = N.lib().hb_launch_count()
    barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record()
    pts_local = 0
    for _ in range(args.steps):
        recs = one_step()
        pts_local += sum(r.n_points for r in recs)
    t_end.record()
    torch.cuda.synchronize()
    barrier()
    launches = N.lib().hb_launch_count() - launches0
    elapsed = max_over_ranks(t_start.elapsed_time(t_end) / 1e3)
    clk = clocks.stop() if clocks else None
    total_pts = sum_over_ranks(pts_local)
    value = total_pts / elapsed
    ms_step = 1e3 * elapsed / args.steps
    peak, peak_src = measured_peak_hbm()
    # roofline of the dominant kernel over every launch of the timed region
    # (steps are identical, so the last step's records size every launch)
    n_it = cfg.iterations
    roof = roofline_from_trace(eng.trace, eng.records, eng, peak, peak_src)
    eng.trace = None
    pts_per_step = pts_local // args.steps

    # end to end through the public API (host numpy in, host numpy out)
    e2e = None
    if not args.no_e2e:
        k_e2e = args.e2e_steps or args.steps
        for _ in range(2):  # warm: allocator pools, pinned result block
            res = B.bundle(w.graph, cfg, bins=w.bins, matrix=w.matrix, group=group)
            del res
        torch.cuda.synchronize()
        IO_BYTES["h2d"] = IO_BYTES["d2h"] = 0
        barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            res = B.bundle(w.graph, cfg, bins=w.bins, matrix=w.matrix, group=group)
            assert res.sampled_edges.world.shape[0] == int(res.sampled_edges.starts[-1])
            del res  # a caller that consumed the result; its pinned block is reused
        torch.cuda.synchronize()
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": total_pts / args.steps * k_e2e / e2e_s, "unit": "points/s",
               "h2d_bytes_per_step": IO_BYTES["h2d"] // k_e2e,
               "d2h_bytes_per_step": IO_BYTES["d2h"] // k_e2e,
               "steps": k_e2e, "s_per_step": e2e_s / k_e2e,
               "note": "bundle(graph, config) with host numpy graph arrays; timed region "
                       "includes host transform/sampling, H2D, all iterations, device "
                       "grid->world + endpoint pinning and D2H of the packed polylines"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        v, run, _ = cpu_reference_sample(w, args.cpu_iterations, cores)
        n_pts = sum(m.n_points for m in run.metrics)
        cpu = {"value": v, "unit": "points/s", "cores": cores, "kind": "port",
               "sample": f"{w.name}: iterations 0-{args.cpu_iterations - 1} of "
                         f"{cfg.iterations}, all {w.graph.n_edges} edges, {n_pts} point "
                         f"updates, oracle port (oracle/hb_oracle.c) on {cores} threads"}

    if rank == 0:
        par = f"edge-shard x{world}"
        if dist_on:
            par += f" + {backend_name} int32 histogram allreduce"
        line = {
            "metric": "sample-point updates/sec", "value": value, "unit": "points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "ms_per_iteration": ms_step / n_it,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config(w, (eng.nbins, eng.nv, eng.nu), total_pts // args.steps),
            "run": {"parallelism": par, "backend": backend_name,
                    "histogram_path": eng.wkind,
                    "splat": {1: "segment-key table", 0: "tile records",
                              -1: "direct"}[eng.tile_mode],
                    "segment_key_ratio": [round(x, 4) for x in eng.key_ratio]},
            "roofline": roof, "cpu_baseline": cpu, "clocks": clk, "e2e": e2e,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
