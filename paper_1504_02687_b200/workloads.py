"""Seeded synthetic graphs standing in for BASELINE.json's five configs.

The reference publishes no datasets for this path; these
generators produce graphs with the shapes, sizes and distributions that
BASELINE.json describes. Every generator is a pure function of its seed, and
self-loops / coincident endpoints are dropped because the reference's
``Graph`` rejects them (``model.py:132-134``).

``workload(k)`` returns ``(graph, config, bins, matrix)`` ready for
``bundle(graph, config, bins=bins, matrix=matrix)``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .model import BundleConfig, Graph, interaction_matrix, make_transform

__all__ = ["Workload", "workload", "uniform_graph", "mixture_graph",
           "powerlaw_mixture_graph", "stress_graph", "mean_edge_cells",
           "random_graph", "table1_workload", "WORKLOAD_NAMES"]

WORKLOAD_NAMES = {
    1: "cfg1-uniform-2k-256",
    2: "cfg2-gmm12-50k-512",
    3: "cfg3-gmm12-500k-8x512",
    4: "cfg4-powerlaw-2m-1024",
    5: "cfg5-stress-20m-4x2048",
}


def random_graph(n_edges: int, samples_per_edge: float = 24.0, delta: float = 3.0,
                 grid_size: int = 800, padding_cells: int = 41, seed: int = 0,
                 world: float = 1000.0) -> Graph:
    """The reference's scalability graph (``cli.py:142-163``, the paper's
    Table 1 "random" row): uniform sources in a ``world`` square, targets at
    a uniform angle and a length ~U(0.5, 1.5) x the mean that gives about
    ``samples_per_edge`` initial samples, clipped to the square.  The same
    seeded numpy draws in the same order, so the arrays equal the
    reference's (tests/golden/make_golden_r2.py checks the digests)."""
    rng = np.random.default_rng(seed)
    cell = world / (grid_size - 2 * padding_cells - 1)
    mean_len = max(samples_per_edge - 1.5, 0.7) * delta * cell
    src = rng.uniform(0.0, world, size=(n_edges, 2))
    angle = rng.uniform(0.0, 2.0 * math.pi, size=n_edges)
    length = rng.uniform(0.5, 1.5, size=n_edges) * mean_len
    dst = src + np.stack([np.cos(angle), np.sin(angle)], axis=1) * length[:, None]
    np.clip(dst, 0.0, world, out=dst)
    positions = np.concatenate([src, dst], axis=0)
    return Graph(positions, np.arange(n_edges, dtype=np.int64),
                 np.arange(n_edges, 2 * n_edges, dtype=np.int64))


def table1_workload(n_edges: int = 200_000, nbins: int = 1, seed: int = 0,
                    iterations: int = 10) -> Workload:
    """``cli.bench`` (``cli.py:166-192``) for one (size, B) pair: default
    BundleConfig, bins = arange % B, ``interaction_matrix(B, alpha)`` -- the
    reference's repulsive model, non-dyadic for B = 4 / 16."""
    cfg = BundleConfig(iterations=iterations, random_seed=seed)
    g = random_graph(n_edges, 24.0, cfg.delta, cfg.grid_size, cfg.padding_cells, seed)
    bins = np.arange(n_edges, dtype=np.int64) % nbins
    mat = interaction_matrix(nbins, cfg.alpha)
    g = Graph(g.positions, g.sources, g.targets, None, bins)
    return Workload(f"table1-random-{n_edges // 1000}k-b{nbins}", g, cfg, bins, mat)


@dataclass
class Workload:
    name: str
    graph: Graph
    config: BundleConfig
    bins: np.ndarray
    matrix: np.ndarray


def _drop_degenerate(pos, s, t):
    keep = (s != t)
    keep &= ~np.all(pos[s] == pos[t], axis=1)
    return s[keep], t[keep]


def uniform_graph(n_nodes: int, n_edges: int, seed: int = 0):
    """Config 1: uniform nodes, uniform endpoints with t != s."""
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0.0, 1.0, size=(n_nodes, 2))
    s = rng.integers(0, n_nodes, size=n_edges)
    t = (s + 1 + rng.integers(0, n_nodes - 1, size=n_edges)) % n_nodes
    s, t = _drop_degenerate(pos, s, t)
    return Graph(pos, s, t)


def _gmm_nodes(rng, n_nodes, n_comp, sd):
    centres = rng.uniform(0.1, 0.9, size=(n_comp, 2))
    comp = rng.integers(0, n_comp, size=n_nodes)
    pos = centres[comp] + sd * rng.standard_normal((n_nodes, 2))
    np.clip(pos, 0.0, 1.0, out=pos)
    return centres, comp, pos


def _pair_probs(centres, scale):
    d = np.linalg.norm(centres[:, None, :] - centres[None, :, :], axis=2)
    p = np.exp(-d / scale)
    return (p / p.sum()).ravel()


def _pick_in_component(rng, members, member_cdf, comp_of_edge):
    """Pick one node per edge inside the edge's component.

    ``members[c]`` lists node ids of component c and ``member_cdf[c]`` their
    cumulative (normalised) weights; uniform weights when cdf is None.
    """
    out = np.empty(comp_of_edge.shape[0], dtype=np.int64)
    order = np.argsort(comp_of_edge, kind="stable")
    sorted_comp = comp_of_edge[order]
    bounds = np.searchsorted(sorted_comp, np.arange(len(members) + 1))
    for c in range(len(members)):
        lo, hi = bounds[c], bounds[c + 1]
        if lo == hi:
            continue
        idx = order[lo:hi]
        mem = members[c]
        if member_cdf is None:
            out[idx] = mem[rng.integers(0, mem.shape[0], size=hi - lo)]
        else:
            u = rng.uniform(0.0, 1.0, size=hi - lo)
            k = np.minimum(np.searchsorted(member_cdf[c], u, side="right"),
                           mem.shape[0] - 1)
            out[idx] = mem[k]
    return out


def mixture_graph(n_nodes: int, n_edges: int, n_comp: int = 12,
                  sd: float = 0.05, scale: float = 0.3, seed: int = 0):
    """Configs 2/3: GMM nodes; component pair of an edge ~ exp(-d/scale)."""
    rng = np.random.default_rng(seed)
    centres, comp, pos = _gmm_nodes(rng, n_nodes, n_comp, sd)
    members = [np.flatnonzero(comp == c) for c in range(n_comp)]
    occupied = np.array([m.size > 0 for m in members])
    probs = _pair_probs(centres, scale).reshape(n_comp, n_comp)
    probs *= occupied[:, None] & occupied[None, :]
    probs = (probs / probs.sum()).ravel()
    pair = rng.choice(n_comp * n_comp, size=n_edges, p=probs)
    cs, ct = pair // n_comp, pair % n_comp
    s = _pick_in_component(rng, members, None, cs)
    t = _pick_in_component(rng, members, None, ct)
    s, t = _drop_degenerate(pos, s, t)
    return Graph(pos, s, t)


def powerlaw_mixture_graph(n_nodes: int, n_edges: int, n_comp: int = 64,
                           sd: float = 0.05, gamma: float = 2.1,
                           scale: float = 0.3, seed: int = 0):
    """Config 4: GMM nodes, Chung-Lu power-law degrees, distance-biased pairs.

    Node i gets expected-degree weight ``(i+1)^(-1/(gamma-1))`` (a random
    permutation decides which node is i). The source is drawn by weight; the
    target component is drawn ~ exp(-d(c_s, c_t)/scale) and the target node
    by weight inside that component.
    """
    rng = np.random.default_rng(seed)
    centres, comp, pos = _gmm_nodes(rng, n_nodes, n_comp, sd)
    w = np.empty(n_nodes)
    w[rng.permutation(n_nodes)] = (np.arange(1, n_nodes + 1, dtype=np.float64)
                                   ** (-1.0 / (gamma - 1.0)))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    s = np.minimum(np.searchsorted(cdf, rng.uniform(size=n_edges), side="right"),
                   n_nodes - 1)
    members = [np.flatnonzero(comp == c) for c in range(n_comp)]
    member_cdf = []
    comp_w = np.zeros(n_comp)
    for c, m in enumerate(members):
        if m.size:
            cw = np.cumsum(w[m])
            comp_w[c] = cw[-1]
            member_cdf.append(cw / cw[-1])
        else:
            member_cdf.append(np.ones(0))
    # target component: distance kernel x component mass
    d = np.linalg.norm(centres[:, None, :] - centres[None, :, :], axis=2)
    kern = np.exp(-d / scale) * comp_w[None, :]
    kern_cdf = np.cumsum(kern, axis=1)
    kern_cdf /= kern_cdf[:, -1:]
    cs = comp[s]
    u = rng.uniform(size=n_edges)
    ct = np.empty(n_edges, dtype=np.int64)
    for c in range(n_comp):
        sel = np.flatnonzero(cs == c)
        if sel.size:
            ct[sel] = np.minimum(np.searchsorted(kern_cdf[c], u[sel], side="right"),
                                 n_comp - 1)
    t = _pick_in_component(rng, members, member_cdf, ct)
    s, t = _drop_degenerate(pos, s, t)
    return Graph(pos, s, t)


def stress_graph(n_nodes: int, n_edges: int, n_comp: int = 256,
                 sd: float = 0.02, seed: int = 0):
    """Config 5: half uniform nodes, half from a 256-component GMM;
    uniform random endpoint pairs."""
    rng = np.random.default_rng(seed)
    n_u = n_nodes // 2
    pos_u = rng.uniform(0.0, 1.0, size=(n_u, 2))
    _, _, pos_g = _gmm_nodes(rng, n_nodes - n_u, n_comp, sd)
    pos = np.concatenate([pos_u, pos_g], axis=0)
    s = rng.integers(0, n_nodes, size=n_edges)
    t = (s + 1 + rng.integers(0, n_nodes - 1, size=n_edges)) % n_nodes
    s, t = _drop_degenerate(pos, s, t)
    return Graph(pos, s, t)


def mean_edge_cells(graph: Graph, config: BundleConfig) -> float:
    """Mean straight-edge length in grid cells under the config's transform."""
    tr = make_transform(graph.positions, config.grid_size, config.padding_cells)
    src = tr.world_to_grid(graph.positions[graph.sources])
    dst = tr.world_to_grid(graph.positions[graph.targets])
    return float(np.linalg.norm(dst - src, axis=1).mean())


def workload(k: int, *, scale: float = 1.0, seed: int = 0) -> Workload:
    """Config k (1..5) of BASELINE.json. ``scale`` < 1 shrinks node and edge
    counts proportionally (for quick tests); grid and parameters stay."""
    def n(x):
        return max(4, int(round(x * scale)))

    if k == 1:
        g = uniform_graph(n(300), n(2000), seed)
        cfg = BundleConfig(grid_size=256, sigma=16.0, delta=256 / 64,
                           iterations=10)
        bins = np.zeros(g.n_edges, dtype=np.int64)
        mat = np.eye(1, dtype=np.float32)
    elif k in (2, 3):
        if k == 2:
            g = mixture_graph(n(5000), n(50000), seed=seed)
            bins = np.zeros(g.n_edges, dtype=np.int64)
            mat = np.eye(1, dtype=np.float32)
        else:
            g = mixture_graph(n(20000), n(500000), seed=seed)
            rng = np.random.default_rng(seed + 3)
            bins = rng.integers(0, 8, size=g.n_edges).astype(np.int64)
            # inter-group attraction 0.5: every layer sum stays exact
            mat = (np.eye(8) + 0.5 * (1.0 - np.eye(8))).astype(np.float32)
        cfg = BundleConfig(grid_size=512, sigma=24.0, lambda_=0.75,
                           iterations=15)
    elif k == 4:
        g = powerlaw_mixture_graph(n(100_000), n(2_000_000), seed=seed)
        cfg = BundleConfig(grid_size=1024, iterations=10)
        cfg.delta = mean_edge_cells(g, cfg) / 63.0
        bins = np.zeros(g.n_edges, dtype=np.int64)
        mat = np.eye(1, dtype=np.float32)
    elif k == 5:
        g = stress_graph(n(1_000_000), n(20_000_000), seed=seed)
        cfg = BundleConfig(grid_size=2048, iterations=10)
        cfg.delta = mean_edge_cells(g, cfg) / 31.0
        rng = np.random.default_rng(seed + 5)
        bins = rng.integers(0, 4, size=g.n_edges).astype(np.int64)
        mat = np.eye(4, dtype=np.float32)
    else:
        raise ValueError(f"unknown config {k}")
    g = Graph(g.positions, g.sources, g.targets, None, bins)
    name = WORKLOAD_NAMES[k] + ("" if scale == 1.0 else f"@{scale:g}")
    return Workload(name, g, cfg, bins, mat)
