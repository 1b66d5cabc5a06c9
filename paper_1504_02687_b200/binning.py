"""Edge binning on the device: the API of the reference's ``binning.py``.

Mirrors ``/root/reference/pkg/src/histobundle/binning.py`` (same names,
arguments, results and ``ValueError`` messages) so ``assign_bins`` and friends
are a drop-in.  The dense work -- every Lloyd iteration of every restart, the
centroid sums, the empty-cluster re-seed, the restart inertias and the
Davies-Bouldin scatter -- runs in ``hb_binning.cu`` (C ABI in
``include/histobundle_b200.h``), all active restarts of an iteration at once.

What stays on the host, as in the reference and for the same bits:
  * ``np.unique`` of the feature rows and the seeded ``rng.choice`` picks of
    the initial centroids (binning.py:72-77, 103-109): the random stream is
    numpy's;
  * the k x k part of Davies-Bouldin (binning.py:172-177) and the winning
    restart's ``inertia`` value (binning.py:127-129), both numpy expressions
    on k or n*d values computed once per ``kmeans`` call;
  * ``bin_by_orientation`` (binning.py:59-70): numpy's arctan2/rint per edge.
The restart with the smallest inertia is chosen from device sums (a fixed
tree order, not einsum's); restarts that converge to the same clustering tie
exactly, and the reference's first-index tie-break is kept.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .engine import ptr, stream_ptr
from .model import Graph

__all__ = ["CRITERIA", "Clustering", "edge_features", "bin_by_orientation", "kmeans",
           "davies_bouldin", "select_bins", "assign_bins"]

CRITERIA = ("none", "orientation", "origin", "destination", "od", "length", "file")

_MAX_LLOYD_ITER = 100  # binning.py:31
_CHECK_EVERY = 8       # Lloyd steps per host check for live restarts


@dataclass
class Clustering:
    """Result of one K-means run: the best restart by inertia (binning.py:34-41)."""

    k: int
    assignment: np.ndarray  # (n,) int64
    centroids: np.ndarray   # (k, d) float64
    inertia: float


def _ends(graph: Graph) -> tuple[np.ndarray, np.ndarray]:
    pos = graph.positions
    return pos[graph.sources], pos[graph.targets]


# criterion -> feature rows from (source, target) world points
_FEATURES = {
    "od": lambda a, b: np.hstack([a, b]),
    "origin": lambda a, b: a.copy(),
    "destination": lambda a, b: b.copy(),
    "length": lambda a, b: np.linalg.norm(b - a, axis=1)[:, None],
}


def edge_features(graph: Graph, criterion: str) -> np.ndarray:
    """Per-edge feature rows in world units (binning.py:44-56)."""
    make = _FEATURES.get(criterion)
    if make is None:
        raise ValueError(f"criterion {criterion!r} has no feature representation")
    return make(*_ends(graph))


def bin_by_orientation(graph: Graph, slices: int = 4) -> np.ndarray:
    """Nearest angular slice of each edge's direction (binning.py:59-70):
    slice centres at multiples of 360/slices degrees, modal bins."""
    if slices < 2:
        raise ValueError("slices must be >= 2")
    a, b = _ends(graph)
    vec = b - a
    deg = np.degrees(np.arctan2(vec[:, 1], vec[:, 0]))
    return np.rint(deg / (360.0 / slices)).astype(np.int64) % slices


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise N.NativeError("binning needs a CUDA device (no CPU fallback)")
    return torch.device("cuda")


class _DeviceFeatures:
    """Features resident on the device, shared by every kmeans of a select_bins."""

    def __init__(self, features: np.ndarray):
        self.host = features
        self.n, self.d = features.shape
        if self.d > 4:
            raise ValueError("features with more than 4 columns are not supported")
        self.t = torch.from_numpy(np.ascontiguousarray(features)).to(_dev())
        self.unique_rows = np.unique(features, axis=0)  # shared by every k


def _kmeans_device(df: _DeviceFeatures, k: int, restarts: int,
                   seed: int | np.random.SeedSequence) -> Clustering:
    f = df.host
    n, d = df.n, df.d
    if k < 1:
        raise ValueError("k must be >= 1")
    if restarts < 1:
        raise ValueError("restarts must be >= 1")
    if n < k:
        raise ValueError("k exceeds distinct points")
    unique_rows = df.unique_rows
    if unique_rows.shape[0] < k:
        raise ValueError("k exceeds distinct points")
    if k > 64:
        raise ValueError("k above 64 is not supported")
    # initial centroids: numpy's seeded stream, drawn restart by restart as
    # binning.py:72-77 does
    rng = np.random.default_rng(seed)
    picks = np.stack([rng.choice(len(unique_rows), size=k, replace=False)
                      for _ in range(restarts)])
    dev = df.t.device
    cent = torch.from_numpy(np.ascontiguousarray(unique_rows[picks])).to(dev)  # (R, k, d)
    assign = torch.full((restarts, n), -1, dtype=torch.int8, device=dev)
    # restart bookkeeping on the device (hb_kmeans_lloyd): [live | changed | empty]
    flags = torch.zeros(3 * restarts, dtype=torch.int32, device=dev)
    flags[:restarts] = 1
    wsb = int(N.lib().hb_kmeans_reseed_workspace_bytes(n, restarts))
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=dev)
    s = stream_ptr()
    done = 0
    while done < _MAX_LLOYD_ITER:  # one host check per _CHECK_EVERY iterations
        step = min(_CHECK_EVERY, _MAX_LLOYD_ITER - done)
        N.call("hb_kmeans_lloyd", ptr(df.t), n, d, k, ptr(cent), restarts, ptr(assign),
               ptr(flags), step, ptr(ws), ws.numel(), s)
        done += step
        if not bool(flags[:restarts].any()):
            break
    nb = int(N.lib().hb_kmeans_inertia_blocks())
    part = torch.empty((restarts, nb), dtype=torch.float64, device=dev)
    N.call("hb_kmeans_inertia", ptr(df.t), n, d, k, ptr(cent), restarts, ptr(assign),
           ptr(part), s)
    inertia = part.cpu().numpy().sum(axis=1)  # ordered per-block partials
    best = int(np.argmin(inertia))
    a = assign[best].cpu().numpy().astype(np.int64)
    c = cent[best].cpu().numpy()
    delta = f - c[a]  # the winner's inertia as binning.py:128 computes it
    return Clustering(k, a, c, float(np.einsum("nd,nd->", delta, delta)))


def kmeans(features: np.ndarray, k: int, restarts: int = 100,
           seed: int | np.random.SeedSequence = 0) -> Clustering:
    """Best-of-restarts Lloyd's K-means on Euclidean distance (binning.py:81-133)."""
    features = np.asarray(features, dtype=np.float64)
    if features.ndim != 2:
        raise ValueError("features must be a 2D matrix")
    return _kmeans_device(_DeviceFeatures(features), k, restarts, seed)


def _davies_bouldin(df: _DeviceFeatures, clustering: Clustering) -> float:
    k = clustering.k
    if k < 2:
        raise ValueError("davies_bouldin needs k >= 2")
    dev = df.t.device
    a = torch.from_numpy(clustering.assignment.astype(np.int8)).to(dev)
    c = torch.from_numpy(np.ascontiguousarray(clustering.centroids)).to(dev)
    scatter = torch.empty(k, dtype=torch.float64, device=dev)
    counts = torch.empty(k, dtype=torch.int64, device=dev)
    N.call("hb_kmeans_scatter", ptr(df.t), df.n, df.d, k, ptr(c), ptr(a), ptr(scatter),
           ptr(counts), stream_ptr())
    counts = counts.cpu().numpy()
    if (counts == 0).any():
        raise ValueError("degenerate clustering: empty cluster")
    scatter = scatter.cpu().numpy() / counts  # binning.py:171
    cen = clustering.centroids
    cd = np.linalg.norm(cen[:, None, :] - cen[None, :, :], axis=2)
    with np.errstate(divide="ignore"):
        ratio = (scatter[:, None] + scatter[None, :]) / cd
    np.fill_diagonal(ratio, -np.inf)
    return float(np.mean(ratio.max(axis=1)))


def davies_bouldin(features: np.ndarray, clustering: Clustering) -> float:
    """Cluster validity index, lower is better (binning.py:157-177)."""
    features = np.asarray(features, dtype=np.float64)
    return _davies_bouldin(_DeviceFeatures(features), clustering)


def select_bins(features: np.ndarray, kmin: int = 4, kmax: int = 16,
                restarts: int = 100, seed: int = 0) -> tuple[np.ndarray, int]:
    """Bin count in [kmin, kmax] minimising Davies-Bouldin (binning.py:180-201):
    one child seed per candidate k, ties to the smaller k."""
    if kmin < 2:
        raise ValueError("kmin must be >= 2")
    if kmax < kmin:
        raise ValueError("kmax must be >= kmin")
    features = np.asarray(features, dtype=np.float64)
    if features.ndim != 2:
        raise ValueError("features must be a 2D matrix")
    df = _DeviceFeatures(features)
    seeds = np.random.SeedSequence(seed).spawn(kmax - kmin + 1)
    scored = []
    for k, child in zip(range(kmin, kmax + 1), seeds):
        cl = _kmeans_device(df, k, restarts, child)
        scored.append((_davies_bouldin(df, cl), k, cl.assignment))
    # first strict minimum in k order (a NaN index never wins, as `db < best`)
    win = None
    for db, k, a in scored:
        if win is None and db < np.inf or win is not None and db < win[0]:
            win = (db, k, a)
    assert win is not None
    return win[2], win[1]


def _ordinal(assignment: np.ndarray, centroids: np.ndarray) -> np.ndarray:
    """Relabel clusters by ascending first centroid coordinate (stable)."""
    rank = np.argsort(np.argsort(centroids[:, 0], kind="stable"), kind="stable")
    return rank.astype(np.int64)[assignment]


def assign_bins(graph: Graph, criterion: str, bins: int | str = "auto", slices: int = 4,
                restarts: int = 100, seed: int = 0) -> tuple[np.ndarray, int, str]:
    """Per-edge bins for a named criterion (binning.py:211-246):
    (assignment, bin count, palette kind)."""
    if criterion not in CRITERIA:
        raise ValueError(f"unknown criterion {criterion!r}; "
                         f"expected one of {', '.join(CRITERIA)}")
    if criterion == "none":
        return np.zeros(graph.n_edges, dtype=np.int64), 1, "single"
    if criterion == "file":
        return graph.bins.copy(), graph.bin_count, "nominal"
    if criterion == "orientation":
        count = slices if bins == "auto" else int(bins)
        return bin_by_orientation(graph, count), count, "modal"
    feats = edge_features(graph, criterion)
    if bins != "auto":
        cl = kmeans(feats, int(bins), restarts=restarts, seed=seed)
        labels, count, cent = cl.assignment, cl.k, cl.centroids
    else:
        labels, count = select_bins(feats, restarts=restarts, seed=seed)
        cent = np.stack([feats[labels == c].mean(axis=0) for c in range(count)])
    if criterion == "length":  # ordinal palette: bin index grows with length
        return _ordinal(labels, cent), count, "ordinal"
    return labels, count, "nominal"
