"""CPU ORACLE for edge binning -- TEST INFRASTRUCTURE, never the product path.

A numpy restatement of the reference's K-means / Davies-Bouldin selection
(/root/reference/pkg/src/histobundle/binning.py:72-201), written restart by
restart with every reduction order spelled out, so the device version
(paper_1504_02687_b200/binning.py + csrc/hb_binning.cu) can be checked
against it and it can be checked against fixtures made by running the
reference itself (tests/golden/binning.npz, tests/golden/make_binning_golden.py).

Orders the reference inherits from numpy 2.3 (checked in this container):
  * einsum("rnkd,rnkd->rnk") pairs 4 squared columns as (p0+p2)+(p1+p3) and
    adds 1-2 columns in order;
  * np.linalg.norm(axis=1) adds the squared columns in order;
  * np.add.at folds rows in index order, starting from 0.0.
Who may import this module: tests/ only.
"""

from __future__ import annotations

import numpy as np

LLOYD_MAX = 100  # binning.py:31


def sq_dist(F: np.ndarray, C: np.ndarray) -> np.ndarray:
    """(n, d) x (k, d) -> (n, k) squared distances, einsum's association."""
    D = F[:, None, :] - C[None, :, :]
    P = D * D
    if F.shape[1] == 4:
        return (P[..., 0] + P[..., 2]) + (P[..., 1] + P[..., 3])
    acc = P[..., 0]
    for j in range(1, F.shape[1]):
        acc = acc + P[..., j]
    return acc


def row_norm(X: np.ndarray) -> np.ndarray:
    """np.linalg.norm(X, axis=1): squares summed left to right, then sqrt."""
    acc = X[:, 0] * X[:, 0]
    for j in range(1, X.shape[1]):
        acc = acc + X[:, j] * X[:, j]
    return np.sqrt(acc)


def fold_by_label(X: np.ndarray, labels: np.ndarray, k: int) -> np.ndarray:
    """np.add.at(zeros, labels, X): per label a left fold from 0.0 in row order."""
    out = np.zeros((k,) + X.shape[1:])
    for c in range(k):
        rows = X[labels == c]
        if len(rows):
            out[c] = np.cumsum(np.concatenate([out[c:c + 1], rows]), axis=0)[-1]
    return out


def update(F: np.ndarray, labels: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Centroid step with the farthest-point re-seed of emptied clusters."""
    k = C.shape[0]
    n_c = np.bincount(labels, minlength=k).astype(np.float64)
    S = fold_by_label(F, labels, k)
    new = C.copy()
    full = n_c > 0
    new[full] = S[full] / n_c[full][:, None]
    if not full.all():
        far = row_norm(F - new[labels])
        for c in np.flatnonzero(~full):
            i = int(np.argmax(far))
            new[c] = F[i]
            far[i] = -np.inf
    return new


def kmeans(F: np.ndarray, k: int, restarts: int, seed) -> tuple[np.ndarray, np.ndarray, float]:
    """(assignment, centroids, inertia) of the best restart."""
    F = np.asarray(F, dtype=np.float64)
    uniq = np.unique(F, axis=0)
    rng = np.random.default_rng(seed)
    starts = [uniq[rng.choice(len(uniq), size=k, replace=False)] for _ in range(restarts)]
    best = None
    for r in range(restarts):
        C = starts[r].copy()
        lab = np.full(len(F), -1, dtype=np.int64)
        for _ in range(LLOYD_MAX):
            new = np.argmin(sq_dist(F, C), axis=1)
            moved = bool((new != lab).any())
            lab = new
            if not moved:
                break
            C = update(F, lab, C)
        res = F - C[lab]
        inertia = float(np.einsum("nd,nd->", res, res))
        if best is None or inertia < best[2]:
            best = (lab, C, inertia)
    return best


def davies_bouldin(F: np.ndarray, labels: np.ndarray, C: np.ndarray) -> float:
    k = C.shape[0]
    n_c = np.bincount(labels, minlength=k)
    spread = fold_by_label(row_norm(F - C[labels]), labels, k) / n_c
    sep = np.stack([row_norm(C - C[i]) for i in range(k)])
    with np.errstate(divide="ignore"):
        worst = (spread[:, None] + spread[None, :]) / sep
    np.fill_diagonal(worst, -np.inf)
    return float(np.mean(worst.max(axis=1)))


def select_bins(F: np.ndarray, restarts: int, seed: int, kmin: int = 4, kmax: int = 16):
    seeds = np.random.SeedSequence(seed).spawn(kmax - kmin + 1)
    win = (np.inf, None, None)
    for k, s in zip(range(kmin, kmax + 1), seeds):
        lab, C, _ = kmeans(F, k, restarts, s)
        db = davies_bouldin(F, lab, C)
        if db < win[0]:
            win = (db, lab, k)
    return win[1], win[2]
