"""Degenerate graphs for parity tests (pure numpy: the golden script and the
GPU tests build them identically)."""

import numpy as np


def small_graphs():
    """Degenerate shapes the reference handles (positions, sources, targets,
    weights, bins, config overrides)."""
    rng = np.random.default_rng(21)
    line = np.column_stack([np.linspace(0, 1, 40), np.zeros(40)])  # collinear nodes
    return {
        "empty": (np.array([[0.0, 0.0], [1.0, 1.0], [0.5, 0.2]]), [], [], None,
                  dict(grid_size=64, iterations=3)),
        "coincident": (np.array([[0.0, 0.0], [1.0, 1.0], [0.5, 0.2], [0.5, 0.2]]),
                       [0, 2, 1], [1, 3, 2], None, dict(grid_size=64, iterations=4)),
        "single": (np.array([[0.1, 0.3], [0.9, 0.6]]), [0], [1], None,
                   dict(grid_size=48, iterations=5)),
        "collinear": (line, rng.integers(0, 20, 60), rng.integers(20, 40, 60), None,
                      dict(grid_size=128, iterations=6)),
        "border_hub": (np.vstack([[[0.0, 0.0]], rng.uniform(0, 1, (200, 2))]),
                       np.zeros(300, np.int64), rng.integers(1, 201, 300),
                       rng.integers(1, 4, 300).astype(np.float64),
                       dict(grid_size=96, iterations=8, delta=2.0)),
    }
