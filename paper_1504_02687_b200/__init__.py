"""B200-native density-guided edge bundling (arXiv 1504.02687, 3DHEB).

Drop-in for the bundling path of the reference ``histobundle`` package:
``bundle(graph, config, *, bins, matrix, workers, on_iteration, _fixed_step)``
with the reference's ``BundleConfig`` and ``BundleResult`` layout; every
iteration runs as hand-written sm_100a kernels behind the C ABI declared in
``include/histobundle_b200.h``.
"""

from .model import (BundleConfig, DensityField, Graph, GridTransform, SampledEdge,
                    interaction_matrix, make_transform)

__all__ = ["BundleConfig", "DensityField", "Graph", "GridTransform", "SampledEdge",
           "interaction_matrix", "make_transform", "bundle", "BundleResult",
           "IterationMetrics"]


def __getattr__(name):
    # torch-dependent modules load lazily so the host types import anywhere
    if name in ("bundle", "BundleResult", "IterationMetrics", "bundle_packed"):
        from . import bundler
        return getattr(bundler, name)
    raise AttributeError(name)
