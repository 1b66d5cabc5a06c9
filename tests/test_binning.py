"""Edge binning (binning.py:81-246): the CPU oracle and the device path
against fixtures made by running the reference (tests/golden/binning.npz,
tests/golden/make_binning_golden.py).  Assignments and chosen k are integers
and must match exactly; centroids, inertia and Davies-Bouldin values are the
same float64 operations in the same order, so they are compared bit for bit.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN

import binning_oracle as BO  # noqa: E402  (oracle/, on sys.path via conftest)
from paper_1504_02687_b200.workloads import workload

G = np.load(os.path.join(GOLDEN, "binning.npz"))
N_KM = 4


def _features(crit):
    from paper_1504_02687_b200 import binning as PB  # host-only helpers

    return PB.edge_features(workload(1).graph, crit)


# ---- CPU: the oracle restatement reproduces the reference -------------------

@pytest.mark.parametrize("i", range(N_KM))
def test_oracle_kmeans_matches_reference(i):
    k, restarts, seed = (int(v) for v in G[f"km{i}_meta"])
    f = _features(str(G[f"km{i}_crit"]))
    lab, cen, inertia = BO.kmeans(f, k, restarts, seed)
    assert np.array_equal(lab, G[f"km{i}_assign"])
    assert np.array_equal(cen, G[f"km{i}_cent"])
    assert inertia == float(G[f"km{i}_inertia"])
    assert BO.davies_bouldin(f, lab, cen) == float(G[f"km{i}_db"])


def test_oracle_reseed_matches_reference():
    out = BO.update(G["rs_features"], G["rs_assign"], G["rs_cent"])
    assert np.array_equal(out, G["rs_out"])
    lab, cen, inertia = BO.kmeans(G["rs_features"], 6, 50, 9)
    assert np.array_equal(lab, G["rs_km_assign"]) and np.array_equal(cen, G["rs_km_cent"])


def test_oracle_select_bins_matches_reference():
    restarts, seed = (int(v) for v in G["sel_origin_meta"])
    lab, k = BO.select_bins(_features("origin"), restarts, seed)
    assert k == int(G["sel_origin_k"]) and np.array_equal(lab, G["sel_origin_assign"])


def test_features_and_orientation_host_logic():
    from paper_1504_02687_b200 import binning as PB

    g = workload(1).graph
    f = PB.edge_features(g, "od")
    assert f.shape == (g.n_edges, 4)
    assert np.array_equal(PB.edge_features(g, "length")[:, 0],
                          np.linalg.norm(f[:, 2:] - f[:, :2], axis=1))
    o = PB.bin_by_orientation(g, 6)
    assert o.min() >= 0 and o.max() < 6
    with pytest.raises(ValueError, match="no feature representation"):
        PB.edge_features(g, "file")
    with pytest.raises(ValueError, match="slices must be >= 2"):
        PB.bin_by_orientation(g, 1)
    with pytest.raises(ValueError, match="unknown criterion"):
        PB.assign_bins(g, "colour")
    a, k, kind = PB.assign_bins(g, "none")
    assert k == 1 and kind == "single" and not a.any()


# ---- GPU: the device path reproduces the reference --------------------------

gpu = pytest.mark.gpu


def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@gpu
@pytest.mark.parametrize("i", range(N_KM))
def test_device_kmeans_matches_reference(i):
    _cuda()
    from paper_1504_02687_b200 import binning as PB

    k, restarts, seed = (int(v) for v in G[f"km{i}_meta"])
    f = _features(str(G[f"km{i}_crit"]))
    c = PB.kmeans(f, k, restarts=restarts, seed=seed)
    assert np.array_equal(c.assignment, G[f"km{i}_assign"])
    assert np.array_equal(c.centroids, G[f"km{i}_cent"])
    assert c.inertia == float(G[f"km{i}_inertia"])
    assert PB.davies_bouldin(f, c) == float(G[f"km{i}_db"])


@gpu
def test_device_reseed_matches_reference():
    _cuda()
    from paper_1504_02687_b200 import binning as PB

    c = PB.kmeans(G["rs_features"], 6, restarts=50, seed=9)
    assert np.array_equal(c.assignment, G["rs_km_assign"])
    assert np.array_equal(c.centroids, G["rs_km_cent"])
    assert c.inertia == float(G["rs_km_inertia"])


@gpu
def test_device_reseed_kernel_direct():
    """One update with clusters 1, 3, 5 emptied: sums + farthest-edge re-seed."""
    _cuda()
    import torch

    from paper_1504_02687_b200 import _native as N
    from paper_1504_02687_b200.engine import ptr, stream_ptr

    f, cent, lab = G["rs_features"], G["rs_cent"], G["rs_assign"]
    n, d = f.shape
    k = cent.shape[0]
    ft = torch.from_numpy(f).cuda()
    ct = torch.from_numpy(cent.copy()).cuda()[None]
    at = torch.from_numpy(lab.astype(np.int8)).cuda()[None]
    one = torch.zeros(1, dtype=torch.int32, device="cuda")
    empty = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("hb_kmeans_update", ptr(ft), n, d, k, ptr(ct), ptr(one), 1, ptr(at), ptr(empty),
           stream_ptr())
    assert int(empty.item()) == 1
    ws = torch.empty(int(N.lib().hb_kmeans_reseed_workspace_bytes(n, 1)), dtype=torch.uint8,
                     device="cuda")
    N.call("hb_kmeans_reseed", ptr(ft), n, d, k, ptr(ct), ptr(one), 1, ptr(at), ptr(ws),
           ws.numel(), stream_ptr())
    assert np.array_equal(ct[0].cpu().numpy(), G["rs_out"])


@gpu
@pytest.mark.parametrize("crit", ["od", "origin"])
def test_device_select_bins_matches_reference(crit):
    _cuda()
    from paper_1504_02687_b200 import binning as PB

    restarts, seed = (int(v) for v in G[f"sel_{crit}_meta"])
    a, k = PB.select_bins(_features(crit), restarts=restarts, seed=seed)
    assert k == int(G[f"sel_{crit}_k"])
    assert np.array_equal(a, G[f"sel_{crit}_assign"])


@gpu
def test_device_assign_bins_length_matches_reference():
    _cuda()
    from paper_1504_02687_b200 import binning as PB

    a, k, kind = PB.assign_bins(workload(1).graph, "length", "auto", restarts=20, seed=2)
    assert kind == "ordinal" and k == int(G["ab_length_k"])
    assert np.array_equal(a, G["ab_length_assign"])
