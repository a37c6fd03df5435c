"""GPU backward (grad.hpp, grad.cpp:69-246).

Compared with the reference's own backward (tests/golden/backward/, generated through
oracle/_ref by tests/golden/make_golden_backward.py) for every colour model, adaptive
and overridden SH degree, and tile sizes 8, 16 and 24 (several pixel chunks per
tile). Both are FP64; the per-splat sums run in a different order (fixed-order GPU
trees instead of the reference's worker-merged buffers), so the tolerance is
|ours - ref| <= 1e-9 * max|ref| per parameter. The result is deterministic run to run.
"""
import glob
import os

import numpy as np
import pytest

import paper_2501_00342_b200 as sg
from oracle_lib import camera_from_dict

pytestmark = pytest.mark.gpu

CASES = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "backward", "*.npz")))


def _load(path):
    d = np.load(path)
    scene = sg.Scene(str(d["kind"]), int(d["degree"]), d["params"], d["axes"], d["background"])
    cam_d = {k[4:]: d[k] for k in d.files if k.startswith("cam_")}
    cam_d = {k: (v.item() if v.ndim == 0 else v) for k, v in cam_d.items()}
    cam = sg.Camera._from_c(sg._capi.sgs_camera.from_buffer_copy(bytes(camera_from_dict(cam_d))))
    return d, scene, cam


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(p)[:-4] for p in CASES])
def test_backward_matches_reference(path):
    d, scene, cam = _load(path)
    r = sg.Renderer(0)
    ds = r.upload(scene)
    try:
        g = r.backward(ds, cam, d["upstream"], tile_size=int(d["tile"]), degree_override=int(d["override"]))
        ref = d["grads"]
        assert g.shape == ref.shape
        scale = np.abs(ref).max()
        assert np.abs(g - ref).max() <= 1e-9 * scale, np.abs(g - ref).max() / scale
        assert np.array_equal(np.abs(g).sum(1) > 0, np.abs(ref).sum(1) > 0)  # same culled set
        again = r.backward(ds, cam, d["upstream"], tile_size=int(d["tile"]), degree_override=int(d["override"]))
        assert np.array_equal(g, again)  # deterministic
    finally:
        ds.free()


def test_backward_device_upstream_and_errors():
    import torch

    d, scene, cam = _load(CASES[0])
    r = sg.Renderer(0)
    ds = r.upload(scene)
    try:
        host = r.backward(ds, cam, d["upstream"], tile_size=int(d["tile"]), degree_override=int(d["override"]))
        dev = r.backward(ds, cam, torch.as_tensor(d["upstream"], device="cuda"), tile_size=int(d["tile"]),
                         degree_override=int(d["override"]))
        assert dev.is_cuda and np.array_equal(dev.cpu().numpy(), host)
        bad = d["upstream"].copy()
        bad[3, 4, 1] = np.nan
        with pytest.raises(sg.NumericError, match="non-finite upstream gradient"):
            r.backward(ds, cam, bad, degree_override=int(d["override"]))
        with pytest.raises(sg.InvalidArgumentError):
            r.backward(ds, cam, d["upstream"][:-1], degree_override=int(d["override"]))
    finally:
        ds.free()
