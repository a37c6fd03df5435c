"""The C-ABI multi-GPU path (sgs_group_*) on the one GPU of the box:
world-size-1 groups made both ways (sgs_group_create: ncclCommInitAll in one
process; sgs_group_init_rank: a shipped NCCL unique id, as one process per GPU under
torchrun does), the scene through the NCCL broadcast, the views through the
gather-to-root path. Frames must equal a plain render_batch bit for bit.
(More ranks need more GPUs: NCCL refuses two ranks on one device. The block
partition and the multi-rank host logic are covered by tests/test_multiview_gloo.py.)"""
import threading

import numpy as np
import pytest

import paper_2501_00342_b200 as sg
from paper_2501_00342_b200.multiview import RenderGroup

pytestmark = pytest.mark.gpu


def _scene_cams():
    scene = sg.synth_scene(150_000, "mixed", 2026, log_scale_range=(-5.0, -3.5))
    cams = sg.orbit_cameras(11, 320, 180, 4.0, 216.0)  # 11: not a multiple of the sub-batch
    return scene, cams


def _reference(scene, cams):
    r = sg.Renderer(0)
    ds = r.upload(scene)
    try:
        return r.render_batch(ds, cams, degree_override=1)
    finally:
        ds.free()


def test_group_create_world1_matches_render_batch():
    scene, cams = _scene_cams()
    want = _reference(scene, cams)
    (g,) = RenderGroup.create([0])
    try:
        ds = g.broadcast_scene(scene, root=0)
        for _ in range(3):  # direct, captured, replayed frames
            rgb, T = g.render_views(ds, cams, root=0, degree_override=1)
            assert np.array_equal(rgb, want[0]) and np.array_equal(T, want[1])
        rgb, T = g.render_views(ds, cams, root=0, degree_override=1, T=False)
        assert np.array_equal(rgb, want[0])
        ds.free()
    finally:
        g.close()


def test_group_init_rank_world1_device_outputs():
    import torch

    scene, cams = _scene_cams()
    want = _reference(scene, cams)
    uid = RenderGroup.unique_id()
    r = sg.Renderer(0)
    out = {}

    def rank0():  # the collective calls of rank 0 (a thread, as one per rank would be)
        g = RenderGroup.init_rank(r, 1, 0, uid)
        try:
            ds = g.broadcast_scene(scene, root=0)
            rgb = torch.empty((len(cams), 180, 320, 3), device="cuda")
            T = torch.empty((len(cams), 180, 320, 1), device="cuda")
            g.render_views(ds, cams, root=0, degree_override=1, rgb=rgb.data_ptr(), T=T.data_ptr(),
                           device_out=True)
            torch.cuda.synchronize()
            out["rgb"], out["T"] = rgb.cpu().numpy(), T.cpu().numpy()
            ds.free()
        finally:
            g.close()

    t = threading.Thread(target=rank0)
    t.start()
    t.join(timeout=600)
    assert not t.is_alive()
    assert np.array_equal(out["rgb"], want[0]) and np.array_equal(out["T"], want[1])


def test_group_errors():
    with pytest.raises(sg.InvalidArgumentError):
        RenderGroup.create([])
    r = sg.Renderer(0)
    with pytest.raises(sg.InvalidArgumentError):
        RenderGroup.init_rank(r, 2, 2, bytes(128))
    # views of different sizes cannot share the gather stride
    scene, cams = _scene_cams()
    (g,) = RenderGroup.create([0])
    try:
        ds = g.broadcast_scene(scene, root=0)
        mixed = cams[:2] + sg.orbit_cameras(1, 160, 90, 4.0, 108.0)
        with pytest.raises(sg.InvalidArgumentError):
            g.render_views(ds, mixed, root=0, degree_override=1)
        ds.free()
    finally:
        g.close()
