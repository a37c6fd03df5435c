"""Frames for ncu: one 8-view batch (config C) with the multi-view K1 (SGS_K1_GROUP)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2501_00342_b200 as sg  # noqa: E402
scene = sg.synth_scene(3_000_000, "mixed", 20260003, log_scale_range=(-5.5, -4.0))
r = sg.Renderer(0)
ds = r.upload(scene)
cams = sg.orbit_cameras(8, 1920, 1080, 4.0, 1296.0, 0.35)
out = torch.empty((8, 1080, 1920, 3), device="cuda")
for _ in range(2):
    r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
torch.cuda.synchronize()
print("ok")
