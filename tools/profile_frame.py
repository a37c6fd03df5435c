"""Render a few frames of BASELINE config C (device outputs) for ncu / nsys-style capture.

    python tools/profile_frame.py [frames] [n_gaussians]
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_00342_b200 as sg  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3_000_000
scene = sg.synth_scene(n, "mixed", 20260003, log_scale_range=(-5.5, -4.0))
r = sg.Renderer(0)
ds = r.upload(scene)
cams = sg.orbit_cameras(256, 1920, 1080, 4.0, 1296.0, 0.35)
rgb = torch.empty((1080, 1920, 3), device="cuda")
T = torch.empty((1080, 1920, 1), device="cuda")
for i in range(frames):
    r.render(ds, cams[i % 256], degree_override=1, rgb=rgb.data_ptr(), T=T.data_ptr(), device_out=True)
torch.cuda.synchronize()
print("frames", frames, "ok")
