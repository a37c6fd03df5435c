"""One 32-view config C batch with SGS_TRACE=1: per-frame lane timeline (host outputs
when argv[1] == 'host', else device outputs)."""
import os, sys
os.environ["SGS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2501_00342_b200 as sg  # noqa: E402
scene = sg.synth_scene(3_000_000, "mixed", 20260003, log_scale_range=(-5.5, -4.0))
r = sg.Renderer(0)
ds = r.upload(scene)
cams = sg.orbit_cameras(32, 1920, 1080, 4.0, 1296.0)
host = len(sys.argv) > 1 and sys.argv[1] == "host"
hb = torch.empty((32, 1080, 1920, 3), pin_memory=True).numpy()
hT = torch.empty((32, 1080, 1920, 1), pin_memory=True).numpy()
out = torch.empty((32, 1080, 1920, 3), device="cuda")
for _ in range(2):
    if host:
        r.render_batch(ds, cams, degree_override=1, rgb=hb, T=hT)
    else:
        r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
