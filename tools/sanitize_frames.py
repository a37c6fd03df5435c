"""Frames for compute-sanitizer (tests/test_sanitizers.py): a small scene rendered
through the default pipeline -- depth chunks (forced), tight rectangles, lanes -- as
direct, captured and replayed frames, device and host outputs, plus one stats frame.

    compute-sanitizer --tool racecheck python tools/sanitize_frames.py [n_gaussians]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SGS_DEPTH_CHUNKS", "16,4")  # every chunked code path, at a small size

import numpy as np  # noqa: E402

import paper_2501_00342_b200 as sg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
scene = sg.synth_scene(n, "mixed", 4242, log_scale_range=(-5.0, -3.5))
cams = sg.orbit_cameras(4, 256, 144, 4.0, 172.0)
r = sg.Renderer(0)
ds = r.upload(scene)
first = None
for rep in range(3):  # direct, captured, replayed
    rgb, T = r.render_batch(ds, cams, degree_override=1)
    if first is None:
        first = rgb.copy()
    assert np.array_equal(rgb, first), rep
rgb, T, st = r.render(ds, cams[0], degree_override=1, stats=True)
assert st.visible > 0
ds.free()
print("sanitize frames ok", n)
