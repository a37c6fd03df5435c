"""Host-side cost per frame: a tiny scene / image makes the GPU work negligible, so a
batch's wall time per frame is the enqueue + per-frame settle overhead."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2501_00342_b200 as sg  # noqa: E402
for n, w, h in ((1000, 64, 64), (100_000, 256, 256)):
    scene = sg.synth_scene(n, "mixed", 5, log_scale_range=(-5.0, -3.5))
    r = sg.Renderer(0)
    ds = r.upload(scene)
    cams = sg.orbit_cameras(64, w, h, 4.0, 0.9 * h)
    out = torch.empty((64, h, w, 3), device="cuda")
    for _ in range(3):
        r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
    torch.cuda.synchronize()
    print(f"N={n} {w}x{h}: {(time.perf_counter() - t) / 5 / 64 * 1e6:.1f} us/frame")
    ds.free()
