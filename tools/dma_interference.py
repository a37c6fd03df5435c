"""Does DMA traffic slow the render? Config C batch time (32 views, device outputs)
alone and with a concurrent stream of copies on another stream and host thread:
device->host (the host-frame pattern), host->device, and device->device (copy engine
moving HBM to HBM), 33 MB each, back to back."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2501_00342_b200 as sg  # noqa: E402
scene = sg.synth_scene(3_000_000, "mixed", 20260003, log_scale_range=(-5.5, -4.0))
r = sg.Renderer(0)
ds = r.upload(scene)
cams = sg.orbit_cameras(32, 1920, 1080, 4.0, 1296.0)
out = torch.empty((32, 1080, 1920, 3), device="cuda")
d = torch.empty(33_177_600, dtype=torch.uint8, device="cuda")
d2 = torch.empty(33_177_600, dtype=torch.uint8, device="cuda")
h = torch.empty(33_177_600, dtype=torch.uint8, pin_memory=True)
cs = torch.cuda.Stream()
stop = False
moved = [0]


def copier(kind):
    with torch.cuda.stream(cs):
        while not stop:
            for _ in range(8):
                if kind == "d2h":
                    h.copy_(d, non_blocking=True)
                elif kind == "h2d":
                    d.copy_(h, non_blocking=True)
                else:
                    d2.copy_(d, non_blocking=True)
                moved[0] += d.numel()
            cs.synchronize()


def batch(k=5):
    for _ in range(2):
        r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k / 32 * 1e3


print(f"alone: {batch():.3f} ms/frame", flush=True)
for kind in ("d2h", "h2d", "d2d"):
    stop = False
    moved[0] = 0
    th = threading.Thread(target=copier, args=(kind,))
    th.start()
    time.sleep(0.1)
    t0, m0 = time.perf_counter(), moved[0]
    ms = batch()
    gbs = (moved[0] - m0) / (time.perf_counter() - t0) / 1e9
    stop = True
    th.join()
    print(f"with continuous {kind} copies: {ms:.3f} ms/frame (copies at {gbs:.1f} GB/s)", flush=True)
