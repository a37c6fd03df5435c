"""Does device-to-host DMA slow the render? Batch time with and without a concurrent
stream of D2H copies (separate buffers, separate stream)."""
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
h = torch.empty(33_177_600, dtype=torch.uint8, pin_memory=True)
cs = torch.cuda.Stream()
stop = False


def copier():
    with torch.cuda.stream(cs):
        while not stop:
            for _ in range(8):
                h.copy_(d, non_blocking=True)
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


print(f"alone: {batch():.3f} ms/frame")
th = threading.Thread(target=copier)
th.start()
time.sleep(0.1)
print(f"with continuous D2H copies: {batch():.3f} ms/frame")
stop = True
th.join()
