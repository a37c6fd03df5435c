"""D2H copy bandwidth alone and while the renderer runs a device-output batch
(context for the e2e number: do frame copies slow down under load?)."""
import sys, threading, time
sys.path.insert(0, '.')
import torch
import paper_2501_00342_b200 as sg

n = 33_177_600
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s = torch.cuda.Stream()


def copies(k):
    with torch.cuda.stream(s):
        for _ in range(k):
            h.copy_(d, non_blocking=True)
    s.synchronize()


copies(3)
t = time.perf_counter(); copies(40); dt = (time.perf_counter() - t) / 40
print(f"alone: {n / dt / 1e9:.1f} GB/s")

scene = sg.synth_scene(3_000_000, "mixed", 20260003, log_scale_range=(-5.5, -4.0))
r = sg.Renderer(0)
ds = r.upload(scene)
cams = sg.orbit_cameras(32, 1920, 1080, 4.0, 1296.0)
out = torch.empty((32, 1080, 1920, 3), device="cuda")
r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
torch.cuda.synchronize()
stop = False


def render_loop():
    while not stop:
        r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)


th = threading.Thread(target=render_loop)
th.start()
time.sleep(0.2)
t = time.perf_counter(); copies(40); dt = (time.perf_counter() - t) / 40
stop = True
th.join()
print(f"under render load: {n / dt / 1e9:.1f} GB/s")
