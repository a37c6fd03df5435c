"""Timings of the next-row features at config C scale (1 B200): backward, SSIM,
PLY device load. Prints one line per feature."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_00342_b200 as sg  # noqa: E402

scene = sg.synth_scene(3_000_000, "mixed", 20260003, log_scale_range=(-5.5, -4.0))
r = sg.Renderer(0)
ds = r.upload(scene)
cam = sg.orbit_camera([0, 0, 0], 4.0, 0.5, 0.3, 1920, 1080, 1296.0)
up = torch.randn((1080, 1920, 3), dtype=torch.float64, device="cuda")
for _ in range(2):
    g = r.backward(ds, cam, up, degree_override=1)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    g = r.backward(ds, cam, up, degree_override=1)
torch.cuda.synchronize()
print(f"backward 3M 1080p: {(time.perf_counter() - t) / 5 * 1e3:.1f} ms/call (device upstream and grads)")
a = torch.rand((1080, 1920, 3), dtype=torch.float64, device="cuda")
b = torch.rand((1080, 1920, 3), dtype=torch.float64, device="cuda")
sg.ssim_with_grad(a, b)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    sg.ssim(a, b)
torch.cuda.synchronize()
t1 = time.perf_counter()
for _ in range(10):
    sg.ssim_with_grad(a, b)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"ssim 1080p: {(t1 - t) * 100:.2f} ms, ssim_with_grad: {(t2 - t1) * 100:.2f} ms")
# PLY: write the scene as an SG-extended checkpoint with numpy (mixed layout), load on device
p = "/tmp/sgs_c.ply"
prm = scene.params
n = prm.shape[0]
cols = [prm[:, 0], prm[:, 1], prm[:, 2], prm[:, 11], prm[:, 12], prm[:, 13]]
lobes = prm[:, 11 + 27:11 + 39].reshape(n, 3, 4)
cols += [lobes[:, i, c] for i in range(3) for c in range(3)] + [lobes[:, i, 3] for i in range(3)]
cols += [np.zeros(n)] * 3
sh = prm[:, 11:11 + 27].reshape(n, 9, 3)
cols += [sh[:, 1 + k % 8, k // 8] for k in range(24)]
cols += [prm[:, 10], prm[:, 7], prm[:, 8], prm[:, 9], prm[:, 3], prm[:, 4], prm[:, 5], prm[:, 6]]
names = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2"] + [f"sg_alpha_{i}_{c}" for i in range(3) for c in range(3)]
names += [f"sg_lambda_{i}" for i in range(3)] + ["sg_mu_0", "sg_mu_1", "sg_mu_2"] + [f"sh2_{k}" for k in range(24)]
names += ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
with open(p, "wb") as f:
    f.write(("ply\nformat binary_little_endian 1.0\ncomment sg_model mixed\n"
             f"element vertex {n}\n" + "".join(f"property float {c}\n" for c in names) + "end_header\n").encode())
    f.write(np.stack(cols, 1).astype("<f4").tobytes())
t = time.perf_counter()
d2 = r.load_ply(p)
torch.cuda.synchronize()
t1 = time.perf_counter()
s2 = sg.load_scene(p)
t2 = time.perf_counter()
print(f"ply {os.path.getsize(p) / 1e6:.0f} MB: device load {(t1 - t) * 1e3:.0f} ms, host read {(t2 - t1) * 1e3:.0f} ms, "
      f"params equal to the source scene: {np.array_equal(s2.params, scene.params)}")
