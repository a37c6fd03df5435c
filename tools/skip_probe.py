"""Marginal cost of each stage in the 4-lane batch: config C, 32 views, device outputs,
timed with SGS_SKIP masks (1 = no K7, 2 = no K1, 4 = no K2; the skipped stage's
outputs are stale, so images are garbage -- a timing probe only). One subprocess per mask."""
import os, subprocess, sys

CHILD = r'''
import os, sys, time; sys.path.insert(0, '.')
import torch, paper_2501_00342_b200 as sg
scene = sg.synth_scene(3_000_000, "mixed", 20260003, log_scale_range=(-5.5, -4.0))
r = sg.Renderer(0); ds = r.upload(scene)
cams = sg.orbit_cameras(32, 1920, 1080, 4.0, 1296.0)
out = torch.empty((32, 1080, 1920, 3), device="cuda")
for _ in range(3): r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
torch.cuda.synchronize()
os.environ["SGS_SKIP"] = sys.argv[1]  # after warm-up: skipped stages keep the last real frame's outputs
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record()
    r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
    e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / 32)
print("RESULT", best)
'''
masks = [int(a) for a in sys.argv[1:]] or [0, 2, 4, 6]
for m in masks:
    o = subprocess.run([sys.executable, "-c", CHILD, str(m)], capture_output=True, text=True)
    res = [l for l in o.stdout.splitlines() if l.startswith("RESULT")]
    print(f"SGS_SKIP={m}: {res[0].split()[1] if res else o.stderr[-500:]} ms/frame", flush=True)
