"""Batch throughput (config C, 32 views, device outputs, best of 5) under pipeline
knobs given as environment assignments, one subprocess per setting:

    python tools/env_sweep.py "" "SGS_BIN_FUSED=1" "SGS_LANES=6" "SGS_DEPTH_CHUNKS=32,8,2"
"""
import os, subprocess, sys

CHILD = r'''
import sys; sys.path.insert(0, '.')
import torch, paper_2501_00342_b200 as sg
scene = sg.synth_scene(3_000_000, "mixed", 20260003, log_scale_range=(-5.5, -4.0))
r = sg.Renderer(0); ds = r.upload(scene)
cams = sg.orbit_cameras(32, 1920, 1080, 4.0, 1296.0)
out = torch.empty((32, 1080, 1920, 3), device="cuda")
for _ in range(3): r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record()
    r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
    e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / 32)
print("RESULT", best)
'''
for setting in sys.argv[1:] or [""]:
    env = dict(os.environ)
    for kv in setting.split():
        k, v = kv.split("=", 1)
        env[k] = v
    o = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    res = [l for l in o.stdout.splitlines() if l.startswith("RESULT")]
    print(f"[{setting or 'default'}] {res[0].split()[1] if res else o.stderr[-400:]} ms/frame", flush=True)
