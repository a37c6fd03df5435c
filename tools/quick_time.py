import sys, time; sys.path.insert(0, '.')
import numpy as np, paper_2501_00342_b200 as sg
t0=time.time(); scene = sg.synth_scene(3_000_000, "mixed", 20260003, log_scale_range=(-5.5, -4.0)); t1=time.time()
r = sg.Renderer(0); ds = r.upload(scene); t2=time.time()
print(f"synth {t1-t0:.1f}s upload {t2-t1:.1f}s", flush=True)
cam = sg.orbit_camera([0,0,0], 4.0, 0.5, 0.3, 1920, 1080, 1296.0)
for i in range(5):
    rgb, T, st = r.render(ds, cam, degree_override=1, stats=True, timing=True)
print("V P E_t guard", st.visible, st.tile_entries, st.block_entries, st.guard_hits)
print({k: round(v,3) for k,v in st.ms.items()})
import torch
out = torch.empty((1080,1920,3), device='cuda'); 
for i in range(3): r.render(ds, cam, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
torch.cuda.synchronize(); t=time.time()
for i in range(20): r.render(ds, cam, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
torch.cuda.synchronize(); print("wall ms/frame", (time.time()-t)/20*1000)
