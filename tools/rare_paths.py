import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, paper_2501_00342_b200 as sg
import oracle_lib as ol
from test_gpu_parity import _adversarial, to_scene, to_cam, cfg_kwargs
orc = ol.OrcLib()
r = sg.Renderer(0)
for name in (sys.argv[1:] or ["ties", "spike", "huge", "culled", "tile32"]):
    f, ocam, cfg = _adversarial(orc, name)
    ds = r.upload(to_scene(f)); cam = to_cam(ocam)
    a = r.launch_count()
    rgb, T, st = r.render(ds, cam, stats=True, **cfg_kwargs(cfg))
    b = r.launch_count()
    print(name, "own", b[0]-a[0], "lib", b[1]-a[1], "V", st.visible, "P", st.tile_entries)
    ds.free()
