"""Every BASELINE.json / SURVEY.md §8(d) configuration on one GPU, with the reference's
own CPU render beside it (oracle/_ref/libsgsref_fast.so on this host, all threads):

    python tools/config_table.py [out.json]

Rows: A (100K, 3 SG + SH0 via override 0, 800x800), A-sg3 (make_synthetic_scene's sg3
model: diffuse + 3 orthogonal SG lobes, same N / seed / resolution; its positions come
from the sg3 draw order, synth.cpp:44-101), B (1M, SG + SH1, 1080p), C (3M, SG + SH1,
1080p), C-adaptive (C without the override: per-splat degree from its radius, the
paper's Eq. 9), D (C's geometry with degree-3 SH colour, no override). GPU: frames/s of
a 32-view batch on the config's orbit ring (device outputs, best of 5 after warm-up)
and of single frames; V / P / E_t from the frame counters. CPU: median of the
reference's render of view 0 (1 frame for the 1M/3M rows, 3 for the 100K rows).
"""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_00342_b200 as sg  # noqa: E402
from oracle_lib import KINDS, REF_FAST_SO, RefLib, make_config  # noqa: E402  (CPU reference leg only)

CONFIGS = [
    # name, N, seed, kind, log-scale, W, H, focal, override
    ("A", 100_000, 20260001, "mixed", (-4.5, -2.5), 800, 800, 960.0, 0),
    ("A-sg3", 100_000, 20260001, "sg3", (-4.5, -2.5), 800, 800, 960.0, -1),
    ("B", 1_000_000, 20260002, "mixed", (-5.5, -4.0), 1920, 1080, 1296.0, 1),
    ("C", 3_000_000, 20260003, "mixed", (-5.5, -4.0), 1920, 1080, 1296.0, 1),
    ("C-adaptive", 3_000_000, 20260003, "mixed", (-5.5, -4.0), 1920, 1080, 1296.0, -1),
    ("D", 3_000_000, 20260003, "sh3", (-5.5, -4.0), 1920, 1080, 1296.0, -1),
]


def scene_for(name, n, seed, kind, ls, cache):
    if kind == "sh3":
        base = cache.get(("mixed", n, seed)) or sg.synth_scene(n, "mixed", seed, log_scale_range=ls)
        return sg.synth_sh3_from_mixed(base, seed + 1)
    key = (kind, n, seed)
    if key not in cache:
        cache[key] = sg.synth_scene(n, kind, seed, log_scale_range=ls)
    return cache[key]


def gpu_rows(r, scene, W, H, f, ov):
    ds = r.upload(scene)
    cams = sg.orbit_cameras(32, W, H, 4.0, f)
    out = torch.empty((32, H, W, 3), device="cuda")
    one = torch.empty((H, W, 3), device="cuda")
    kw = dict(degree_override=ov)
    for _ in range(2):
        r.render_batch(ds, cams, rgb=out.data_ptr(), T=None, device_out=True, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    batch = 1e9
    for _ in range(5):
        e0.record()
        r.render_batch(ds, cams, rgb=out.data_ptr(), T=None, device_out=True, **kw)
        e1.record()
        torch.cuda.synchronize()
        batch = min(batch, e0.elapsed_time(e1) / 32)
    single = []
    for c in cams[:8]:
        e0.record()
        r.render(ds, c, rgb=one.data_ptr(), T=None, device_out=True, **kw)
        e1.record()
        torch.cuda.synchronize()
        single.append(e0.elapsed_time(e1))
    _, _, st = r.render(ds, cams[0], stats=True, **kw)
    ds.free()
    return {"batch_ms_per_frame": batch, "batch_fps": 1e3 / batch, "single_ms": float(np.median(single)),
            "single_fps": 1e3 / float(np.median(single)), "V": st.visible, "P": st.tile_entries,
            "E_t": st.block_entries}


def cpu_row(lib, scene, W, H, f, ov, frames):
    kind = KINDS[scene.kind]
    p = np.ascontiguousarray(scene.params)
    axes = np.ascontiguousarray(scene.shared_axes, dtype=np.float64).reshape(9)
    bg = np.ascontiguousarray(scene.background, dtype=np.float64).reshape(3)
    h = lib.lib.ref_scene_from_params(scene.num_gaussians, kind, scene.sh_degree, p.ctypes.data,
                                      axes.ctypes.data, bg.ctypes.data)
    cam = lib.orbit_cameras(32, W, H, 4.0, f, 0.35)[0]
    cfg = make_config(degree_override=ov, threads=0)
    rgb, T = np.zeros((H, W, 3)), np.zeros((H, W, 1))
    times = []
    for i in range(frames + 1):
        t0 = time.perf_counter()
        rc = lib.lib.ref_render(h, ctypes.byref(cam), ctypes.byref(cfg), rgb.ctypes.data, T.ctypes.data)
        if rc != 0:
            raise RuntimeError(lib.err())
        if i:
            times.append(time.perf_counter() - t0)
    lib.lib.ref_scene_free(h)
    med = float(np.median(times))
    return {"cpu_ms": med * 1e3, "cpu_fps": 1.0 / med, "cpu_frames": frames, "cpu_threads": os.cpu_count()}


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "configs.json")
    r = sg.Renderer(0)
    lib = RefLib(REF_FAST_SO)
    cache, rows = {}, []
    for name, n, seed, kind, ls, W, H, f, ov in CONFIGS:
        scene = scene_for(name, n, seed, kind, ls, cache)
        row = {"config": name, "gaussians": n, "model": kind, "width": W, "height": H,
               "sh_degree_override": ov}
        row.update(gpu_rows(r, scene, W, H, f, ov))
        row.update(cpu_row(lib, scene, W, H, f, ov, 3 if n <= 100_000 else 1))
        row["gpu_over_cpu"] = row["batch_fps"] / row["cpu_fps"]
        rows.append(row)
        print(json.dumps(row), flush=True)
    with open(out_path, "w") as fh:
        json.dump({"device": torch.cuda.get_device_name(0), "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
